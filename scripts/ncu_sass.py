#!/usr/bin/env python
"""Aggregate ncu per-instruction data (source page, SASS) by opcode: executed warp-instructions
and warp-stall samples.  Usage: scripts/ncu_sass.py REPORT.ncu-rep [top]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
I = {h: i for i, h in enumerate(hdr)}
inst = collections.Counter(); samp = collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr): continue
    src = r[I["Source"]].strip()
    if not src: continue
    op = src.split()[0]
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    try:
        inst[op] += int(r[I["Instructions Executed"]] or 0)
        samp[op] += int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        pass
ti = sum(inst.values()) or 1; ts = sum(samp.values()) or 1
print(f"{'op':10s} {'inst%':>7s} {'stall%':>7s}")
for op, v in samp.most_common(top):
    print(f"{op:10s} {100*inst[op]/ti:7.2f} {100*v/ts:7.2f}")
