#!/usr/bin/env python
"""Per-opcode stall-reason breakdown from an ncu report's SASS source page.
Usage: scripts/ncu_stall_op.py REPORT.ncu-rep [top]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
I = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr): continue
    src = r[I["Source"]].strip()
    if not src: continue
    toks = src.split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    for h in reasons:
        try: v = int(r[I[h]] or 0)
        except ValueError: v = 0
        by[op][h] += v; tot[h] += v
T = sum(tot.values()) or 1
print("all:", ", ".join(f"{h[6:]} {100*v/T:.1f}" for h, v in tot.most_common(8)))
for op, c in sorted(by.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    print(f"{op:8s} {100*s/T:5.1f}%: " + ", ".join(f"{h[6:]} {100*v/T:.1f}" for h, v in c.most_common(4) if v))
