#!/usr/bin/env python
"""Aggregate ncu source-page warp-stall samples by CUDA source line (needs -lineinfo and
--import-source on).  Usage: scripts/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
res = collections.Counter(); inst = collections.Counter(); src = {}
for r in rows:
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    key = d.get("# Address", d.get("Line", d.get("Address", "")))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        ie = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    res[key] += s; inst[key] += ie; src[key] = d["Source"][:110]
tot = sum(res.values()) or 1
print(f"total samples {tot}")
for k, v in res.most_common(top):
    print(f"{100*v/tot:5.1f}%  inst={inst[k]:>10}  L{k}: {src[k]}")
