#!/usr/bin/env python
"""Aggregate ncu source-page warp-stall samples and executed instructions by CUDA source line
(needs -lineinfo and --import-source on).  Inlined helpers are attributed to their own lines.
Usage: scripts/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, res = "", None, []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        s, ie = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    if s or ie:
        res.append((s, ie, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in res) or 1
itot = sum(x[1] for x in res) or 1
print(f"total stall samples {tot}, warp instructions {itot}")
for s, ie, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% inst {100*ie/itot:5.1f}%  {loc}: {src}")
