#!/usr/bin/env python
"""Summarise an ncu report (--set full) into profiles/: key throughput metrics, DRAM traffic vs
algorithmic bytes, stall mix.  Usage: scripts/ncu_summary.py REPORT.ncu-rep OUT.json --unknowns U"""
import argparse
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--unknowns", type=float, required=True, help="space-time unknowns per launch")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {"report": a.report, "note": a.note, "unknowns_per_launch": a.unknowns, "kernels": []}
    for r in rows[2:]:
        k = {"name": r[hdr.index("Kernel Name")]}
        for key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                try:
                    k[key] = float(r[i]) * SCALE.get(units[i], 1) if units[i] in SCALE else float(r[i])
                except ValueError:
                    k[key] = r[i]
        st = {hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[i])
              for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not hdr[i].endswith("not_issued") and r[i]}
        tot = sum(st.values()) or 1
        k["stall_mix_pct"] = {s: round(100 * v / tot, 1) for s, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        dram = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        k["dram_bytes_per_unknown"] = dram / a.unknowns
        k["algorithmic_bytes_per_unknown"] = 32.0
        k["achieved_GBs_under_ncu"] = dram / k["gpu__time_duration.sum"] / 1e9
        res["kernels"].append(k)
    json.dump(res, open(a.out, "w"), indent=1)
    for k in res["kernels"]:
        print(k["name"][:60], f"{k['gpu__time_duration.sum']*1e3:.3f} ms", f"dram {k['dram_bytes_per_unknown']:.1f} B/unknown",
              f"fp64 {k.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.0f}%", k["stall_mix_pct"])


if __name__ == "__main__":
    main()
