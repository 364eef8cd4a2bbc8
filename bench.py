#!/usr/bin/env python
"""Benchmark: space-time unknowns per second per WR iteration (complex128), BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A step is one waveform-relaxation iteration (S-pass + fused T-pass, all of SURVEY §8(a)'s
per-iteration rows) over the whole space-time array, inputs resident in HBM.  Default
workload C4 (2D heat 1023^2, N = 2048, BDF6, kappa = 0.01: 2.14e9 unknowns, 34.3 GB per
buffer) — the config the metric's 1/2/4/8-GPU scaling is quoted on.
For N > 1 (torchrun) each rank owns an x-mode slab (strong scaling, no data-path collective;
the update norm is all-reduced with NCCL).  Rank 0 prints one JSON line.
`--impl reference` times the CPU oracle (the reference arm of this tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time unknowns/sec per WR iteration (complex128) and HBM fraction, 1/2/4/8 GPU"
UNIT = "unknowns/s"
BYTES_PER_UNKNOWN_PASS = 32        # each pass reads 16 B and writes 16 B per unknown
FP64_FMA_PER_CLK_SM = 64           # B200 FP64 units per SM (peak = 2 x 64 x SMs x clock)


def fused_flops_per_unknown(k: int, nk: int) -> float:
    """Algorithmic FP64 flops (FMA = 2) per space-time unknown of the fused heat iteration
    (DESIGN.md §5): Step-1 synthesis ((nk-1) twiddles + DFT8 per 8 unknowns), Step-3 window
    (DFT8 + k twiddled accumulations per 8 unknowns), Step-2 solve (4 first-order recurrence
    sweeps + the final scaling)."""
    dft8 = 60.0
    synth = (6.0 * (nk - 1) + dft8) / 8.0
    window = (dft8 + 8.0 * k) / 8.0
    solve = 4 * 10.0 + 8.0
    return synth + window + solve


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def make_problem(name: str, mx: int | None = None):
    from paper_2007_13125_b200 import inputs
    if name == "C4":
        return inputs.config_c4(m=mx or 1023) if mx is None else _c4_narrow(mx)
    if name == "C3":
        return inputs.config_c3()
    if name == "C5":
        return inputs.config_c5()
    if name == "C2":
        return inputs.config_c2(k=6, kappa=1e-3)
    if name == "C1":
        return inputs.config_c1()
    raise ValueError(name)


def _c4_narrow(mx: int):
    """C4 with fewer x-modes (same N, k, kappa, line length 1023, kernels and tile shapes): profiling."""
    from paper_2007_13125_b200 import inputs
    p = inputs.config_c4()
    v = p.v.reshape(1023, 1023)[:, :mx].copy().reshape(-1)
    return p.with_(mx=mx, v=v, g=np.zeros((0, 1023 * mx), np.complex128))


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML polled every 5 ms from a
    thread (one sample is also taken on entry and exit, so sub-millisecond regions are covered);
    nvidia-smi -lms 200 when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device, self.rows, self.proc, self.nv, self.stop = device, [], None, None, threading.Event()

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(self.device)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)

    def _nvml_sample(self):
        nv, h = self.nv
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.rows.append([str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                          str(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), hex(r)]
                         + ["Active" if r & b else "Not Active" for b in bits]
                         + [f"{nv.nvmlDeviceGetPowerUsage(h) / 1000.0:.2f}"])

    def _nvml_loop(self):
        while not self.stop.wait(0.005):
            self._nvml_sample()

    def __enter__(self):
        try:
            self.nv = self._nvml_handle()
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:   # noqa: BLE001 - no NVML: fall back to nvidia-smi
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.nv:
            self._nvml_sample()
            self.stop.set()
            self.t.join(1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = list(self.rows)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        pw = [float(r[7]) for r in rows if len(r) > 7 and r[7].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None,
                "source": "nvml" if self.nv else "nvidia-smi"}


def cpu_baseline(prob_name: str, budget_s: float = 30.0, fast: bool = True):
    """The oracle (oracle.wr.wr_naive, as it stands) on host cores, one WR iteration on a bounded
    sample of the workload: same N, k, kappa, alpha and recipe on a reduced spatial grid."""
    from oracle import wr
    from paper_2007_13125_b200 import inputs
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:   # noqa: BLE001
        cores = os.cpu_count()
    if prob_name == "C4":
        prob = inputs.config_c4(m=95)
        sample = "oracle O2 (naive-DFT WR) 1 iteration on the C4 recipe at 95x95, N=2048, BDF6, kappa=0.01"
    elif prob_name == "C5":
        prob = inputs.config_c5(m=31)
        sample = "oracle O2 1 iteration on the C5 recipe at 31x31, N=1024, CQ-BDF2"
    elif prob_name == "C3":
        prob = inputs.config_c3(m=127)
        sample = "oracle O2 1 iteration on the C3 recipe at 127x127, N=256, BDF4"
    else:
        prob = make_problem(prob_name)
        sample = f"oracle O2 1 iteration on {prob_name} (full size)"
    t = []
    wr.wr_naive(prob, 1, keep=False, timings=t)
    out = {"value": prob.M * prob.N / t[0], "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": sample, "seconds": t[0], "os_cpu_count": os.cpu_count()}
    if fast:
        # SURVEY §8(d) "fast CPU" comparator: the same iteration with library FFTs for the time DFTs and
        # the CQ wrap (scipy.fft, all host threads; O(MN log N)) and the DST eigen-solves (workers=-1)
        tf = []
        wr.wr_naive(prob, 1, keep=False, timings=tf, dft="fft", wrap="fft")
        out["fast_cpu"] = {"value": prob.M * prob.N / tf[0], "unit": UNIT, "threads": os.cpu_count(),
                           "kind": "oracle O2 with dft='fft', wrap='fft' (scipy.fft workers=-1)",
                           "sample": sample, "seconds": tf[0]}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals, secs = [], []
    base = None
    for _ in range(args.warmup + args.steps):
        base = cpu_baseline(args.config, fast=False)
        vals.append(base["value"])
        secs.append(base["seconds"])
    v = vals[args.warmup:]
    value = statistics.mean(v)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(secs[args.warmup:]),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
           "data": "synthetic (seeded recipe, SURVEY §8(d))",
           "config": {"workload": f"{args.config} (oracle sample)", "sample": base["sample"]},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                            "sample": base["sample"]},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` (N > 1) started without torchrun: re-launch this script as N ranks on this
    node (one process per GPU, 127.0.0.1 rendezvous), NCCL's INFO log on stderr so the communicator
    lines show the N ranks.  Returns the launcher's exit code; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--mx", type=int, default=None, help="C4 only: fewer x-modes (profiling)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-warmup", type=int, default=2, help="untimed e2e steps first (graph re-capture after the timing-mode run, allocator)")
    ap.add_argument("--e2e-full", action="store_true",
                    help="e2e reads the FULL converged U (all N levels, pint_get_solution) to the host")
    ap.add_argument("--path", default="fused", choices=["fused", "stream"],
                    help="heat: fused one-kernel iteration (default) or the two-pass streaming one")
    ap.add_argument("--modal", action="store_true",
                    help="fully modal variant (SURVEY §8(f) 2a): DST along the line axis too, divisions instead of "
                         "line solves (heat: fused modal kernel; CQ: streaming path with a division pass)")
    ap.add_argument("--real", action="store_true",
                    help="real-data half spectrum (SURVEY §8(f) 2b; fused path): solves p <= N/2 only")
    ap.add_argument("--dst-per-iter", action="store_true",
                    help="ablation (SURVEY §8(a) A6): DST-x around every S-pass instead of hoisted (streaming)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)   # timing rule: at least 3 untimed warm-up steps (reported as run)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2007_13125_b200 import pint

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    ndev = torch.cuda.device_count()
    # one rank per GPU over NCCL; more ranks than GPUs (a 1-GPU box checking the launch path) time-slice
    # one device and use gloo for the one-double all-reduce (NCCL refuses two ranks on one device);
    # such a line is flagged "oversubscribed" and is not a scaling measurement
    oversub = world > ndev
    backend = "gloo" if oversub else "nccl"
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    rdev = dev if backend == "nccl" else torch.device("cpu")
    red = torch.zeros(1, dtype=torch.float64, device=rdev)

    def allreduce_max(x: float) -> float:
        red.fill_(x)
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
        return float(red.item())

    prob = make_problem(args.config, args.mx)
    stream = torch.cuda.Stream(device=dev)
    plan = pint.Plan(prob.mx, prob.my, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha, device=local_dev,
                     stream=stream.cuda_stream, u0_zero=(prob.u0 == "zero"), rank=rank, nranks=world,
                     allreduce_max=allreduce_max if world > 1 else None, stream_path=(args.path == "stream"),
                     dst_per_iter=args.dst_per_iter, real_data=args.real, modal=args.modal)
    v = torch.from_numpy(prob.v).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(prob.g)).to(dev) if prob.R else None
    plan.set_problem(v, g, prob.phi if prob.R else None, prob.dphi if prob.R else None)
    q0, q1 = plan.partition()
    local_unknowns = (q1 - q0) * (prob.M // prob.mx) * prob.N if prob.my > 1 else prob.M * prob.N

    # warm-up through the timed call itself: run(1) then run(W-1) builds the device-loop graphs of both
    # ping-pong parities (the timed run(K) then replays one), W iterations in total
    plan.run(1)
    plan.run(args.warmup - 1)
    launches0 = plan.info()["kernel_launches"]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
        e0.record(stream)
        upd = [plan.run(args.steps)]     # K iterations enqueued back to back, one synchronisation (pint_wr_run)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = plan.info()["kernel_launches"] - launches0
    # per-kernel durations for the roofline: the same K iterations again with CUDA events around
    # every kernel on the plan stream (event nodes inside the replayed graph; kept out of the timed
    # region above, where they would cost small problems several microseconds per iteration)
    plan.set_timing(True)
    with ClockSampler(local_dev) as clk_k:
        plan.run(args.steps)
        tm = plan.get_timing()
    plan.set_timing(False)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    total_unknowns = prob.M * prob.N
    value = total_unknowns / (ms_step / 1e3)

    # roofline of the dominant kernel (CUDA events around each launch on the plan stream)
    hbm, peak_src = peaks()
    t_avg = tm["tpass_ms"] / max(tm["tpass_launches"], 1)
    s_avg = tm["spass_ms"] / max(tm["spass_launches"], 1)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    path = plan.path()
    if path["fused"]:
        # one fused kernel per iteration (Steps 1-3 for every unknown) + a finish kernel on the
        # k-level window: FP64-ALU bound (no space-time array in HBM)
        nk = path["nk"]
        fl = fused_flops_per_unknown(prob.k, nk)
        if args.modal:   # Step 2 is one complex division (~12 flops) instead of the 48-flop line solve
            fl = fl - 48.0 + 12.0
        if args.real:   # half spectrum: N/16 + 1 of the N/8 frequency groups are solved
            fl *= (prob.N // 16 + 1) / (prob.N // 8)
        smx = 1965.0
        try:
            smx = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        except Exception:   # noqa: BLE001
            pass
        peak = 2 * FP64_FMA_PER_CLK_SM * torch.cuda.get_device_properties(dev).multi_processor_count * smx * 1e6 / 1e12
        flops_launch = fl * local_unknowns
        achieved = flops_launch / (s_avg / 1e3) / 1e12
        if os.path.exists(tf) and not args.real:   # per variant: the line path's or the modal kernel's capture
            traffic = json.load(open(tf)).get(f"{args.config}:{'modal' if args.modal else 'fused'}")
        roofline = {"bound": "alu", "kernel": "wr_modal_kernel" if args.modal else "wr_fused_kernel",
                    "achieved": achieved, "peak": peak,
                    "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                    "peak_source": f"derived: 2 x {FP64_FMA_PER_CLK_SM} FP64 FMA/clk/SM x SMs x {smx:.0f} MHz (DESIGN.md §5)",
                    "algorithmic_flops_per_unknown": fl, "algorithmic_flops_per_launch": flops_launch,
                    "passes": {"fused_ms": s_avg, "finish_ms": t_avg, "chunks_per_xmode": path["chunks"],
                               "fused_share_of_step": s_avg / ms_step,
                               "timing_pass_clocks": clk_k.summary()}}
    else:
        # streaming: each pass reads and writes the array (32 B/unknown); the CQ T-pass with the paper's
        # full-array monitor also reads U_{m-1} and writes U_m (64 B/unknown)
        full_mon = prob.alpha != 1.0
        t_bytes = (64 if full_mon else BYTES_PER_UNKNOWN_PASS) * local_unknowns
        s_bytes = BYTES_PER_UNKNOWN_PASS * local_unknowns
        dom = ("tpass", t_avg, t_bytes) if t_avg >= s_avg else ("spass", s_avg, s_bytes)
        achieved = dom[2] / (dom[1] / 1e3) / 1e9
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(f"{args.config}:{dom[0]}")
        roofline = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": dom[2],
                    "algorithmic_bytes_per_unknown": dom[2] / local_unknowns,
                    "passes": {"tpass_ms": t_avg, "spass_ms": s_avg,
                               "tpass_GBs": t_bytes / (t_avg / 1e3) / 1e9,
                               "spass_GBs": s_bytes / (s_avg / 1e3) / 1e9,
                               "iteration_GBs": (t_bytes + s_bytes) / (ms_step / 1e3) / 1e9,
                               "iteration_frac": (t_bytes + s_bytes) / (ms_step / 1e3) / 1e9 / hbm,
                               "timing_pass_clocks": clk_k.summary()}}
        if full_mon and prob.N in (256, 1024) and not args.modal:
            # the one-kernel CQ T-pass is also FP64-heavy: four length-N transforms per column
            # (5 N log2 N flops each, radix-2 count) + the pointwise Theta / D' / D W / static / monitor
            # terms (~50 flops per unknown): its fraction of the derived FP64 peak, for reference
            smx = 1965.0
            try:
                smx = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
            except Exception:   # noqa: BLE001
                pass
            fpk = 2 * FP64_FMA_PER_CLK_SM * torch.cuda.get_device_properties(dev).multi_processor_count * smx * 1e6 / 1e12
            fl = 4 * 5.0 * np.log2(prob.N) + 50.0
            roofline["secondary_alu"] = {"algorithmic_flops_per_unknown": fl,
                                         "achieved_TFLOPs": fl * local_unknowns / (t_avg / 1e3) / 1e12,
                                         "peak_TFLOPs": fpk,
                                         "frac": fl * local_unknowns / (t_avg / 1e3) / 1e12 / fpk}

    # materialisation cost: the full U_m = Gamma^{-1} V W_m of all N levels (fused: the STORE_W pass +
    # the inverse T-pass; CQ: read from the full monitor's copy), measured as pint_get_levels of one
    # non-window level into device memory (CUDA events on the plan stream; outside the timed region)
    mat = None
    if world == 1:
        lvl = torch.empty((1, prob.M), dtype=torch.complex128, device=dev)
        plan.iterate()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        plan.get_levels(0, 1, out=lvl)
        m1.record(stream)
        torch.cuda.synchronize(dev)
        mat = {"ms": m0.elapsed_time(m1), "what": "materialise U_m (all N levels) + level 1 through the DST, device"}
        del lvl

    # e2e: the public API with HOST buffers: set_problem(host v) + wr_solve(tol) + final level to host.
    # N > 1: every rank reads its own x-mode slab of the final level (pint_get_modal_levels); the
    # time is the max over ranks.
    e2e = None
    if not args.no_e2e:
        def pinned(a):   # page-locked host copy (the contract's pinned host buffers)
            t = torch.empty(a.shape, dtype=torch.complex128, pin_memory=True)
            t.numpy()[...] = a
            return t.numpy()
        vh = pinned(prob.v)
        gh = pinned(np.ascontiguousarray(prob.g)) if prob.R else None
        nlev = prob.N if args.e2e_full else 1
        if world > 1:
            qb, qe = plan.partition()
            out = torch.empty((nlev, prob.my, qe - qb), dtype=torch.complex128, pin_memory=True).numpy()
        else:
            out = torch.empty((nlev, prob.M), dtype=torch.complex128, pin_memory=True).numpy()
        steps, t_tot, its = args.e2e_steps, 0.0, 0
        out_bytes = 0
        statuses = []
        for i in range(steps + args.e2e_warmup):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            plan.set_problem(vh, gh, prob.phi if prob.R else None, prob.dphi if prob.R else None)
            it, u, st = plan.solve(prob.tol, 20, raise_on_fail=False)
            if world > 1:
                plan.get_modal_levels(prob.N - nlev, nlev, out)
            else:
                plan.get_levels(prob.N - nlev, nlev, out)
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], dtype=torch.float64, device=rdev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if i >= args.e2e_warmup:
                t_tot += dt
                its += it
                statuses.append(int(st))
            out_bytes = out.nbytes
        e2e = {"value": total_unknowns * its / t_tot, "unit": UNIT,
               "h2d_bytes_per_step": int(vh.nbytes + (prob.g.nbytes if prob.R else 0)),
               "d2h_bytes_per_step": int(out_bytes + 8 * its // steps),
               "what": f"set_problem(pinned host v) + wr_solve(tol={prob.tol:g}) ({its / steps:.1f} iterations) + "
                       + (("all N levels (pint_get_solution)" if args.e2e_full else "final time level")
                          + " to host" if world == 1 else "each rank's modal slab of the final level to host")
                       + ", per step (max over ranks); unknowns/s per WR iteration",
               "converged": all(x == pint.PINT_OK for x in statuses), "solve_status": statuses,
               "steps": steps, "warmup_steps": args.e2e_warmup}
        # self-check of the converged e2e solution against the scheme (pint_residual; outside
        # every timed region): max |residual of eqn:BDF| / max |F_static|
        try:
            r_inf, f_inf = plan.residual()
            e2e["self_check_residual_rel"] = r_inf / f_inf if f_inf > 0 else r_inf
        except pint.PintError as exc:   # CQ on the modal path, dense forcing, DST ablation: not available
            e2e["self_check_residual_rel"] = None
            e2e["self_check_note"] = str(exc)[:80]

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (seeded recipe, SURVEY §8(d))",
               "config": {"workload": args.config if args.mx is None else f"{args.config}(mx={args.mx})",
                          "grid": f"{prob.mx}x{prob.my}", "N": prob.N, "k": prob.k, "kappa": prob.kappa,
                          "alpha": prob.alpha, "unknowns": total_unknowns,
                          "parallelism": f"x-mode slabs x{world}" if world > 1 else "1 GPU",
                          "path": ("fused" if path["fused"] else "stream") + ("+dst-per-iter" if args.dst_per_iter else "")
                                  + ("+real-half-spectrum" if args.real else "") + ("+fully-modal" if args.modal else ""),
                          "l2": (f"fused: per-iteration working set (X, line constants, window, partials) "
                                 f"{(16 * (8 + 3 * prob.k) * prob.M + 192 * prob.N * prob.M // prob.my) / 1e9:.2f} GB"
                                 " > L2 126 MB, no flush needed" if path["fused"] else
                                 f"inputs > L2 ({2 * 16 * total_unknowns / 1e9:.1f} GB resident), no flush needed")},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "materialize": mat,
               "comm": ({"collective": f"{backend} all_reduce(max) of the update norm, one double per iteration",
                         "backend": backend, "oversubscribed": oversub,
                         "note": (f"{world} ranks time-slice {ndev} GPU(s): launch-path check, not a scaling "
                                  "measurement") if oversub else "one rank per GPU",
                         "data_path_bytes_per_step": 0, "allreduce_bytes_per_step": 8,
                         "partition": f"x-mode slabs (rank 0: q in [{q0}, {q1}))"} if world > 1 else None),
               "clocks": clk.summary(), "last_update": upd[-1] if upd else None}
        print(json.dumps(res))
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
