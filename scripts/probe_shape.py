"""Probe: fused-kernel efficiency vs line length at C4's N and k (device time per iteration)."""
import sys, json
import numpy as np
import torch
from paper_2007_13125_b200 import inputs, pint
sys.path.insert(0, ".")
import bench
for (mx, my) in [(1023, 1023), (1023, 511), (1023, 255)]:
    prob = inputs.random_complex_problem(mx, my, 2048, 6, 0.01, 1.0, R=0, seed=3)
    st = torch.cuda.Stream()
    with pint.Plan.from_problem(prob, stream=st.cuda_stream) as p:
        for _ in range(3): p.iterate()
        p.set_timing(True)
        for _ in range(5): p.iterate()
        tm = p.get_timing()
        fused = tm["spass_ms"] / tm["spass_launches"]
        fl = bench.fused_flops_per_unknown(prob.k, p.path()["nk"])
        tf = fl * prob.M * prob.N / (fused / 1e3) / 1e12
        print(json.dumps({"mx": mx, "my": my, "fused_ms": fused, "TFLOPs": tf, "frac": tf / 37.22496, "chunks": p.path()["chunks"]}))
