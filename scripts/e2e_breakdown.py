"""Wall-clock breakdown of the C4 e2e step (set_problem from pinned host memory, wr_solve, final level
to host) per phase, with a device synchronisation after each phase.  Diagnostic only."""
import time
import numpy as np
import torch
import bench
from paper_2007_13125_b200 import pint

prob = bench.make_problem("C4")
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
plan = pint.Plan(prob.mx, prob.my, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha, device=0,
                 stream=stream.cuda_stream, u0_zero=(prob.u0 == "zero"))


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.complex128, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


vh = pinned(prob.v)
out = torch.empty((1, prob.M), dtype=torch.complex128, pin_memory=True).numpy()
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.set_problem(vh, None, None, None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    it, u, st = plan.solve(prob.tol, 20, raise_on_fail=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    plan.get_levels(prob.N - 1, 1, out)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {i}: set_problem {1e3*(t1-t0):.3f} ms  solve {1e3*(t2-t1):.3f} ms ({it} it, {1e3*(t2-t1)/it:.3f}/it)"
          f"  get_levels {1e3*(t3-t2):.3f} ms  total {1e3*(t3-t0):.3f} ms", flush=True)
