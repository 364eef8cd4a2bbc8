"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
fused heat (graph loop, cooperative loop kernel, materialisation), 2D line path, streaming heat,
one-kernel CQ T-pass (N = 256 and 1024), CQ split (N = 128), fully modal, 1D/2D P1-FEM, Newton-WR,
residual self-check.  Checks each against the CPU oracle (test infrastructure)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import wr                                   # noqa: E402
from paper_2007_13125_b200 import inputs, pint          # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(name, prob, iters=2, solve=False, **kw):
    o = wr.wr_naive(prob, iters, dft="fft", wrap="fft")
    with pint.Plan.from_problem(prob, **kw) as p:
        if solve:
            p.run(iters)
        else:
            for _ in range(iters):
                p.iterate()
        e = rel(p.get_solution(), o[iters])
        try:
            p.residual()
        except pint.PintError:
            pass
    print(f"{name}: rel {e:.2e}", flush=True)
    assert e < 1e-10, (name, e)


run("c1 fused (cooperative loop)", inputs.config_c1(), solve=True)
run("2d fused graph loop", inputs.random_complex_problem(31, 30, 64, 3, 0.05, 1.0, R=1, seed=2), solve=True)
run("2d fused eager", inputs.random_complex_problem(31, 30, 64, 3, 0.05, 1.0, R=1, seed=2))
run("1d stream", inputs.random_complex_problem(63, 1, 256, 2, 0.1, 1.0, R=1, seed=3), stream_path=True)
run("cq N=256 one kernel", inputs.random_complex_problem(31, 20, 256, 2, 0.1, 0.6, R=1, seed=4))
run("cq N=1024 one kernel", inputs.random_complex_problem(15, 8, 1024, 2, 0.05, 0.5, R=1, seed=5))
run("cq N=128 split", inputs.random_complex_problem(31, 9, 128, 2, 0.1, 0.5, R=1, seed=6))
run("modal heat", inputs.random_complex_problem(31, 31, 64, 3, 0.05, 1.0, R=1, seed=7), modal=True, solve=True)
run("fem1d", inputs.random_complex_problem(63, 1, 64, 2, 0.05, 1.0, R=1, seed=8).with_(space="fem"))
run("fem2d cq", inputs.random_complex_problem(15, 15, 32, 2, 0.1, 0.7, R=1, seed=9).with_(space="fem"))
from oracle import nonlinear as nl                      # noqa: E402
prob = inputs.example4_allen_cahn(0.75, 2, M=63, N=32)
G, DG = nl.allen_cahn(1.0)
Us, counts = nl.newton_wr(prob, G, DG, 1)
with pint.Plan.from_problem(prob) as p:
    p.set_nonlinearity(1.0)
    c, u, st = p.newton_solve(1)
    e = rel(p.get_solution(), Us[1])
print(f"newton: rel {e:.2e}", flush=True)
assert e < 1e-10
print("sanitize cases: ok")
