"""Debug: unread iterations (pruned heat T-pass) vs full-FFT and vs the oracle."""
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import wr
from paper_2007_13125_b200 import inputs, pint

def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))

cases = [("C2k3", inputs.config_c2(k=3, kappa=0.01))]
for (mx, my, N, k, kap, R) in [(200, 1, 256, 2, 0.1, 0), (200, 1, 512, 3, 0.1, 0), (100, 1, 1024, 1, 0.1, 0),
                               (100, 1, 2048, 6, 0.05, 1), (31, 40, 256, 4, 0.05, 1), (63, 20, 2048, 6, 0.01, 0)]:
    cases.append((f"{mx}x{my}N{N}k{k}R{R}", inputs.random_complex_problem(mx, my, N, k, kap, 1.0, R=R, seed=7)))
for name, prob in cases:
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    for m in (1, 2, 3):
        res = []
        for ff in (False, True):
            with pint.Plan.from_problem(prob, full_fft=ff) as p:
                ups = [p.iterate() for _ in range(m)]
                res.append((rel(p.get_solution(), o[m]), ups[-1]))
        print(f"{name} m={m} pruned err={res[0][0]:.2e} upd={res[0][1]:.3e} | full err={res[1][0]:.2e} upd={res[1][1]:.3e}", flush=True)
