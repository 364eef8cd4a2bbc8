"""O1: corrected sequential BDFk / CQ-BDFk time stepping — the WR fixed point.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Not data-parallel; this is what the
waveform relaxation converges to.
"""
from __future__ import annotations

import numpy as np

from . import bdf, problem, spatial


def _solver(prob, shift: complex, method: str):
    space = getattr(prob, "space", "fd")
    if method == "dst":
        return lambda b: spatial.solve_shifted_dst(np.array([shift]), b[None, :], prob.mx, prob.my, space)[0]
    if method == "banded":
        if prob.my != 1:
            raise ValueError("banded LU is 1D only")
        return lambda b: spatial.solve_shifted_banded(shift, b[None, :], prob.mx, space)[0]
    if method == "lu":
        lu = spatial.ShiftedLU(shift, prob.mx, prob.my)
        return lu.solve
    raise ValueError(method)


def sequential(prob, method: str | None = None) -> np.ndarray:
    """U^1..U^N as rows [N][M].

    Heat (alpha = 1), PAPER.md:281-288 (eqn:BDF):
        (1/tau) sum_{j=0}^k omega_j U^{n-j} + A U^n = f̄_n,  U^{-(k-1)} = ... = U^0 = v,
      i.e. (omega_0/tau + A) U^n = f̄_n - (1/tau) sum_{j=1}^k omega_j U^{n-j}.
    CQ (0 < alpha < 1), PAPER.md:946-950 (eqn:CQ-1) + eqn:BDF-frac:
        tau^{-alpha} sum_{j=0}^n omega_j^{(alpha)} (U^{n-j} - v) + A U^n = f̄_n,  U^0 = v,
      i.e. (omega_0/tau^a + A) U^n = f̄_n + tau^{-a} [omega_0 v - sum_{j=1}^{n} omega_j (U^{n-j} - v)].
    """
    if method is None:
        method = "banded" if prob.my == 1 else "dst"
    N, M, k, tau, a = prob.N, prob.M, prob.k, prob.tau, prob.alpha
    fb = problem.fbar(prob)
    U = np.zeros((N, M), np.complex128)
    if a == 1.0:
        w = [float(x) for x in bdf.bdf_weights(k)]
        solve = _solver(prob, w[0] / tau, method)
        hist = lambda i: prob.v if i <= 0 else U[i - 1]       # noqa: E731
        for n in range(1, N + 1):
            rhs = fb[n - 1].copy()
            for j in range(1, k + 1):
                rhs -= (w[j] / tau) * hist(n - j)
            U[n - 1] = solve(rhs)
        return U
    w = bdf.cq_weights(k, a, N + 1)
    ta = tau ** -a
    solve = _solver(prob, w[0] * ta, method)
    for n in range(1, N + 1):
        rhs = fb[n - 1] + ta * w[0] * prob.v
        # j = n term vanishes (U^0 - v = 0); j = 1..n-1 as one vectorised sum
        if n >= 2:
            hist = U[n - 2::-1] if n >= 2 else None          # U^{n-1}, ..., U^1
            rhs -= ta * (w[1:n] @ (hist - prob.v[None, :]))
        U[n - 1] = solve(rhs)
    return U
