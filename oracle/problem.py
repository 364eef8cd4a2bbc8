"""Corrected source f̄_n and the static part of the all-at-once right-hand side.

TEST INFRASTRUCTURE (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from . import bdf, spatial


def forcing_at(prob, n: int) -> np.ndarray:
    """f(t_n) = sum_r phi_r(t_n) g_r  (separable data from inputs.Problem)."""
    if prob.R == 0:
        return np.zeros(prob.M, np.complex128)
    return prob.phi[:, n] @ prob.g


def fbar(prob) -> np.ndarray:
    """f̄_n, n = 1..N, as rows [N][M]:
    f̄_n = f(t_n) + a_n^{(k)} (f(0) - A v) + sum_{l=1}^{k-2} b_{l,n}^{(k)} tau^l d^l f/dt^l (0)
    (PAPER.md:281-288 eqn:BDF; the same f̄ for CQ-BDFk, PAPER.md:974-982 eqn:BDF-frac).
    Corrections vanish for n >= k."""
    N, M, k, tau = prob.N, prob.M, prob.k, prob.tau
    Av = spatial.apply_A(prob.v, prob.mx, prob.my, getattr(prob, "space", "fd"))
    f0 = forcing_at(prob, 0)
    out = np.zeros((N, M), np.complex128)
    for n in range(1, N + 1):
        row = forcing_at(prob, n)
        a = bdf.correction_a(k, n)
        if a != 0:
            row = row + float(a) * (f0 - Av)
        for l in range(1, k - 1):
            b = bdf.correction_b(k, l, n)
            if b != 0 and prob.R > 0:
                dlf = prob.dphi[:, l - 1] @ prob.g
                row = row + float(b) * tau ** l * dlf
        out[n - 1] = row
    return out


def static_rhs(prob) -> np.ndarray:
    """F_static_n = f̄_n + tau^{-alpha} (sum_{j=0}^{n-1} omega_j) v, n = 1..N
    (PAPER.md:411-414 eqn:BDF-k-F last term; PAPER.md:1025-1027 eq:BDF-subdiff-F last term).
    Heat: the partial sums vanish for n > k because sum_j omega_j = 0."""
    if prob.alpha == 1.0:
        # exact rational partial sums: zero for n > k (sum_j omega_j = 0)
        w = bdf.bdf_weights(prob.k)
        psum = np.array([float(sum(w[:min(n, prob.k + 1)])) for n in range(1, prob.N + 1)])
    else:
        w = bdf.time_weights(prob.k, prob.alpha, prob.N)
        psum = np.cumsum(w)[:prob.N]      # psum[n-1] = sum_{j=0}^{n-1} omega_j
    return fbar(prob) + (prob.tau ** -prob.alpha) * psum[:, None] * prob.v[None, :]
