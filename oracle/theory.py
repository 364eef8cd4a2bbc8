"""Exact per-mode WR contraction factor — the computable form of the paper's gamma(kappa).

TEST INFRASTRUCTURE (see oracle/__init__.py).
For one eigenmode A -> lambda the error of the iteration obeys (eqn:BDF-iter-1)
    (B_k(kappa)/tau^a + lambda) e_m = (kappa/tau^a) Wup e_{m-1},
Wup the strictly upper kappa-part of B_k(kappa) without kappa.  Its spectral radius is the exact
asymptotic ratio e_{m+1}/e_m of that mode; the paper's bound eq:gamma-heat
carries an unknown constant c, so this replaces it as a pin (SURVEY §8(c) "WR rate").
For BDF1 it has the closed form kappa R/(1 - kappa R), R = (1 + tau lambda)^{-N} (Gander-Wu,
quoted in Remark 2.8).
"""
from __future__ import annotations

import numpy as np

from . import bdf, dense


def iteration_matrix(k: int, alpha: float, N: int, kappa: float, tau: float, lam: float) -> np.ndarray:
    B = dense.bk_kappa(k, alpha, N, kappa)
    low = np.tril(B)
    Wup = (B - low) / kappa
    ta = tau ** -alpha
    return np.linalg.solve(ta * B + lam * np.eye(N), kappa * ta * Wup)


def contraction_factor(k: int, alpha: float, N: int, kappa: float, tau: float, lam: float) -> float:
    return float(np.max(np.abs(np.linalg.eigvals(iteration_matrix(k, alpha, N, kappa, tau, lam)))))


def bdf1_closed_form(N: int, kappa: float, tau: float, lam: float) -> float:
    R = (1.0 + tau * lam) ** (-N)
    return kappa * R / (1.0 - kappa * R)
