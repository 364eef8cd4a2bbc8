"""O3: one WR iteration as a dense linear system assembled from the scheme's own
equations (tiny sizes only: N*M <= ~1000).

TEST INFRASTRUCTURE (see oracle/__init__.py).  This assembles the iteration directly from
eqn:BDF-iter / eqn:BDF-frac-iter with the wrap truncated as in
eq:BDF-subdiff-F (READING R-CQwrap), by writing every equation's terms
one by one — it does NOT use the F formula, Gamma, V or d_p — so it pins the wrap, the
static right-hand side and the diagonalization of oracle/wr.py at once.
"""
from __future__ import annotations

import numpy as np

from . import bdf, problem, spatial


def iteration_system(prob, U_prev: np.ndarray):
    """(K, rhs): K vec(U_m) = rhs, vec time-major (index (n-1)*M + i).

    Equation n (n = 1..N):  tau^{-a} sum_j omega_j U^{n-j} + A U^n = f̄_n  with
      n-j >= 1                 -> unknown U_m^{n-j}
      n-j <= 0, j <= J_wrap    -> v + kappa (U_m^{N+n-j} - U_{m-1}^{N+n-j})   (the kappa wrap)
      n-j <= 0, j >  J_wrap    -> v                                           (history)
    heat: j = 0..k, J_wrap = k (U_m^{-i} = v + kappa(...), i = 0..k-1);
    CQ:   j = 0..infinity, J_wrap = N-1, tail sum_{j>=N} omega_j = -sum_{j<N} omega_j.
    """
    N, M, tau, kap, a = prob.N, prob.M, prob.tau, prob.kappa, prob.alpha
    if getattr(prob, "space", "fd") == "fem":        # A = M^{-1} K (P1 FEM, 1D / 2D)
        K_, M_ = (x.toarray() for x in (spatial.fem_matrices(prob.mx) if prob.my == 1
                                        else spatial.fem2d_matrices(prob.mx, prob.my)))
        A = np.linalg.solve(M_, K_)
    else:
        A = spatial.laplacian_sparse(prob.mx, prob.my).toarray()
    fb = problem.fbar(prob)
    if a == 1.0:
        w = [float(x) for x in bdf.bdf_weights(prob.k)]
        jmax, jwrap = prob.k, prob.k
        tail = 0.0
    else:
        w = list(bdf.cq_weights(prob.k, a, N + 1))
        jmax, jwrap = N - 1, N - 1
        tail = -sum(w[:N])            # sum_{j >= N} omega_j  (delta_k(1)^alpha = 0)
    ta = tau ** -a
    C = np.zeros((N, N), np.complex128)       # coefficient of U_m^s in equation n
    rhs = fb.copy()
    for n in range(1, N + 1):
        for j in range(0, jmax + 1):
            i = n - j
            if i >= 1:
                C[n - 1, i - 1] += ta * w[j]
            elif j <= jwrap:
                s = N + i                      # U^{i} = v + kappa (U_m^{N+i} - U_{m-1}^{N+i})
                rhs[n - 1] -= ta * w[j] * prob.v
                C[n - 1, s - 1] += ta * w[j] * kap
                rhs[n - 1] += ta * w[j] * kap * U_prev[s - 1]
            else:
                rhs[n - 1] -= ta * w[j] * prob.v
        rhs[n - 1] -= ta * tail * prob.v
    K = np.kron(C, np.eye(M)) + np.kron(np.eye(N), A)
    return K, rhs.reshape(-1)


def dense_iteration(prob, U_prev: np.ndarray) -> np.ndarray:
    K, r = iteration_system(prob, U_prev)
    return np.linalg.solve(K, r).reshape(prob.N, prob.M)


def bk_kappa(k: int, alpha: float, N: int, kappa: float) -> np.ndarray:
    """B_k(kappa) as drawn in PAPER.md:416-428 (heat) / PAPER.md:1029-1038 (CQ):
    B[i,j] = omega_{i-j} (i >= j), kappa * omega_{N+i-j} (i < j)."""
    w = bdf.time_weights(k, alpha, N)
    B = np.zeros((N, N))
    for i in range(N):
        for j in range(N):
            B[i, j] = w[i - j] if i >= j else kappa * w[N + i - j]
    return B
