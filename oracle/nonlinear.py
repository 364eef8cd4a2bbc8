"""O5: semilinear (sub)diffusion — the modified CQ-BDFk / BDFk scheme solved sequentially, and
Algorithm 3 (Newton's iteration with waveform-relaxation inner solves), literally.

TEST INFRASTRUCTURE (see oracle/__init__.py).  1D FD operator A = -Delta_h (READING R-FD).

  Scheme (eqn:BDF-CQ-m-r):
      dbar^a U^n + A U^n + g(U^n) = fbar_n,  U^n = v (n <= 0),
      fbar_n = f(t_n) + a_n (f(0) - A v - g(v)) + sum_l b_{l,n} tau^l d^l f/dt^l (0)
  Newton (eqn:BDF-CQ-m-r-N): U_l = U_{l-1} + W_l with
      (dbar^a + A) W^n + g'(Ubar_{l-1}) W^n = fbar_n - (dbar^a + A) U_{l-1}^n - g(U_{l-1}^n),  W^{<=0} = 0,
      Ubar = (1/N) sum_{n=1}^N U_{l-1}^n
    READING R-NL-sign: the print has "- g'(Ubar) W"; the Jacobian of dbar U + A U + g(U) is
    dbar + A + g'(U), so the sign is +.
  Inner WR (eqn:BDF-CQ-m-r-N-w): the kappa-wrap iteration of Algorithm 1/2 for
    this linear system (zero initial value, dense right-hand side, operator A + diag(g'(Ubar))),
    stopped when max_n ||W_{l,m}^n - W_{l,m-1}^n||_inf < tol, W_{l,0} = 0.
  Algorithm 3: U_0^n = v for all n.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import scipy.linalg

from . import bdf, problem, spatial, wr


def allen_cahn(eps: float):
    """g(u) = (u^3 - u) / eps^2 and g'(u) (Example 4)."""
    e2 = eps * eps
    return (lambda u: (u ** 3 - u) / e2), (lambda u: (3.0 * u ** 2 - 1.0) / e2)


def fbar_nl(prob, g) -> np.ndarray:
    """fbar_n, n = 1..N: the linear f̄ (oracle.problem.fbar, which carries a_n (f(0) - A v)) plus the
    nonlinear part of the starting correction, -a_n g(v)."""
    out = problem.fbar(prob)
    gv = g(prob.v)
    for n in range(1, prob.N + 1):
        a = bdf.correction_a(prob.k, n)
        if a != 0:
            out[n - 1] -= float(a) * gv
    return out


def dbar(prob, U: np.ndarray) -> np.ndarray:
    """dbar^a U^n, n = 1..N, with U^{<=0} = v (eqn:BDF P:281-288; eqn:CQ-1 P:946-950):
    heat (1/tau) sum_{j=0}^{k} omega_j U^{n-j};  CQ tau^{-a} sum_{j=0}^{n} omega_j (U^{n-j} - v)."""
    N, k, tau, a = prob.N, prob.k, prob.tau, prob.alpha
    out = np.zeros_like(U)
    if a == 1.0:
        w = [float(x) for x in bdf.bdf_weights(k)]
        for n in range(1, N + 1):
            for j in range(0, k + 1):
                out[n - 1] += (w[j] / tau) * (U[n - j - 1] if n - j >= 1 else prob.v)
        return out
    w = bdf.cq_weights(k, a, N + 1)
    D = U - prob.v[None, :]
    for n in range(1, N + 1):
        out[n - 1] = tau ** -a * (w[:n] @ D[n - 1::-1])       # j = 0..n-1 (j = n: U^0 - v = 0)
    return out


def residual(prob, U: np.ndarray, g, fb: np.ndarray) -> np.ndarray:
    """R^n = fbar_n - dbar^a U^n - A U^n - g(U^n)  (right-hand side of eqn:BDF-CQ-m-r-N)."""
    AU = np.stack([spatial.apply_A(U[n], prob.mx, 1) for n in range(prob.N)])
    return fb - dbar(prob, U) - AU - g(U)


def _banded(shift, c: np.ndarray, b: np.ndarray, m: int) -> np.ndarray:
    """(shift + A + diag(c)) x = b, 1D, LAPACK banded LU."""
    h2 = spatial.hstep(m) ** 2
    ab = np.zeros((3, m), dtype=np.complex128)
    ab[0, 1:] = -1.0 / h2
    ab[1, :] = 2.0 / h2 + shift + c
    ab[2, :-1] = -1.0 / h2
    return scipy.linalg.solve_banded((1, 1), ab, b.T).T


class VarOperator:
    """Shifted solves with the spatially varying Newton coefficient: (s_p + A + diag(c)) Q_p = H_p.
    The DST no longer diagonalises the operator, so each is a banded solve."""

    def __init__(self, prob, c: np.ndarray):
        self.prob, self.c = prob, np.asarray(c, np.complex128)

    def solve(self, shifts: np.ndarray, H: np.ndarray) -> np.ndarray:
        return np.stack([_banded(shifts[p], self.c, H[p], self.prob.mx) for p in range(len(shifts))])


def sequential_nl(prob, g, dg, tol: float = 1e-15, maxit: int = 50) -> np.ndarray:
    """U^1..U^N of eqn:BDF-CQ-m-r by stepping, each step solved by Newton's method on
    (w_0 tau^-a + A) U + g(U) = rhs_n (history terms known)."""
    if prob.my != 1:
        raise ValueError("1D only")
    N, k, tau, a = prob.N, prob.k, prob.tau, prob.alpha
    fb = fbar_nl(prob, g)
    U = np.zeros((N, prob.M), np.complex128)
    if a == 1.0:
        w = [float(x) for x in bdf.bdf_weights(k)]
        s0 = w[0] / tau
    else:
        w = bdf.cq_weights(k, a, N + 1)
        s0 = w[0] * tau ** -a
    for n in range(1, N + 1):
        rhs = fb[n - 1].copy()
        if a == 1.0:
            for j in range(1, k + 1):
                rhs -= (w[j] / tau) * (U[n - j - 1] if n - j >= 1 else prob.v)
        else:
            rhs += tau ** -a * w[0] * prob.v
            if n >= 2:
                rhs -= tau ** -a * (w[1:n] @ (U[n - 2::-1] - prob.v[None, :]))
        x = U[n - 2].copy() if n >= 2 else prob.v.astype(np.complex128).copy()
        for _ in range(maxit):
            F = s0 * x + spatial.apply_A(x, prob.mx, 1) + g(x) - rhs
            dx = _banded(s0, dg(x), F[None, :], prob.mx)[0]
            x = x - dx
            if np.max(np.abs(dx)) <= tol * max(1.0, np.max(np.abs(x))):
                break
        U[n - 1] = x
    return U


def newton_wr(prob, g, dg, outer: int, inner_tol: float = 1e-12, max_inner: int = 60):
    """Algorithm 3.  Returns ([U_0, U_1, ..., U_outer], [m_1, ..., m_outer])
    with m_l the number of inner WR iterations of Newton step l."""
    if prob.my != 1:
        raise ValueError("1D only")
    fb = fbar_nl(prob, g)
    lin = dataclasses.replace(prob, u0="zero")          # the inner WR runs on W, W^{<=0} = 0
    U = np.tile(prob.v.astype(np.complex128), (prob.N, 1))
    Us, counts = [U.copy()], []
    for _ in range(outer):
        c = dg(U.mean(axis=0))
        R = residual(prob, U, g, fb)
        op = VarOperator(prob, c)
        W = np.zeros_like(U)
        m = 0
        while m < max_inner:
            Wn = wr.wr_naive(lin, 1, U0=W, op=op, F_static=R, dft="fft", wrap="fft")[1]
            m += 1
            upd = float(np.max(np.abs(Wn - W)))
            W = Wn
            if upd < inner_tol:
                break
        U = U + W
        Us.append(U.copy())
        counts.append(m)
    return Us, counts


def l2_error(prob, a: np.ndarray, b: np.ndarray) -> float:
    """Discrete L2(Omega) norm sqrt(h sum |a - b|^2) (READING R-norm; e_l^N of PAPER.md:1742)."""
    return float(math.sqrt(spatial.hstep(prob.mx) * np.sum(np.abs(a - b) ** 2)))
