"""O4: per-sine-mode scalar waveform relaxation.

TEST INFRASTRUCTURE (see oracle/__init__.py).  For FD Dirichlet operators the grid sine
modes are exact eigenvectors: A sin(p pi x) sin(q pi y) = (lambda_p + lambda_q) sin sin
(pinned in tests).  When v and every g_r lie in the span of a few modes (C4: 32 x 32), the
WR iterate stays in that span and each mode coefficient obeys the scalar version of the same
all-at-once iteration (PAPER.md:521-537 Remark "FFT" is the same decoupling).  This module
runs oracle.wr.wr_naive on the coefficient vector with a diagonal operator.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import spatial, wr


@dataclasses.dataclass
class ModalBasis:
    mx: int
    my: int
    px: np.ndarray      # x mode numbers (1-based)
    py: np.ndarray      # y mode numbers

    def eig(self) -> np.ndarray:
        lx = spatial.fd_eigenvalues(self.mx)[self.px - 1]
        if self.my == 1:
            return lx
        ly = spatial.fd_eigenvalues(self.my)[self.py - 1]
        return (ly[:, None] + lx[None, :]).ravel()       # coefficient layout [q][p]

    def synth_x(self) -> np.ndarray:
        x = (np.arange(self.mx) + 1.0) / (self.mx + 1)
        return np.sin(np.pi * np.outer(x, self.px))       # [ix][p]

    def synth_y(self) -> np.ndarray:
        y = (np.arange(self.my) + 1.0) / (self.my + 1)
        return np.sin(np.pi * np.outer(y, self.py))       # [iy][q]

    def to_grid(self, C: np.ndarray) -> np.ndarray:
        """C [..., nq*np] -> grid values [..., my*mx]: u[iy,ix] = sum_{q,p} C[q,p] sin(q pi y) sin(p pi x)."""
        Sx = self.synth_x()
        if self.my == 1:
            return C @ Sx.T
        Sy = self.synth_y()
        Cq = C.reshape(C.shape[:-1] + (len(self.py), len(self.px)))
        G = np.einsum("yq,...qp,xp->...yx", Sy, Cq, Sx)
        return G.reshape(C.shape[:-1] + (self.my * self.mx,))


def modal_problem(prob, basis: ModalBasis, v_coef: np.ndarray, g_coef: np.ndarray):
    """The coefficient-space problem: same T, N, k, kappa, alpha; M = #modes."""
    nm = len(v_coef)
    return dataclasses.replace(prob, mx=nm, my=1, v=v_coef.astype(np.complex128),
                               g=g_coef.astype(np.complex128).reshape(prob.R, nm))


class _ModalOp(wr.Operator):
    pass


def modal_wr(prob, basis: ModalBasis, v_coef, g_coef, iters: int):
    """Scalar WR per mode; returns the list of coefficient iterates [N][#modes].

    The static right-hand side needs A v: in coefficient space A is diag(eig), so f̄'s
    a_n (f(0) - A v) term is formed with the modal eigenvalues (oracle/problem.fbar would
    apply the grid stencil, so it is rebuilt here in the same way, term by term)."""
    from . import bdf
    mp = modal_problem(prob, basis, v_coef, g_coef)
    lam = basis.eig()
    N, k, tau = prob.N, prob.k, prob.tau
    Av = lam * mp.v
    f0 = prob.phi[:, 0] @ mp.g if prob.R else np.zeros_like(mp.v)
    fb = np.zeros((N, len(lam)), np.complex128)
    for n in range(1, N + 1):
        row = prob.phi[:, n] @ mp.g if prob.R else np.zeros_like(mp.v)
        a = bdf.correction_a(k, n)
        if a != 0:
            row = row + float(a) * (f0 - Av)
        for l in range(1, k - 1):
            b = bdf.correction_b(k, l, n)
            if b != 0 and prob.R:
                row = row + float(b) * tau ** l * (prob.dphi[:, l - 1] @ mp.g)
        fb[n - 1] = row
    if prob.alpha == 1.0:    # exact: zero for n > k
        bw = bdf.bdf_weights(k)
        psum = np.array([float(sum(bw[:min(n, k + 1)])) for n in range(1, N + 1)])
    else:
        psum = np.cumsum(bdf.time_weights(k, prob.alpha, N))[:N]
    F_static = fb + (tau ** -prob.alpha) * psum[:, None] * mp.v[None, :]
    op = wr.Operator(mp, diag=lam)
    return wr.wr_naive(mp, iters, op=op, F_static=F_static)
