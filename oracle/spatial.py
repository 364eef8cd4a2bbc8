"""Finite-difference Laplacian A = -Delta_h on the unit interval / square (homogeneous
Dirichlet, h = 1/(m+1)), its DST-I eigenbasis, and shifted solves (s I + A) x = b.

TEST INFRASTRUCTURE (see oracle/__init__.py).
The paper discretizes with P1 FEM; BASELINE fixes the FD analog
(READING R-FD): A = -Delta_h, mass = I.
2D arrays are flattened [iy][ix] (x fastest).

space="fem" (1D only): piecewise-linear Galerkin on the uniform mesh
(PAPER.md:1374-1375), stiffness K = (1/h) tridiag(-1, 2, -1), mass M = (h/6) tridiag(1, 4, 1).
The semi-discrete problem M U' + K U = M f~ is U' + A U = f~ with A = M^{-1} K (the discrete
Laplacian -Delta_h of PAPER.md:196-203 in its FEM form); the shifted solves of Step 2 are
(s M + K) x = M b.  Vectors are nodal coefficients.
"""
from __future__ import annotations

import numpy as np
import scipy.fft
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def hstep(m: int) -> float:
    return 1.0 / (m + 1)


def fem_matrices(m: int) -> tuple[sp.csc_matrix, sp.csc_matrix]:
    """(K, M) of P1 FEM on the uniform mesh of (0,1), h = 1/(m+1), interior nodes."""
    h = hstep(m)
    e = np.ones(m - 1)
    K = sp.diags([-e, 2 * np.ones(m), -e], [-1, 0, 1]) / h
    Mm = sp.diags([e, 4 * np.ones(m), e], [-1, 0, 1]) * (h / 6)
    return sp.csc_matrix(K), sp.csc_matrix(Mm)


def _banded3(lo, d, up, b: np.ndarray) -> np.ndarray:
    """Tridiagonal solve (LAPACK banded LU), right-hand sides along the last axis."""
    m = len(d)
    ab = np.zeros((3, m), dtype=np.result_type(lo, d, up, np.complex128))
    ab[0, 1:] = up
    ab[1, :] = d
    ab[2, :-1] = lo
    return scipy.linalg.solve_banded((1, 1), ab, np.moveaxis(b, -1, 0)).T if b.ndim > 1 else \
        scipy.linalg.solve_banded((1, 1), ab, b)


def apply_A(u: np.ndarray, mx: int, my: int, space: str = "fd") -> np.ndarray:
    """A u with the 3-point (1D, my == 1) or 5-point (2D) stencil, zero Dirichlet values.
    space="fem": A u = M^{-1} K u (1D).  Works on [..., M] arrays."""
    if space == "fem":
        if my != 1:
            raise ValueError("P1 FEM is 1D only")
        K, _ = fem_matrices(mx)
        h = hstep(mx)
        Ku = (K @ u.reshape(-1, mx).T).T
        Mu = _banded3(np.full(mx - 1, h / 6), np.full(mx, 4 * h / 6), np.full(mx - 1, h / 6), Ku)
        return Mu.reshape(u.shape)
    if my == 1:
        h2 = hstep(mx) ** 2
        p = np.zeros(u.shape[:-1] + (mx + 2,), dtype=u.dtype)
        p[..., 1:-1] = u
        return (2 * p[..., 1:-1] - p[..., :-2] - p[..., 2:]) / h2
    hx2, hy2 = hstep(mx) ** 2, hstep(my) ** 2
    U = u.reshape(u.shape[:-1] + (my, mx))
    p = np.zeros(u.shape[:-1] + (my + 2, mx + 2), dtype=u.dtype)
    p[..., 1:-1, 1:-1] = U
    c = p[..., 1:-1, 1:-1]
    out = (2 * c - p[..., 1:-1, :-2] - p[..., 1:-1, 2:]) / hx2 \
        + (2 * c - p[..., :-2, 1:-1] - p[..., 2:, 1:-1]) / hy2
    return out.reshape(u.shape)


def laplacian_sparse(mx: int, my: int) -> sp.csc_matrix:
    """Sparse A (for LU-based solves and dense tiny systems)."""
    def lap1(m):
        h2 = hstep(m) ** 2
        return sp.diags([-np.ones(m - 1), 2 * np.ones(m), -np.ones(m - 1)], [-1, 0, 1]) / h2
    if my == 1:
        return sp.csc_matrix(lap1(mx))
    return sp.csc_matrix(sp.kron(sp.identity(my), lap1(mx)) + sp.kron(lap1(my), sp.identity(mx)))


def fd_eigenvalues(m: int) -> np.ndarray:
    """lambda_j = (4/h^2) sin^2(j pi h / 2), j = 1..m: eigenvalues of the 3-point -d^2/dx^2,
    eigenvectors sin(j pi x_i) (textbook; pinned in tests against the dense matrix)."""
    h = hstep(m)
    j = np.arange(1, m + 1)
    return (4.0 / h ** 2) * np.sin(j * np.pi * h / 2) ** 2


def fem_eigenvalues(m: int) -> np.ndarray:
    """Eigenvalues of A = M^{-1} K (P1 FEM, 1D): lambda_j = K_j / M_j with the DST-I eigenvalues
    K_j = (4/h) sin^2(j pi h/2) of K and M_j = (h/3)(2 + cos(j pi h)) of M (both Toeplitz
    tridiagonal, same sine eigenvectors), i.e. (4/h^2) s^2 / (1 - (2/3) s^2), s = sin(j pi h/2).
    Pinned in tests against the generalised eigenproblem K x = lambda M x (LAPACK)."""
    h = hstep(m)
    s2 = np.sin(np.arange(1, m + 1) * np.pi * h / 2) ** 2
    return (4.0 / h ** 2) * s2 / (1.0 - 2.0 * s2 / 3.0)


def eigenvalues(m: int, space: str = "fd") -> np.ndarray:
    return fem_eigenvalues(m) if space == "fem" else fd_eigenvalues(m)


def dst1(x: np.ndarray, axis: int = -1) -> np.ndarray:
    """Orthonormal DST-I, S_{qi} = sqrt(2/(m+1)) sin(pi q i/(m+1)); S = S^T = S^{-1}.
    Library primitive (scipy.fft), applied separately to real and imaginary parts."""
    if np.iscomplexobj(x):
        return (scipy.fft.dst(x.real, type=1, norm="ortho", axis=axis, workers=-1)
                + 1j * scipy.fft.dst(x.imag, type=1, norm="ortho", axis=axis, workers=-1))
    return scipy.fft.dst(x, type=1, norm="ortho", axis=axis, workers=-1)


def dst1_matrix(m: int) -> np.ndarray:
    i = np.arange(1, m + 1)
    return np.sqrt(2.0 / (m + 1)) * np.sin(np.pi * np.outer(i, i) / (m + 1))


def solve_shifted_dst(shift: np.ndarray, b: np.ndarray, mx: int, my: int, space: str = "fd") -> np.ndarray:
    """x_p = (shift_p I + A)^{-1} b_p for each row p of b [P][M], by DST eigen-decomposition
    (exact in the shift: the shift is added to each eigenvalue, never rounded into 2/h^2;
    SURVEY §8(c) item 15).  shift: [P] complex.  space="fem": A = M^{-1} K (1D)."""
    shift = np.asarray(shift)
    if my == 1:
        lam = eigenvalues(mx, space)
        bh = dst1(b, axis=-1)
        return dst1(bh / (shift[:, None] + lam[None, :]), axis=-1)
    lx, ly = fd_eigenvalues(mx), fd_eigenvalues(my)
    B = b.reshape(b.shape[0], my, mx)
    Bh = dst1(dst1(B, axis=2), axis=1)
    Xh = Bh / (shift[:, None, None] + ly[None, :, None] + lx[None, None, :])
    return dst1(dst1(Xh, axis=2), axis=1).reshape(b.shape)


def solve_shifted_banded(shift: complex, b: np.ndarray, m: int, space: str = "fd") -> np.ndarray:
    """1D (shift I + A) x = b by LAPACK banded LU with partial pivoting (scipy solve_banded).
    Note: this rounds 2/h^2 + shift once (the plain form).
    space="fem": (shift M + K) x = M b."""
    if space == "fem":
        h = hstep(m)
        Mb = (b * (4 * h / 6)).astype(np.complex128)
        Mb[..., 1:] += b[..., :-1] * (h / 6)
        Mb[..., :-1] += b[..., 1:] * (h / 6)
        off = np.full(m - 1, shift * h / 6 - 1.0 / h, dtype=np.complex128)
        return _banded3(off, np.full(m, shift * 4 * h / 6 + 2.0 / h, dtype=np.complex128), off, Mb)
    h2 = hstep(m) ** 2
    ab = np.zeros((3, m), dtype=np.complex128)
    ab[0, 1:] = -1.0 / h2
    ab[1, :] = 2.0 / h2 + shift
    ab[2, :-1] = -1.0 / h2
    return scipy.linalg.solve_banded((1, 1), ab, b.T).T


class ShiftedLU:
    """Sparse LU of (shift I + A) for repeated solves (sequential stepping, 2D)."""

    def __init__(self, shift: complex, mx: int, my: int):
        A = laplacian_sparse(mx, my).astype(np.complex128)
        self.lu = spla.splu(sp.csc_matrix(A + shift * sp.identity(mx * my, format="csc")))

    def solve(self, b: np.ndarray) -> np.ndarray:
        return self.lu.solve(b)
