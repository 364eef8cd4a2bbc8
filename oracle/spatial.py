"""Finite-difference Laplacian A = -Delta_h on the unit interval / square (homogeneous
Dirichlet, h = 1/(m+1)), its DST-I eigenbasis, and shifted solves (s I + A) x = b.

TEST INFRASTRUCTURE (see oracle/__init__.py).
The paper discretizes with P1 FEM; BASELINE fixes the FD analog
(READING R-FD): A = -Delta_h, mass = I.
2D arrays are flattened [iy][ix] (x fastest).

space="fem": piecewise-linear Galerkin.
  1D: the uniform mesh of (0,1): stiffness K = (1/h) tridiag(-1, 2, -1), mass M = (h/6) tridiag(1, 4, 1).
  2D: the uniform triangulation of (0,1)^2 (Example 3 PAPER.md:1567-1575): every cell
      [x_a, x_a+1] x [y_b, y_b+1] split by the diagonal from (x_a, y_b) to (x_a+1, y_b+1) (reading
      R-FEM2D); K and M assembled triangle by triangle from the P1 element matrices.
The semi-discrete problem M U' + K U = M f~ is U' + A U = f~ with A = M^{-1} K (the discrete
Laplacian -Delta_h of PAPER.md:196-203 in its FEM form); the shifted solves of Step 2 are
(s M + K) x = M b.  Vectors are nodal coefficients of the interior nodes (homogeneous Dirichlet).
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


def fem2d_matrices(mx: int, my: int) -> tuple[sp.csc_matrix, sp.csc_matrix]:
    """(K, M) of P1 FEM on the uniform triangulation of (0,1)^2 with mx x my interior nodes
    (h_x = 1/(mx+1), h_y = 1/(my+1)), interior node (ix, iy) -> index iy*mx + ix.  Assembled element
    by element: for a triangle with vertices p_1..p_3 and area A, K_e[i,j] = (b_i b_j + c_i c_j)/(4A)
    (b_i = y_{i+1} - y_{i+2}, c_i = x_{i+2} - x_{i+1}, indices cyclic) and M_e[i,j] = (A/12)(1 + [i = j]);
    entries of boundary vertices are dropped (their coefficients are zero)."""
    hx, hy = 1.0 / (mx + 1), 1.0 / (my + 1)
    rows, cols, kv, mv = [], [], [], []

    def idx(a, b):                    # grid vertex (a, b), a = 0..mx+1 -> interior index or -1
        return (b - 1) * mx + (a - 1) if (1 <= a <= mx and 1 <= b <= my) else -1

    for a in range(mx + 1):
        for b in range(my + 1):
            for tri in (((a, b), (a + 1, b), (a + 1, b + 1)), ((a, b), (a + 1, b + 1), (a, b + 1))):
                xs = [v[0] * hx for v in tri]
                ys = [v[1] * hy for v in tri]
                area = 0.5 * abs((xs[1] - xs[0]) * (ys[2] - ys[0]) - (xs[2] - xs[0]) * (ys[1] - ys[0]))
                bb = [ys[(i + 1) % 3] - ys[(i + 2) % 3] for i in range(3)]
                cc = [xs[(i + 2) % 3] - xs[(i + 1) % 3] for i in range(3)]
                ids = [idx(*v) for v in tri]
                for i in range(3):
                    for j in range(3):
                        if ids[i] < 0 or ids[j] < 0:
                            continue
                        rows.append(ids[i])
                        cols.append(ids[j])
                        kv.append((bb[i] * bb[j] + cc[i] * cc[j]) / (4.0 * area))
                        mv.append(area / 12.0 * (2.0 if i == j else 1.0))
    n = mx * my
    K = sp.csc_matrix((kv, (rows, cols)), shape=(n, n))
    M = sp.csc_matrix((mv, (rows, cols)), shape=(n, n))
    return K, M


def solve_shifted_fem2d(shift: np.ndarray, b: np.ndarray, mx: int, my: int) -> np.ndarray:
    """x_p = (shift_p M + K)^{-1} M b_p for each row p (2D P1 FEM; sparse LU, SuperLU)."""
    K, Mm = fem2d_matrices(mx, my)
    out = np.empty(b.shape, np.complex128)
    for p in range(b.shape[0]):
        lu = spla.splu(sp.csc_matrix(shift[p] * Mm.astype(np.complex128) + K))
        out[p] = lu.solve((Mm @ b[p]).astype(np.complex128))
    return out


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
    space="fem": A u = M^{-1} K u (1D banded, 2D sparse LU).  Works on [..., M] arrays."""
    if space == "fem" and my != 1:
        K, Mm = fem2d_matrices(mx, my)
        lu = spla.splu(sp.csc_matrix(Mm.astype(np.complex128)))
        U = u.reshape(-1, mx * my)
        return np.stack([lu.solve(K @ r) for r in U.astype(np.complex128)]).reshape(u.shape)
    if space == "fem":
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
    if space == "fem" and my != 1:        # 2D FEM: M is not diagonalised by the DST (R-FEM2D)
        return solve_shifted_fem2d(shift, b, mx, my)
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
