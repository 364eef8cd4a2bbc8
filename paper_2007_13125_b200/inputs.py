"""Seeded synthetic problem data for the BASELINE configs C1..C5 and the paper's
Example 1/2 finite-difference analogs.

This module holds NO arithmetic of the method (no BDF weights, no transforms, no
solves): it only evaluates the problem data v(x), f(x, t) = sum_r phi_r(t) g_r(x)
on the grid, from the recipes in SURVEY.md §8(d) / BASELINE.json `configs`.
It is the one module shared by `oracle/` (test infrastructure) and the CUDA path
(bench / tests), as DESIGN.md §"Input recipe" states.

Grid convention (both sides): unit interval / unit square, homogeneous Dirichlet,
h = 1/(m+1), interior points x_i = (i+1) h, i = 0..m-1.  2D arrays are stored
row-major [iy][ix] (x fastest), flattened index i = iy*mx + ix.

Forcing is separable: f(t_n, x) = sum_r phi[r, n] * g[r, x], n = 0..N (t_n = n*tau),
with dphi[r, l-1] = d^l phi_r/dt^l (0) for l = 1..k-2 (needed by the Table-1
starting corrections, PAPER.md:281-288 eqn:BDF).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEEDS = {"C2": 2007131252, "C3": 2007131253, "C4": 2007131254}


@dataclasses.dataclass
class Problem:
    name: str
    mx: int            # points along x (1D: the only axis)
    my: int            # points along y (1D: 1)
    T: float
    N: int
    k: int
    kappa: float
    alpha: float       # 1.0 = heat (BDFk); (0,1) = Caputo CQ-BDFk
    v: np.ndarray      # complex128 [M]
    g: np.ndarray      # complex128 [R][M]
    phi: np.ndarray    # float64 [R][N+1], phi_r(t_n)
    dphi: np.ndarray   # float64 [R][max(k-2,0)]
    u0: str = "v"      # WR initial guess: "v" or "zero" (tables)
    tol: float = 1e-12
    space: str = "fd"  # "fd": 3/5-point stencil (BASELINE); "fem": P1 Galerkin (1D mesh / 2D uniform
                       # triangulation),
                       # v and g_r are then nodal coefficient vectors

    @property
    def dim(self) -> int:
        return 1 if self.my == 1 else 2

    @property
    def M(self) -> int:
        return self.mx * self.my

    @property
    def tau(self) -> float:
        return self.T / self.N

    @property
    def R(self) -> int:
        return int(self.g.shape[0])

    def with_(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)

    def real_part(self) -> "Problem":
        """The same record with real v and g (real-data variants of the random problems)."""
        return dataclasses.replace(self, name=self.name + "_real", v=self.v.real.astype(np.complex128),
                                   g=self.g.real.astype(np.complex128))


def grid1d(m: int) -> np.ndarray:
    h = 1.0 / (m + 1)
    return (np.arange(m, dtype=np.float64) + 1.0) * h


def _no_forcing(M: int, N: int, k: int):
    return (np.zeros((0, M), np.complex128), np.zeros((0, N + 1)),
            np.zeros((0, max(k - 2, 0))))


def config_c1(N: int = 64, M: int = 63, k: int = 2, kappa: float = 0.1) -> Problem:
    """C1: 1D heat, v = sin(pi x) + x(1-x), f from u = exp(-t) sin(pi x)(1+t):
    f = u_t - u_xx = exp(-t)(pi^2 (1+t) - t) sin(pi x)."""
    x = grid1d(M)
    T = 1.0
    v = (np.sin(np.pi * x) + x * (1 - x)).astype(np.complex128)
    t = np.arange(N + 1) * (T / N)
    phi = (np.exp(-t) * (np.pi ** 2 * (1 + t) - t))[None, :]
    g = np.sin(np.pi * x).astype(np.complex128)[None, :]
    # d^l/dt^l [e^{-t}(pi^2(1+t) - t)] at 0 = (-1)^l [pi^2 - l(pi^2 - 1)]
    dphi = np.array([[(-1) ** l * (np.pi ** 2 - l * (np.pi ** 2 - 1))
                      for l in range(1, max(k - 2, 0) + 1)]], dtype=np.float64)
    return Problem("C1", M, 1, T, N, k, kappa, 1.0, v, g, phi, dphi)


def config_c2(k: int = 2, kappa: float = 1e-1, N: int = 1024, M: int = 1023) -> Problem:
    """C2: 1D heat, v = sum_{j<=32} c_j j^-2 sin(j pi x), c ~ N(0,1) seed 2007131252, f=0."""
    x = grid1d(M)
    c = np.random.default_rng(SEEDS["C2"]).standard_normal(32)
    j = np.arange(1, 33)
    v = (np.sin(np.pi * np.outer(x, j)) @ (c / j ** 2)).astype(np.complex128)
    g, phi, dphi = _no_forcing(M, N, k)
    return Problem(f"C2_k{k}_kappa{kappa:g}", M, 1, 1.0, N, k, kappa, 1.0, v, g, phi, dphi)


def indicator_square(m: int) -> np.ndarray:
    """1 on the CLOSED square [0.25,0.75]^2, [iy][ix] flattened."""
    # exact grid test on integer indices avoids rounding at the interval ends:
    # x_i = (i+1)/(m+1) in [1/4, 3/4]  <=>  4(i+1) >= m+1 and 4(i+1) <= 3(m+1)
    i = np.arange(m)
    inside = (4 * (i + 1) >= (m + 1)) & (4 * (i + 1) <= 3 * (m + 1))
    return (inside[:, None] & inside[None, :]).astype(np.complex128).ravel()


def box5_random_field(m: int, seed: int) -> np.ndarray:
    """xi ~ N(0,1) iid on the m x m grid, smoothed by a 5x5 mean with zero padding."""
    xi = np.random.default_rng(seed).standard_normal((m, m))
    p = np.zeros((m + 4, m + 4))
    p[2:-2, 2:-2] = xi
    out = np.zeros((m, m))
    for dy in range(5):
        for dx in range(5):
            out += p[dy:dy + m, dx:dx + m]
    return (out / 25.0).astype(np.complex128).ravel()


def config_c3(m: int = 511, N: int = 256, k: int = 4, kappa: float = 0.05) -> Problem:
    """C3: 2D heat, v = indicator of [0.25,0.75]^2, f = box5x5-smoothed N(0,1) field, time-constant."""
    v = indicator_square(m)
    g = box5_random_field(m, SEEDS["C3"])[None, :]
    phi = np.ones((1, N + 1))
    dphi = np.zeros((1, max(k - 2, 0)))
    return Problem("C3", m, m, 0.5, N, k, kappa, 1.0, v, g, phi, dphi)


def smooth_modes_2d(m: int, seed: int, modes: int = 32) -> np.ndarray:
    """sum_{p,q<=modes} c_pq (p^2+q^2)^-1 sin(p pi x) sin(q pi y), c ~ N(0,1); c[p-1,q-1]."""
    x = grid1d(m)
    c = np.random.default_rng(seed).standard_normal((modes, modes))
    p = np.arange(1, modes + 1)
    C = c / (p[:, None] ** 2 + p[None, :] ** 2)
    Sx = np.sin(np.pi * np.outer(x, p))          # [ix][p]
    # v[iy, ix] = sum_{p,q} C[p,q] sin(p pi x_ix) sin(q pi y_iy)
    V = Sx @ C @ Sx.T                              # [ix][iy]
    return V.T.astype(np.complex128).ravel()


def c4_mode_coefficients(seed: int = SEEDS["C4"], modes: int = 32) -> np.ndarray:
    c = np.random.default_rng(seed).standard_normal((modes, modes))
    p = np.arange(1, modes + 1)
    return c / (p[:, None] ** 2 + p[None, :] ** 2)


def config_c4(m: int = 1023, N: int = 2048, k: int = 6, kappa: float = 0.01) -> Problem:
    """C4: 2D heat, smooth seeded Fourier-mode v (32x32 modes), f = 0."""
    v = smooth_modes_2d(m, SEEDS["C4"])
    g, phi, dphi = _no_forcing(m * m, N, k)
    return Problem("C4", m, m, 1.0, N, k, kappa, 1.0, v, g, phi, dphi)


def config_c5(m: int = 511, N: int = 1024, k: int = 2, kappa: float = 0.05,
              alpha: float = 0.5) -> Problem:
    """C5: 2D subdiffusion (Caputo alpha=0.5), CQ-BDF2, v = indicator, f = 0."""
    v = indicator_square(m)
    g, phi, dphi = _no_forcing(m * m, N, k)
    return Problem("C5", m, m, 1.0, N, k, kappa, alpha, v, g, phi, dphi)


def example1_fd(k: int, M: int = 999, N: int = 100, kappa: float = 0.5) -> Problem:
    """FD analog of the paper's Example 1: T=0.5, v = chi_(0,1/2),
    f = e^t cos x, U_0 = 0."""
    x = grid1d(M)
    T = 0.5
    v = (x < 0.5).astype(np.complex128)
    t = np.arange(N + 1) * (T / N)
    phi = np.exp(t)[None, :]
    g = np.cos(x).astype(np.complex128)[None, :]
    dphi = np.ones((1, max(k - 2, 0)))
    return Problem(f"E1_k{k}", M, 1, T, N, k, kappa, 1.0, v, g, phi, dphi, u0="zero")


def example1_fem(k: int, M: int = 999, N: int = 100, kappa: float = 0.5) -> Problem:
    """The paper's Example 1 in its own discretisation (P1 FEM):
    v_h and f~ = the nodal interpolants of chi_(0,1/2) and e^t cos x (READING R-FEMdata), U_0 = 0."""
    return example1_fd(k, M, N, kappa).with_(name=f"E1fem_k{k}", space="fem")


def example3_fem(k: int = 3, m: int = 63, N: int = 128, T: float = 0.1, kappa: float = 0.05,
                 alpha: float = 0.5) -> Problem:
    """The paper's Example 3 in its own discretisation on a reduced grid: 2D
    subdiffusion on the uniform triangulation of the unit square (P1 FEM, space="fem", m x m interior
    nodes), v = chi_{(0,1/2)^2}, f = cos(t) chi_{(1/2,1)^2}, as nodal interpolants of the OPEN sets
    (READING R-FEMdata); the paper uses h = 1e-2, tau = 1e-3 (Figure 3)."""
    x = grid1d(m)
    X, Y = np.meshgrid(x, x)                       # [iy][ix]
    v = ((X < 0.5) & (Y < 0.5)).astype(np.complex128).reshape(-1)
    g = ((X > 0.5) & (Y > 0.5)).astype(np.complex128).reshape(1, -1)
    t = np.arange(N + 1) * (T / N)
    phi = np.cos(t)[None, :]
    nd = max(k - 2, 0)
    dphi = np.array([[[1.0, 0.0, -1.0, 0.0][l % 4] for l in range(1, nd + 1)]]).reshape(1, nd)   # cos^(l)(0)
    return Problem(f"E3fem_k{k}_a{alpha}", m, m, T, N, k, kappa, alpha, v, g, phi, dphi, space="fem")


def example2_fd(k: int, M: int = 999, N: int = 100, kappa: float = 0.1,
                alpha: float = 0.5) -> Problem:
    """FD analog of the paper's Example 2: T=0.1, alpha=0.5,
    v = discrete delta at x=1/2 (e_{500}/h), f = 0, U_0 = 0."""
    h = 1.0 / (M + 1)
    v = np.zeros(M, np.complex128)
    v[(M + 1) // 2 - 1] = 1.0 / h
    g, phi, dphi = _no_forcing(M, N, k)
    return Problem(f"E2_k{k}", M, 1, 0.1, N, k, kappa, alpha, v, g, phi, dphi, u0="zero")


def example4_allen_cahn(alpha: float, k: int, M: int = 999, N: int = 100, T: float = 0.4,
                        kappa: float = 0.1, eps: float = 1.0, discrete: bool = False) -> Problem:
    """Example 4 (Table 4): Allen-Cahn nonlinearity g(u) = (u^3 - u)/eps^2 on
    (0,1) with the forcing that makes u = t^2/Gamma(3) sin(2 pi x) exact (continuous operators):
      f = [t^{2-a}/Gamma(3-a) + (2 pi^2 - 1/(2 eps^2)) t^2] sin(2 pi x) + t^6/(8 eps^2) sin^3(2 pi x),
    v = u(0) = 0.  Separable with R = 2; d^l phi/dt^l (0) = 0 for l = 1..k-2 when a < 1 (k <= 3 in
    Table 4), and phi_1'(0) = 1 for a = 1.  The nonlinearity itself is not part of this record.
    discrete=True replaces 4 pi^2 by the FD eigenvalue (4/h^2) sin^2(pi h) of sin(2 pi x), so that
    the exact solution also solves the semi-discrete problem (time-discretisation error only)."""
    x = grid1d(M)
    t = np.arange(N + 1) * (T / N)
    s1 = np.sin(2 * math.pi * x)
    g = np.stack([s1, s1 ** 3]).astype(np.complex128)
    h = 1.0 / (M + 1)
    lam = (4.0 / h ** 2) * math.sin(math.pi * h) ** 2 if discrete else 4 * math.pi ** 2
    phi = np.stack([t ** (2 - alpha) / math.gamma(3 - alpha) + (lam / 2 - 0.5 / eps ** 2) * t ** 2,
                    t ** 6 / (8 * eps ** 2)])
    nd = max(k - 2, 0)
    dphi = np.zeros((2, nd))
    if nd >= 1 and alpha == 1.0:
        dphi[0, 0] = 1.0                        # d/dt t^{2-a}/Gamma(3-a) at 0 for a = 1
    if nd >= 2:
        dphi[0, 1] = (2.0 if alpha == 1.0 else 0.0) + 2 * (lam / 2 - 0.5 / eps ** 2)
    return Problem(f"E4_a{alpha}_k{k}", M, 1, T, N, k, kappa, alpha, np.zeros(M, np.complex128), g, phi, dphi)


def allen_cahn_exact(prob, n: int) -> np.ndarray:
    """u(t_n) = t_n^2/2 sin(2 pi x) of Example 4 (for error measurement)."""
    t = n * prob.tau
    return (t * t / 2.0 * np.sin(2 * math.pi * grid1d(prob.mx))).astype(np.complex128)


def random_complex_problem(mx: int, my: int, N: int, k: int, kappa: float, alpha: float,
                           R: int = 2, seed: int = 1, T: float = 1.0) -> Problem:
    """Generic complex-valued data (exercises the complex path)."""
    rng = np.random.default_rng(seed)
    M = mx * my
    v = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    g = rng.standard_normal((R, M)) + 1j * rng.standard_normal((R, M))
    t = np.arange(N + 1) * (T / N)
    freqs = rng.uniform(0.5, 3.0, R)
    phi = np.cos(np.outer(freqs, t)) + 0.5
    # d^l/dt^l [cos(w t) + 0.5] at 0
    dphi = np.array([[(math.cos(l * math.pi / 2) * w ** l) for l in range(1, max(k - 2, 0) + 1)]
                     for w in freqs]).reshape(R, max(k - 2, 0))
    return Problem(f"rand_{mx}x{my}_N{N}_k{k}", mx, my, T, N, k, kappa, alpha,
                   v.astype(np.complex128), g.astype(np.complex128), phi, dphi)


def random_dense_forcing(mx: int, my: int, N: int, k: int, kappa: float, alpha: float, seed: int = 3,
                         T: float = 1.0):
    """A non-separable forcing f(t_n, x) (random, complex) for pint_set_problem, and the same data as
    a separable record for the oracle: g_r = f(t_r), phi_r(t_n) = [n = r] (r = 0..N), plus one source
    per derivative d^l f/dt^l (0) (l = 1..k-2) with phi = 0, dphi = e_l.
    Returns (problem, f [N][M] = f(t_1..t_N), f0 = f(0), fderiv [k-2][M])."""
    rng = np.random.default_rng(seed)
    M = mx * my
    F = rng.standard_normal((N + 1, M)) + 1j * rng.standard_normal((N + 1, M))
    nd = max(k - 2, 0)
    D = rng.standard_normal((nd, M)) + 1j * rng.standard_normal((nd, M))
    v = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    g = np.concatenate([F, D]).astype(np.complex128)
    R = N + 1 + nd
    phi = np.zeros((R, N + 1))
    phi[np.arange(N + 1), np.arange(N + 1)] = 1.0
    dphi = np.zeros((R, nd))
    for l in range(nd):
        dphi[N + 1 + l, l] = 1.0
    prob = Problem(f"dense_{mx}x{my}_N{N}_k{k}", mx, my, T, N, k, kappa, alpha, v.astype(np.complex128), g, phi, dphi)
    return prob, np.ascontiguousarray(F[1:]), np.ascontiguousarray(F[0]), np.ascontiguousarray(D)


CONFIGS = {
    "C1": config_c1,
    "C2": config_c2,
    "C3": config_c3,
    "C4": config_c4,
    "C5": config_c5,
}
