"""O2: the waveform-relaxation iteration solved by Algorithm 1 / Algorithm 2, literally.

TEST INFRASTRUCTURE (see oracle/__init__.py).

One iteration U_{m-1} -> U_m (PAPER.md:388-401 eqn:BDF-iter):
  F_{m-1} = F_static + kappa-wrap(U_{m-1})                (eqn:BDF-k-F / eq:BDF-subdiff-F)
  Step 1  H = S^{-1} F = V^{-1} Gamma F                   (Algorithm 1/2 step 1)
  Step 2  (d_p/tau^a + A) Q_p = H_p, p = 0..N-1           (step 2 with tau^a moved across)
  Step 3  U_m = S Q = Gamma^{-1} V Q                      (step 3)
with S = Lambda V, Lambda = diag(kappa^{-(n-1)/N}) = Gamma^{-1}, V_{lp} = e^{+2 pi i l p/N}
(Lemma 2.3, PAPER.md:433-465 and eqn:Fourier-matrix).
"""
from __future__ import annotations

import time

import numpy as np
import scipy.fft

from . import bdf, problem, spatial


def dft_matrix(N: int, sign: int) -> np.ndarray:
    """E[a, b] = exp(sign * 2 pi i ((a b) mod N) / N) with exact integer reduction."""
    a = np.arange(N)
    ang = (np.outer(a, a) % N) * (2.0 * np.pi / N)
    return np.exp(sign * 1j * ang)


def wrap_heat(prob, U_prev: np.ndarray, w: np.ndarray) -> np.ndarray:
    """(kappa/tau) sum_{j=n}^{k} omega_j U_{m-1}^{N+n-j}, n = 1..k, as rows [N][M] (zero for n > k).
    READING R-wrap: eqn:BDF-k-F is garbled; this is the
    sum that B_k(kappa) and G_m^n give."""
    N, k = prob.N, prob.k
    out = np.zeros_like(U_prev)
    c = prob.kappa / prob.tau
    for n in range(1, min(k, N) + 1):
        for j in range(n, k + 1):
            out[n - 1] += c * w[j] * U_prev[N + n - j - 1]
    return out


def wrap_cq_matrix(N: int, w: np.ndarray) -> np.ndarray:
    """Wup[n-1, s-1] = omega_{N+n-s} for s > n (else 0): the strictly upper-triangular Toeplitz
    part of the kappa-circulant B_k(kappa) of PAPER.md:1029-1038 without kappa, so that
    (Wup U)_n = sum_{j=n}^{N-1} omega_j U^{N+n-j}  (eq:BDF-subdiff-F, PAPER.md:1025-1027;
    READING R-CQwrap)."""
    Wup = np.zeros((N, N))
    for n in range(1, N + 1):
        for s in range(n + 1, N + 1):
            Wup[n - 1, s - 1] = w[N + n - s]
    return Wup


def wrap_cq_fft(U_prev: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Same product via the paper's 2N circulant embedding [[Z, W],[W, Z]] [0; U],
    as a correlation with c_s = omega_{N-s}, s = 1..N-1, using a library FFT of length 2N."""
    N = U_prev.shape[0]
    c = np.zeros(2 * N)
    c[1:N] = w[N - 1:0:-1]                   # c[s] = omega_{N-s}
    Up = np.zeros((2 * N,) + U_prev.shape[1:], np.complex128)
    Up[:N] = U_prev
    # y_n = sum_{s>=1} c_s U^{n+s}  (0-based: y[i] = sum_s c[s] U[i+s])
    cf = np.conj(np.fft.fft(c))
    y = scipy.fft.ifft(cf.reshape((2 * N,) + (1,) * (Up.ndim - 1)) * scipy.fft.fft(Up, axis=0, workers=-1),
                       axis=0, workers=-1)[:N]
    return y


def rhs(prob, U_prev: np.ndarray, F_static: np.ndarray, w: np.ndarray, wrap: str = "matrix") -> np.ndarray:
    if prob.alpha == 1.0:
        return F_static + wrap_heat(prob, U_prev, w)
    c = prob.kappa * prob.tau ** -prob.alpha
    if wrap == "matrix":
        return F_static + c * (wrap_cq_matrix(prob.N, w) @ U_prev)
    return F_static + c * wrap_cq_fft(U_prev, w)


class Operator:
    """Spatial operator of the shifted solves: FD Laplacian on the grid (DST eigen-solve), or a
    diagonal operator (per-mode scalars, used by oracle/modal.py)."""

    def __init__(self, prob, diag: np.ndarray | None = None):
        self.prob, self.diag = prob, diag

    def solve(self, shifts: np.ndarray, H: np.ndarray) -> np.ndarray:
        if self.diag is not None:
            return H / (shifts[:, None] + self.diag[None, :])
        return spatial.solve_shifted_dst(shifts, H, self.prob.mx, self.prob.my, getattr(self.prob, "space", "fd"))


def initial_guess(prob) -> np.ndarray:
    """U_0^n = v for all n (Theorem 2.7) or 0 (tables; READING R-U0)."""
    if prob.u0 == "zero":
        return np.zeros((prob.N, prob.M), np.complex128)
    return np.tile(prob.v, (prob.N, 1))


def wr_naive(prob, iters: int, U0: np.ndarray | None = None, dft: str = "naive",
             wrap: str = "matrix", op: Operator | None = None, F_static: np.ndarray | None = None,
             callback=None, keep: bool = True, timings: list | None = None) -> list[np.ndarray]:
    """Run `iters` WR iterations; returns [U_0, U_1, ..., U_iters] (each [N][M]).

    dft="naive": explicit N x N DFT matrices applied by zgemm (the default, obviously correct);
    dft="fft": library FFT (scipy.fft, pocketfft, all host threads) for the same two products (large
    sizes; pinned equal to "naive" in tests).  Eigenvalues d_p from oracle.bdf.eigenvalues (long double)."""
    N = prob.N
    w = bdf.time_weights(prob.k, prob.alpha, N)
    gam = bdf.gamma_scale(N, prob.kappa)
    d = bdf.eigenvalues(prob.k, prob.alpha, N, prob.kappa)
    shifts = d * prob.tau ** -prob.alpha
    op = op or Operator(prob)
    if F_static is None:
        F_static = problem.static_rhs(prob)
    if dft == "naive":
        Vinv = dft_matrix(N, -1) / N          # V^{-1}
        V = dft_matrix(N, +1)
    U = initial_guess(prob) if U0 is None else U0
    out = [U]
    for _ in range(iters):
        t0 = time.perf_counter()
        F = rhs(prob, U, F_static, w, wrap)
        X = gam[:, None] * F                              # Step 1a: Gamma F
        H = (Vinv @ X) if dft == "naive" else scipy.fft.fft(X, axis=0, workers=-1) / N   # Step 1b
        Q = op.solve(shifts, H)                           # Step 2
        Y = (V @ Q) if dft == "naive" else scipy.fft.ifft(Q, axis=0, workers=-1) * N     # Step 3: V Q
        U = Y / gam[:, None]                              # Step 3: Gamma^{-1}
        if timings is not None:
            timings.append(time.perf_counter() - t0)
        if keep:
            out.append(U)
        else:
            out[-1:] = [U]
        if callback is not None:
            callback(U)
    return out
