"""BDFk generating polynomial, Table-1 starting corrections, CQ weights, eigenvalues.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain exact / extended-precision code.
"""
from __future__ import annotations

from fractions import Fraction as Fr
from math import comb

import mpmath
import numpy as np


def bdf_weights(k: int) -> list[Fr]:
    """omega_0..omega_k of delta_k(zeta) = sum_{l=1}^k (1-zeta)^l / l = sum_j omega_j zeta^j.

    PAPER.md:289-296 (eqn:bdf-gen).  Exact binomial expansion in rationals.
    """
    if not 1 <= k <= 6:
        raise ValueError("k must be in 1..6 (PAPER.md:278)")
    w = [Fr(0)] * (k + 1)
    for l in range(1, k + 1):
        for j in range(l + 1):
            w[j] += Fr(comb(l, j) * (-1) ** j, l)
    return w


def delta_eval(k: int, zeta):
    """delta_k(zeta) = sum_{l=1}^k (1-zeta)^l / l, any numeric type."""
    return sum((1 - zeta) ** l / l for l in range(1, k + 1))


# Table 1 (tab:anbn), transcribed as printed.  a[k] = [a_1..a_{k-1}],
# b[k][l] = [b_{l,1}..b_{l,k-1}].  Entries not printed (n >= k) are zero.
# READING R-Table1: b^{(5)}_{3,1} is printed +1/720; the exact
# moment conditions that every other one of the 55 entries satisfies give -1/720, which
# is used here.  No BASELINE config exercises it (their f has no time derivatives).
_TABLE1_A = {
    1: [],
    2: [Fr(1, 2)],
    3: [Fr(11, 12), Fr(-5, 12)],
    4: [Fr(31, 24), Fr(-7, 6), Fr(3, 8)],
    5: [Fr(1181, 720), Fr(-177, 80), Fr(341, 240), Fr(-251, 720)],
    6: [Fr(2837, 1440), Fr(-2543, 720), Fr(17, 5), Fr(-1201, 720), Fr(95, 288)],
}
_TABLE1_B = {
    1: {},
    2: {},
    3: {1: [Fr(1, 12), Fr(0)]},
    4: {1: [Fr(1, 6), Fr(-1, 12), Fr(0)],
        2: [Fr(0), Fr(0), Fr(0)]},
    5: {1: [Fr(59, 240), Fr(-29, 120), Fr(19, 240), Fr(0)],
        2: [Fr(1, 240), Fr(-1, 240), Fr(0), Fr(0)],
        3: [Fr(-1, 720), Fr(0), Fr(0), Fr(0)]},   # printed +1/720, see reading above
    6: {1: [Fr(77, 240), Fr(-7, 15), Fr(73, 240), Fr(-3, 40), Fr(0)],
        2: [Fr(1, 96), Fr(-1, 60), Fr(1, 160), Fr(0), Fr(0)],
        3: [Fr(-1, 360), Fr(1, 720), Fr(0), Fr(0), Fr(0)],
        4: [Fr(0), Fr(0), Fr(0), Fr(0), Fr(0)]},
}
TABLE1_B5_31_AS_PRINTED = Fr(1, 720)


def table1(k: int):
    """(a, b): a[n-1] = a_n^{(k)}, b[l][n-1] = b_{l,n}^{(k)} for n=1..k-1, l=1..k-2."""
    return list(_TABLE1_A[k]), {l: list(v) for l, v in _TABLE1_B[k].items()}


def correction_a(k: int, n: int) -> Fr:
    """a_n^{(k)}, zero for n >= k."""
    a = _TABLE1_A[k]
    return a[n - 1] if 1 <= n <= len(a) else Fr(0)


def correction_b(k: int, l: int, n: int) -> Fr:
    b = _TABLE1_B[k].get(l)
    return b[n - 1] if (b is not None and 1 <= n <= len(b)) else Fr(0)


def cq_weights(k: int, alpha: float, n_terms: int, dps: int = 40) -> np.ndarray:
    """omega_j^{(alpha)}, j=0..n_terms-1: coefficients of delta_k(xi)^alpha (PAPER.md:893-897,
    eqn:delta), "computed ... by recursion": for P(xi) = sum_i p_i xi^i,
    q_0 = p_0^alpha,  q_n = 1/(n p_0) sum_{i=1}^{min(n,k)} ((alpha+1) i - n) p_i q_{n-i}
    (J.C.P. Miller's power-series recurrence), carried out in mpmath then rounded.
    alpha = 1 reproduces bdf_weights(k) padded with zeros.
    """
    mpmath.mp.dps = dps
    p = [mpmath.mpf(w.numerator) / w.denominator for w in bdf_weights(k)]
    a = mpmath.mpf(alpha)
    q = [p[0] ** a]
    for n in range(1, n_terms):
        s = mpmath.mpf(0)
        for i in range(1, min(n, k) + 1):
            s += ((a + 1) * i - n) * p[i] * q[n - i]
        q.append(s / (n * p[0]))
    return np.array([float(x) for x in q], dtype=np.float64)


def time_weights(k: int, alpha: float, N: int) -> np.ndarray:
    """The weights the all-at-once matrix uses: heat (alpha=1) -> omega_0..omega_k, zero beyond;
    CQ -> omega_0^{(alpha)}..omega_N^{(alpha)}.  Length N+1 (fp64)."""
    if alpha == 1.0:
        w = np.zeros(N + 1)
        bw = bdf_weights(k)
        w[:k + 1] = [float(x) for x in bw[:N + 1]]
        return w
    return cq_weights(k, alpha, N + 1)


def first_column(k: int, alpha: float, N: int, kappa: float) -> np.ndarray:
    """First column of the circulant B~_k(kappa) (Lemma 2.3; Lemma 3.2):
    c_j = kappa^{j/N} omega_j, j=0..N-1 (heat: zero for j>k).  numpy longdouble."""
    w = time_weights(k, alpha, N)[:N].astype(np.longdouble)
    j = np.arange(N, dtype=np.longdouble)
    return w * np.power(np.longdouble(kappa), j / np.longdouble(N))


def eigenvalues(k: int, alpha: float, N: int, kappa: float) -> np.ndarray:
    """d_p, p=0..N-1, the diagonal of D_k(kappa) in B_k(kappa) = S D S^{-1}, S = Lambda V
    (PAPER.md:454-464 eqn:Fourier-matrix; PAPER.md:583 gives d = delta_k(kappa^{1/N} e^{-i2pi(n-1)/N})).
    Computed as the plain DFT of the first column, d_p = sum_j c_j e^{-2 pi i (j p mod N)/N},
    in 80-bit long double with exact integer angle reduction, then rounded to complex128.
    For CQ this is the truncated scaled column (READING R-CQeig)."""
    c = first_column(k, alpha, N, kappa)
    j = np.arange(N)
    nz = np.nonzero(c)[0] if alpha == 1.0 else j
    p = np.arange(N)
    # np.pi is float64; build 2*pi in long double for accuracy
    two_pi = np.longdouble(4) * np.arctan(np.longdouble(1)) * 2
    ang = (np.outer(p, nz) % N).astype(np.longdouble) * (two_pi / N)
    re = (np.cos(ang) * c[nz][None, :]).sum(axis=1)
    im = (-np.sin(ang) * c[nz][None, :]).sum(axis=1)
    return (re.astype(np.float64) + 1j * im.astype(np.float64)).astype(np.complex128)


def gamma_scale(N: int, kappa: float) -> np.ndarray:
    """Gamma_kappa = Lambda(kappa)^{-1} = diag(kappa^{(n-1)/N}), n=1..N."""
    n = np.arange(N, dtype=np.longdouble)
    return np.power(np.longdouble(kappa), n / np.longdouble(N)).astype(np.float64)
