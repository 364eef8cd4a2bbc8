"""Pins for oracle/bdf.py: BDF weights, Table 1, CQ weights, eigenvalues d_p.

Each pin is something other than the oracle's own formula: order conditions, closed forms,
independent derivations (Bernoulli-number moment conditions), an independent method
(contour FFT), or a dense eigen-decomposition.
"""
from fractions import Fraction as Fr
from math import comb, factorial

import numpy as np
import pytest

from oracle import bdf, dense


# --- BDF weights -------------------------------------------------------

@pytest.mark.parametrize("k", range(1, 7))
def test_bdf_order_conditions(k):
    """delta_k(e^{-z}) = z + O(z^{k+1}): sum_j omega_j (-j)^m / m! = [m == 1], m = 0..k.
    (BDFk is consistent of order k; this fixes all k+1 weights uniquely.)"""
    w = bdf.bdf_weights(k)
    for m in range(0, k + 1):
        s = sum(wj * Fr((-j) ** m, factorial(m)) for j, wj in enumerate(w))
        assert s == (1 if m == 1 else 0)


@pytest.mark.parametrize("k", range(1, 7))
def test_bdf_special_values(k):
    w = bdf.bdf_weights(k)
    assert sum(w) == 0                                     # delta_k(1) = 0
    assert w[0] == sum(Fr(1, l) for l in range(1, k + 1))   # omega_0 = sum 1/l
    # delta_k(-1) = sum 2^l / l : 2, 4, 20/3, 32/3, 256/15, 416/15
    expect = {1: Fr(2), 2: Fr(4), 3: Fr(20, 3), 4: Fr(32, 3), 5: Fr(256, 15), 6: Fr(416, 15)}
    assert sum(wj * (-1) ** j for j, wj in enumerate(w)) == expect[k]


def test_bdf_textbook_k2_k3():
    assert bdf.bdf_weights(2) == [Fr(3, 2), Fr(-2), Fr(1, 2)]
    assert bdf.bdf_weights(3) == [Fr(11, 6), Fr(-3), Fr(3, 2), Fr(-1, 3)]


# --- Table 1 -----------------------------------------------------------

def _bernoulli(n):
    B = [Fr(1)]
    for m in range(1, n + 1):
        B.append(-sum(comb(m + 1, j) * B[j] for j in range(m)) / (m + 1))
    return B   # B_1 = -1/2 convention


def _moment_rhs(l, mu, B):
    """(-1)^mu mu! [s^mu] (1/s^{l+1} - sum_{n>=1} n^l e^{-ns} / l!)
    = (-1)^mu mu! * ( -B_{mu+l+1}/(mu+l+1)! (-1)^l C(mu+l, l) )."""
    m = mu + l + 1
    coef = -B[m] / factorial(m) * (-1) ** l * comb(mu + l, l)
    return (-1) ** mu * factorial(mu) * coef


def _solve_exact(A, b):
    n = len(b)
    M = [row[:] + [bb] for row, bb in zip(A, b)]
    for c in range(n):
        p = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[c])]
    return [M[i][n] / M[i][i] for i in range(n)]


def derived_table1(k):
    """Starting corrections from the exactness (moment) conditions, l = 0 -> a, l >= 1 -> b_l."""
    B = _bernoulli(20)
    out = {}
    for l in range(0, k - 1):
        nunk = k - 1 - l
        A = [[Fr(j) ** mu for j in range(1, nunk + 1)] for mu in range(nunk)]
        rhs = [_moment_rhs(l, mu, B) for mu in range(nunk)]
        sol = _solve_exact(A, rhs) if nunk else []
        out[l] = sol + [Fr(0)] * (k - 1 - nunk)
    return out


@pytest.mark.parametrize("k", range(2, 7))
def test_table1_matches_moment_conditions(k):
    a, b = bdf.table1(k)
    d = derived_table1(k)
    assert a == d[0]
    for l in range(1, k - 1):
        assert b[l] == d[l], (k, l)


def test_table1_printed_sign_outlier_documented():
    """The one printed entry that violates the conditions is b^{(5)}_{3,1}:
    printed +1/720, derived -1/720 (READING R-Table1)."""
    assert derived_table1(5)[3][0] == -bdf.TABLE1_B5_31_AS_PRINTED
    assert bdf.table1(5)[1][3][0] == Fr(-1, 720)


def test_table1_spot_values_from_paper():
    """Direct transcription spot checks of PAPER.md:320-338."""
    assert bdf.table1(2)[0] == [Fr(1, 2)]
    assert bdf.table1(4)[0] == [Fr(31, 24), Fr(-7, 6), Fr(3, 8)]
    assert bdf.table1(6)[0][4] == Fr(95, 288)
    assert bdf.table1(6)[1][4] == [Fr(0)] * 5


# --- CQ weights (Lemma 3.1) ---------------------------------------------

@pytest.mark.parametrize("k", range(1, 7))
def test_cq_alpha_one_is_bdf(k):
    w = bdf.cq_weights(k, 1.0, 12)
    ref = [float(x) for x in bdf.bdf_weights(k)] + [0.0] * (12 - k - 1)
    assert np.allclose(w, ref, atol=1e-15)


@pytest.mark.parametrize("alpha", [0.25, 0.5, 0.75])
def test_cq_k1_closed_form(alpha):
    """k = 1: omega_n = prod_{j<=n} (1 - (1+alpha)/j)  (binomial series of (1-xi)^alpha;
    the leading minus printed at PAPER.md:906 is a garble)."""
    w = bdf.cq_weights(1, alpha, 40)
    ref = [1.0]
    for j in range(1, 40):
        ref.append(ref[-1] * (1 - (1 + alpha) / j))
    assert np.allclose(w, ref, rtol=1e-14, atol=1e-17)


def _binom_series(alpha, c, n):
    """(1 - c xi)^alpha = sum_j C(alpha, j) (-c)^j xi^j."""
    out = [1.0]
    for j in range(1, n):
        out.append(out[-1] * (alpha - j + 1) / j * (-c))
    return np.array(out)


@pytest.mark.parametrize("alpha", [0.3, 0.5, 0.9])
def test_cq_k2_binomial_product(alpha):
    """delta_2(xi) = (3/2)(1-xi)(1-xi/3)  =>  delta_2^alpha = (3/2)^alpha (1-xi)^alpha (1-xi/3)^alpha."""
    n = 200
    ref = 1.5 ** alpha * np.convolve(_binom_series(alpha, 1.0, n), _binom_series(alpha, 1 / 3, n))[:n]
    assert np.allclose(bdf.cq_weights(2, alpha, n), ref, rtol=1e-12, atol=1e-16)


@pytest.mark.parametrize("k", [3, 4, 6])
def test_cq_contour_fft(k):
    """Independent method the paper names ("fast Fourier transform"): coefficients
    from samples of delta_k(xi)^alpha on |xi| = rho (aliasing error ~ rho^L)."""
    alpha, L, rho, n = 0.5, 4096, 0.9, 60
    xi = rho * np.exp(2j * np.pi * np.arange(L) / L)
    vals = bdf.delta_eval(k, xi) ** alpha
    c = np.fft.fft(vals) / L
    ref = (c[:n] / rho ** np.arange(n)).real
    assert np.allclose(bdf.cq_weights(k, alpha, n), ref, atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 4, 6])
def test_cq_weights_sum_and_decay(k):
    """sum_j omega_j^{(alpha)} -> delta_k(1)^alpha = 0; |omega_n| <= c (n+1)^{-1-alpha} (Lemma 3.1)."""
    alpha = 0.5
    w = bdf.cq_weights(k, alpha, 4001)
    tail = np.abs(w[1000:]) * (np.arange(1000, 4001) + 1.0) ** (1 + alpha)
    assert tail.max() < 2 * tail.min() + 1e-300
    assert abs(w.sum()) < 5 * abs(w[-1]) * 4001 ** (1 + alpha) * 4001 ** (-alpha)


# --- eigenvalues d_p (Lemma 2.3 / 3.2) ----------------------------------------------------

@pytest.mark.parametrize("k,alpha,N,kappa", [(1, 1.0, 8, 0.3), (3, 1.0, 16, 0.1), (6, 1.0, 32, 0.01),
                                              (2, 0.5, 16, 0.05), (4, 0.7, 24, 0.2)])
def test_eigenvalues_dense(k, alpha, N, kappa):
    """d_p are the eigenvalues of B_k(kappa) as drawn in the paper, and S D S^{-1} = B_k(kappa)
    with S = Lambda V."""
    B = dense.bk_kappa(k, alpha, N, kappa)
    d = bdf.eigenvalues(k, alpha, N, kappa)
    ev = np.linalg.eigvals(B)
    for x in d:
        assert np.min(np.abs(ev - x)) < 1e-10 * max(1.0, abs(x))
    n = np.arange(N)
    Lam = np.diag(kappa ** (-n / N))
    V = np.exp(2j * np.pi * np.outer(n, n) / N)
    S = Lam @ V
    Brec = S @ np.diag(d) @ np.linalg.inv(S)
    assert np.linalg.norm(Brec - B) / np.linalg.norm(B) < 1e-12


@pytest.mark.parametrize("k", range(1, 7))
def test_heat_eigenvalues_are_delta_at_scaled_roots(k):
    """d = delta_k(kappa^{1/N} e^{-i 2 pi (n-1)/N})."""
    N, kappa = 64, 0.05
    z = kappa ** (1 / N) * np.exp(-2j * np.pi * np.arange(N) / N)
    assert np.allclose(bdf.eigenvalues(k, 1.0, N, kappa), bdf.delta_eval(k, z), rtol=1e-13, atol=1e-15)
