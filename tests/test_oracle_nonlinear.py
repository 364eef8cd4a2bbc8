"""Pins of the nonlinear oracle (oracle/nonlinear.py, O5): Algorithm 3 and the modified scheme
eqn:BDF-CQ-m-r for the Allen-Cahn nonlinearity (Example 4)."""
import os

import numpy as np
import pytest

from oracle import nonlinear as nl
from oracle import sequential
from paper_2007_13125_b200 import inputs

HERE = os.path.dirname(os.path.abspath(__file__))
G, DG = nl.allen_cahn(1.0)


def test_g_zero_reduces_to_the_linear_scheme():
    """g = 0: the Newton-per-step sequential solver is the linear corrected CQ-BDFk stepping (O1)."""
    z = lambda u: 0 * u          # noqa: E731
    for a, k in [(0.75, 2), (1.0, 3), (0.25, 1)]:
        prob = inputs.example4_allen_cahn(a, k, M=99, N=64)
        U1, U2 = nl.sequential_nl(prob, z, z), sequential.sequential(prob)
        assert np.abs(U1 - U2).max() <= 1e-13 * np.abs(U2).max()


@pytest.mark.parametrize("alpha,k", [(1.0, 1), (0.75, 1), (0.75, 2), (0.25, 1), (0.25, 2)])
def test_temporal_order_on_the_discrete_manufactured_solution(alpha, k):
    """With the FD eigenvalue in the forcing, u = t^2/2 sin(2 pi x) solves the semi-discrete
    problem, so the error is the time discretisation's: observed order k (PAPER.md:1669-1673:
    tau^min(k, 1+2a-eps) for the modified scheme; k <= 2 here)."""
    es = []
    for N in (50, 100, 200):
        prob = inputs.example4_allen_cahn(alpha, k, M=99, N=N, discrete=True)
        es.append(nl.l2_error(prob, nl.sequential_nl(prob, G, DG)[-1], inputs.allen_cahn_exact(prob, N)))
    orders = np.log2(np.array(es[:-1]) / np.array(es[1:]))
    assert np.all(orders > k - 0.1), orders


@pytest.mark.parametrize("k", [2, 3])
def test_bdf_exact_for_quadratic_in_time(k):
    """alpha = 1: BDFk (k >= 2, with the Table-1 corrections) integrates the quadratic-in-time exact
    solution exactly, so only roundoff remains."""
    prob = inputs.example4_allen_cahn(1.0, k, M=99, N=100, discrete=True)
    e = nl.l2_error(prob, nl.sequential_nl(prob, G, DG)[-1], inputs.allen_cahn_exact(prob, prob.N))
    assert e < 1e-11, e


def test_residual_vanishes_at_the_sequential_solution():
    prob = inputs.example4_allen_cahn(0.75, 2, M=199, N=64)
    U = nl.sequential_nl(prob, G, DG)
    R = nl.residual(prob, U, G, nl.fbar_nl(prob, G))
    assert np.abs(R).max() < 1e-9 * np.abs(nl.fbar_nl(prob, G)).max() + 1e-9


def _table4():
    rows = {}
    for line in open(os.path.join(HERE, "golden", "table4_example4.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a, k, l, e, c = line.split()
        rows[(float(a), int(k), int(l))] = (float(e), None if c == "-" else int(c))
    return rows


@pytest.mark.parametrize("alpha,k", [(0.25, 1), (0.25, 2), (0.75, 1), (0.75, 2), (0.75, 3)])
def test_table4_example4(alpha, k):
    """FD analog of Table 4: the inner WR counts (5, 4, 3) are reproduced exactly in every column,
    Newton converges to the sequential solution (e_3 ~ 1e-12), and e_1..e_3 agree with the print
    within a factor 2.5.  e_0 = ||U^N||: the print (6.30e-2 / 5.94e-2) is not ||u(T)|| = 5.66e-2 of
    the stated exact solution (READING R-Table4)."""
    ref = _table4()
    prob = inputs.example4_allen_cahn(alpha, k)
    Useq = nl.sequential_nl(prob, G, DG)
    Us, counts = nl.newton_wr(prob, G, DG, 3)
    assert counts == [ref[(alpha, k, l)][1] for l in (1, 2, 3)]
    e = [nl.l2_error(prob, U[-1], Useq[-1]) for U in Us]
    assert abs(e[0] - np.sqrt(0.5) * 0.4 ** 2 / 2) < 5e-4          # ||u(T)||_L2 = T^2/2 / sqrt(2)
    for l in (1, 2, 3):
        assert ref[(alpha, k, l)][0] / 2.5 < e[l] < ref[(alpha, k, l)][0] * 2.5, (l, e[l])
    assert e[3] < 1e-12
