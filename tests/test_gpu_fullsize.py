"""Full-size parity (SURVEY §8(c) parity plan, VERDICT r1 "next" item 1) and the full-array update
monitor (PINT_FLAG_FULL_UPDATE_NORM; the paper's stopping rule).

* C4 at full size (1023^2 x 2048, BDF6): EVERY level of U_m, m = 1..3, streamed to the host in
  chunks and compared with the per-mode oracle O4 (exact: the data lie in the 32 x 32 sine span).
* C4 grid with a time-constant forcing in the same span: U^N does not decay, so the k window levels
  the fused kernel computes directly are checked per level.
* C5 at full size (511^2 x 1024, CQ-BDF2): the full array against O2 (library-FFT variant).
* CQ plans monitor every level: per-iteration updates and wr_solve stop counts equal the oracle's
  full-array max-norm ones (1D: physical; 2D: in the hoisted DST-x basis, reading R-norm2D).
"""
import numpy as np
import pytest

from oracle import modal, spatial, wr
from paper_2007_13125_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def pint():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_13125_b200 import pint as P
    P.lib()
    return P


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---------------------------------------------------------------------------------------------
# full-array update monitor
# ---------------------------------------------------------------------------------------------
def monitor_basis(prob, U):
    """The array the plan's full monitor sees: physical in 1D, DST-x coefficients (orthonormal
    DST-I along x, the hoisted basis) x physical y in 2D (reading R-norm2D)."""
    if prob.my == 1:
        return U
    return spatial.dst1(U.reshape(U.shape[0], prob.my, prob.mx), axis=2).reshape(U.shape[0], -1)


def oracle_updates(prob, iters):
    o = wr.wr_naive(prob, iters, dft="fft", wrap="fft")
    return [float(np.abs(monitor_basis(prob, o[m]) - monitor_basis(prob, o[m - 1])).max())
            for m in range(1, iters + 1)]


def stop_count(upd, tol):
    return next(m + 1 for m, u in enumerate(upd) if u < tol)


FULL_CASES = [
    ("c5_31", lambda: inputs.config_c5(m=31), {}),
    ("c5_63", lambda: inputs.config_c5(m=63), {}),
    ("c5_1d_511", lambda: inputs.config_c5(m=511).with_(name="C5_1d", my=1, v=inputs.indicator_square(511)[
        255 * 511: 256 * 511].copy()), {}),
    ("cq_rand_1d", lambda: inputs.random_complex_problem(255, 1, 1024, 2, 0.05, 0.5, R=1, seed=5), {}),
    ("heat_c1_flag", lambda: inputs.config_c1(), {"full_update_norm": True}),
    ("heat_2d_flag", lambda: inputs.random_complex_problem(63, 31, 256, 4, 0.05, 1.0, R=1, seed=9),
     {"full_update_norm": True}),
]


@pytest.mark.parametrize("name,make,kw", FULL_CASES, ids=[c[0] for c in FULL_CASES])
def test_full_update_norm_matches_oracle(pint, name, make, kw):
    prob = make()
    iters = 7
    ou = oracle_updates(prob, iters)
    with pint.Plan.from_problem(prob, **kw) as p:
        assert not p.path()["fused"]
        gu = [p.iterate() for _ in range(iters)]
    print(f"{name}: oracle full-array updates " + " ".join(f"{u:.2e}" for u in ou))
    print(f"{name}: GPU    full-array updates " + " ".join(f"{u:.2e}" for u in gu))
    scale = ou[0]
    for g, o in zip(gu, ou):          # the same number down to the round-off floor
        assert abs(g - o) <= 1e-6 * o + 1e-12 * scale, (g, o)
    for tol in (1e-10, 1e-12):
        # a stop count is only well defined when no update straddles the tolerance
        if min(abs(np.log10(u / tol)) for u in ou) < 0.3:
            print(f"{name}: tol {tol:g} straddled by an update, stop count not compared")
            continue
        want = stop_count(ou, tol)
        with pint.Plan.from_problem(prob, **kw) as p:
            it, u, st = p.solve(tol, 20)
        assert st == pint.PINT_OK and it == want, (tol, it, want, ou)


def test_full_monitor_levels_match_materialised(pint):
    """With the full monitor, pint_get_levels reads U_m from the monitor's copy (no Step-3 pass);
    it must equal the oracle iterate like the materialised path (CQ, 2D, m = 1..3)."""
    prob = inputs.random_complex_problem(31, 20, 256, 2, 0.1, 0.6, R=1, seed=21)
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    with pint.Plan.from_problem(prob) as p:
        for m in range(1, 4):
            p.iterate()
            assert rel(p.get_solution(), o[m]) < 1e-12
            assert rel(p.get_levels(100, 7), o[m][100:107]) < 1e-12
        r, f = p.residual()
        assert np.isfinite(r) and f > 0


# ---------------------------------------------------------------------------------------------
# C4 at full size, every level
# ---------------------------------------------------------------------------------------------
def _c4_stream_compare(plan, basis, coef_levels, N, chunk=64):
    """Stream all N levels of the plan's current iterate and compare with the modal oracle's
    coefficient levels [N][32*32] (layout [q][p]).  Returns (full rel L2, per-level rel errors,
    per-level oracle norms)."""
    Sx, Sy = basis.synth_x(), basis.synth_y()
    nq, npx = len(basis.py), len(basis.px)
    e2 = r2 = 0.0
    per, norms = np.zeros(N), np.zeros(N)
    for n0 in range(0, N, chunk):
        c = min(chunk, N - n0)
        g = plan.get_levels(n0, c).reshape(c, basis.my, basis.mx)
        Cn = coef_levels[n0:n0 + c].reshape(c, nq, npx)
        o = np.matmul(Sy, np.matmul(Cn, Sx.T))           # [c][y][x]
        d2 = np.sum(np.abs(g - o) ** 2, axis=(1, 2))
        o2 = np.sum(np.abs(o) ** 2, axis=(1, 2))
        e2 += d2.sum()
        r2 += o2.sum()
        per[n0:n0 + c] = np.sqrt(d2 / o2)
        norms[n0:n0 + c] = np.sqrt(o2)
    return float(np.sqrt(e2 / r2)), per, norms


@pytest.mark.slow
def test_c4_full_array_every_level(pint):
    """C4 (the bench configuration): all 2048 levels x 1023^2 points of U_m, m = 1..3, against O4.
    Gate: full-array relative L2 <= 1e-10 (north_star)."""
    prob = inputs.config_c4()
    basis = modal.ModalBasis(1023, 1023, np.arange(1, 33), np.arange(1, 33))
    C = inputs.c4_mode_coefficients()
    coef = C.T.reshape(-1)
    md = modal.modal_wr(prob, basis, coef, np.zeros((0, coef.size)), 3)
    with pint.Plan.from_problem(prob) as p:
        assert p.path()["fused"]
        for m in range(1, 4):
            p.iterate()
            err, per, norms = _c4_stream_compare(p, basis, md[m], prob.N)
            worst = int(np.argmax(per))
            print(f"C4 m={m}: full-array rel L2 = {err:.3e}; per-level rel error: level 1 {per[0]:.2e}, "
                  f"1024 {per[1023]:.2e}, N {per[-1]:.2e} (|U^N| / |U^1| = {norms[-1] / norms[0]:.1e}); "
                  f"worst level {worst + 1}: {per[worst]:.2e}")
            assert err <= TOL, (m, err)


@pytest.mark.slow
def test_c4_window_levels_nondecaying(pint):
    """C4 grid, N, k, kappa with a time-constant forcing g in the 32 x 32 sine span (phi = 1): the
    solution tends to A^{-1} g instead of decaying, so the window levels n = N-k+1..N that the fused
    kernel produces directly are O(1).  Per-level relative error <= 1e-10 on the window for m = 1..3, and the
    full array <= 1e-10 at m = 3 (O4 stays exact: v and g in the span)."""
    base = inputs.config_c4()
    basis = modal.ModalBasis(1023, 1023, np.arange(1, 33), np.arange(1, 33))
    C = inputs.c4_mode_coefficients()
    Cg = 50.0 * np.random.default_rng(2007131259).standard_normal((32, 32))
    g = basis.to_grid(Cg.T.reshape(-1)).astype(np.complex128)[None, :]
    prob = base.with_(name="C4_forced", g=g, phi=np.ones((1, base.N + 1)), dphi=np.zeros((1, base.k - 2)))
    md = modal.modal_wr(prob, basis, C.T.reshape(-1), Cg.T.reshape(1, -1), 3)
    with pint.Plan.from_problem(prob) as p:
        assert p.path()["fused"]
        for m in range(1, 4):
            p.iterate()
            # the window read path first (wrap state, before any materialisation)
            w = p.get_levels(prob.N - prob.k, prob.k).reshape(prob.k, -1)
            ref = basis.to_grid(md[m][-prob.k:]).reshape(prob.k, -1)
            assert rel(w, ref) <= TOL
            win = np.array([rel(w[j], ref[j]) for j in range(prob.k)])
            print(f"C4 forced m={m}: window levels rel = " + " ".join(f"{e:.2e}" for e in win))
            assert win.max() <= TOL, (m, win)
            if m < 3:
                continue
            # every level of the last iterate (the decaying recipe's test above streams all three; here the
            # per-iterate coverage is the window, which determines the next iterate: PAPER.md:388)
            err, per, norms = _c4_stream_compare(p, basis, md[m], prob.N)
            print(f"C4 forced m={m}: full-array rel L2 = {err:.3e}; window levels (materialised) rel = "
                  + " ".join(f"{e:.2e}" for e in per[-prob.k:]) + f" (|U^N| / |U^1| = {norms[-1] / norms[0]:.2f})")
            assert norms[-1] > 0.1 * norms[0]
            assert err <= TOL and per[-prob.k:].max() <= TOL, (m, err, per[-prob.k:])


@pytest.mark.slow
def test_c5_full_array(pint):
    """C5 at full size (511^2 x 1024, CQ-BDF2, alpha = 0.5; the bench configuration): the full
    space-time array of U_m, m = 1..3, against O2 (library FFT for the DFTs and the 2N circulant
    embedding of the CQ wrap, pinned equal to the naive forms in the oracle tests)."""
    prob = inputs.config_c5()
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    with pint.Plan.from_problem(prob) as p:
        for m in range(1, 4):
            p.iterate()
            g = p.get_solution()
            err = rel(g, o[m])
            last = rel(g[-1], o[m][-1])
            print(f"C5 m={m}: full-array rel L2 = {err:.3e}, final level {last:.3e}")
            assert err <= TOL, (m, err)
