"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element on the same
seeded inputs, at fixed iteration counts m (SURVEY §8(c) "Parity metric").

Gate (BASELINE.json north_star): full space-time array relative L2 <= 1e-10 (fp64 complex).
"""
import numpy as np
import pytest

from oracle import modal, sequential, wr
from paper_2007_13125_b200 import inputs

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def pint():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_13125_b200 import pint as P
    P.lib()
    return P


def gpu_iterates(P, prob, iters, **kw):
    out, upd = [], []
    with P.Plan.from_problem(prob, **kw) as plan:
        for _ in range(iters):
            upd.append(plan.iterate())
            out.append(plan.get_solution())
    return out, upd


def check(P, prob, iters, tol=TOL, oracle_kw=None):
    g, _ = gpu_iterates(P, prob, iters)
    o = wr.wr_naive(prob, iters, **(oracle_kw or {}))
    errs = [rel(g[m], o[m + 1]) for m in range(iters)]
    print(f"{prob.name}: rel L2 per m = " + " ".join(f"{e:.2e}" for e in errs))
    assert max(errs) <= tol, errs
    return errs


def test_c1_parity_and_fixed_point(pint):
    prob = inputs.config_c1()
    errs = check(pint, prob, 5)
    assert max(errs) < 1e-12, errs
    with pint.Plan.from_problem(prob) as p:
        it, u, st = p.solve(1e-12, 20)
        assert st == 0 and it <= 6 and u < 1e-12
        assert rel(p.get_solution(), sequential.sequential(prob)) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("kappa", [1e-1, 1e-2, 1e-3])
def test_c2_sweep(pint, k, kappa):
    """C2: 1D M=1023, N=1024, every k and kappa (18 runs), m = 1..4 (SURVEY §8(c) parity plan)."""
    check(pint, inputs.config_c2(k=k, kappa=kappa), 4)


CASES = [
    # mx, my, N, k, kappa, alpha, R   (ragged line lengths, every FFT length, heat + CQ, 1D + 2D)
    (37, 1, 16, 1, 0.3, 1.0, 2),
    (1, 1, 32, 2, 0.2, 1.0, 1),          # M = 1: scalar ODE (degenerate)
    (100, 1, 32, 3, 0.1, 1.0, 2),
    (200, 1, 128, 6, 0.05, 1.0, 1),
    (1000, 1, 64, 2, 0.1, 0.5, 1),
    (333, 1, 512, 4, 0.02, 0.3, 2),
    (127, 1, 2048, 6, 0.01, 1.0, 0),
    (63, 1, 4096, 2, 0.1, 1.0, 1),
    (15, 9, 64, 4, 0.2, 1.0, 2),
    (31, 40, 256, 5, 0.05, 1.0, 1),
    (63, 33, 128, 2, 0.05, 0.5, 1),
    (7, 100, 512, 3, 0.1, 0.7, 1),
    (255, 17, 1024, 1, 0.1, 0.5, 0),
    (127, 1024, 16, 2, 0.3, 1.0, 1),     # longest line, shortest N
    # one-kernel CQ T-pass (N = 256: 16 x 16, N = 1024: 32 x 32) with S = R + 1 = 4 sources: two
    # staged in shared memory, the others added to the TMEM stash; ragged tile tails
    (63, 5, 256, 2, 0.05, 0.4, 3),
    (31, 3, 1024, 3, 0.1, 0.6, 3),
]


@pytest.mark.parametrize("mx,my,N,k,kappa,alpha,R", CASES)
def test_random_complex(pint, mx, my, N, k, kappa, alpha, R):
    prob = inputs.random_complex_problem(mx, my, N, k, kappa, alpha, R=R, seed=mx + my + N + k)
    check(pint, prob, 3, oracle_kw={"dft": "fft", "wrap": "fft"} if N * mx * my > 2e6 else None)


def test_c3_parity(pint):
    """C3: 2D 511^2, N = 256, BDF4, kappa = 0.05 (full size, full array), m = 1..2."""
    check(pint, inputs.config_c3(), 2)


def test_c5_reduced_parity(pint):
    """C5 recipe at 127^2 (N = 1024, CQ-BDF2, alpha = 0.5): full array, m = 1..3."""
    check(pint, inputs.config_c5(m=127), 3, oracle_kw={"dft": "fft", "wrap": "fft"})


def test_c4_modal_sampled(pint):
    """C4 at full size (1023^2 x 2048, 34 GB per buffer): sampled levels vs the per-mode oracle O4.
    Metric: the full-array relative L2 restricted to the sampled levels, i.e. each level's error
    over the RMS level norm of the whole oracle array (computed exactly in modal space, where
    sum_i sin^2(p pi x_i) = (m+1)/2).  A per-level relative error is ill-posed here: by t = 1 the
    solution has decayed by ~1e-9."""
    prob = inputs.config_c4()
    basis = modal.ModalBasis(1023, 1023, np.arange(1, 33), np.arange(1, 33))
    C = inputs.c4_mode_coefficients()          # C[p-1, q-1] multiplies sin(p pi x) sin(q pi y)
    coef = C.T.reshape(-1)                     # basis layout [q][p]
    iters = 3
    md = modal.modal_wr(prob, basis, coef, np.zeros((0, coef.size)), iters)
    levels = [0, 1, 5, 200, 1023, 2046, 2047]
    with pint.Plan.from_problem(prob) as p:
        for m in range(1, iters + 1):
            p.iterate()
            rms = np.sqrt(np.sum(np.abs(md[m]) ** 2) * (1024 / 2) ** 2 / prob.N)
            worst = 0.0
            for n in levels:
                g = p.get_levels(n, 1)[0]
                o = basis.to_grid(md[m][n])
                worst = max(worst, np.linalg.norm(g - o) / rms)
            print(f"C4 m={m}: max sampled-level error / RMS level norm = {worst:.3e}")
            assert worst < TOL, (m, worst)


def test_c5_full_size_modal_sampled(pint):
    """C5 at full size (511^2 x 1024, CQ-BDF2, alpha = 0.5, the bench configuration): the GPU
    iterate projected on a sample of 7 x 7 sine modes (exact DST projections; the FD sine modes are
    exact eigenvectors, so each mode coefficient follows the scalar WR of the per-mode oracle O4)
    at sampled levels, m = 1..3.  Metric: relative L2 over the sampled (mode, level) set."""
    prob = inputs.config_c5()
    m = prob.mx
    modes = np.array([1, 2, 3, 7, 50, 255, 511])
    basis = modal.ModalBasis(m, m, modes, modes)
    Sx, Sy = basis.synth_x(), basis.synth_y()
    sc = (2.0 / (m + 1)) ** 2

    def project(u):                      # [M] grid -> [q][p] coefficients, layout of the basis
        return (sc * (Sy.T @ u.reshape(m, m) @ Sx)).reshape(-1)

    iters = 3
    md = modal.modal_wr(prob, basis, project(prob.v), np.zeros((0, modes.size ** 2)), iters)
    levels = [0, 1, 2, 100, 511, 1022, 1023]
    with pint.Plan.from_problem(prob) as p:
        for it in range(1, iters + 1):
            p.iterate()
            g = np.stack([project(p.get_levels(n, 1)[0]) for n in levels])
            o = md[it][levels]
            err = float(np.linalg.norm(g - o) / np.linalg.norm(o))
            print(f"C5 full size m={it}: sampled modal relative L2 = {err:.3e}")
            assert err < TOL, (it, err)


def test_u0_zero_and_initial_guess(pint):
    prob = inputs.example1_fd(3, M=99, N=64)            # U_0 = 0 (table setting)
    check(pint, prob, 3)
    check(pint, inputs.example2_fd(2, M=255, N=256), 3)  # CQ, U_0 = 0 (separable CQ bootstrap)
    prob = inputs.config_c1()
    Us = sequential.sequential(prob)
    with pint.Plan.from_problem(prob) as p:
        p.set_initial_guess(np.ascontiguousarray(Us))   # the fixed point
        u = p.iterate()
        assert u < 1e-12
        assert rel(p.get_solution(), Us) < 1e-12


def test_reading_does_not_perturb(pint):
    """Reading U_m (materialised into the H buffer) and continuing re-derives H_{m+1} from the
    time domain; the iterates agree with an unread run to roundoff."""
    prob = inputs.config_c2(k=3, kappa=0.01)
    a, ua = gpu_iterates(pint, prob, 3)
    with pint.Plan.from_problem(prob) as p:
        ub = [p.iterate() for _ in range(3)]
        b = p.get_solution()
    assert rel(a[-1], b) < 1e-13
    assert all(abs(x - y) <= 1e-12 * ua[0] for x, y in zip(ua, ub))


def test_device_arrays_and_levels(pint):
    import torch
    prob = inputs.random_complex_problem(31, 30, 64, 3, 0.1, 1.0, R=2, seed=4)
    with pint.Plan.from_problem(prob, device_arrays=True) as p:
        p.iterate(); p.iterate()
        full = p.get_solution()
        dev = torch.empty((10, prob.M), dtype=torch.complex128, device="cuda")
        p.get_levels(20, 10, out=dev)
        assert np.array_equal(dev.cpu().numpy(), full[20:30])
    o = wr.wr_naive(prob, 2)[2]
    assert rel(full, o) < TOL


def test_state_errors_and_timing(pint):
    P = pint
    with P.Plan(63, 1, 64, 2, 0.1, 1 / 64) as p:
        with pytest.raises(P.PintError) as e:
            p.iterate()
        assert e.value.status == P.PINT_ERR_STATE
        prob = inputs.config_c1()
        p.set_problem(prob.v, prob.g, prob.phi, prob.dphi)
        with pytest.raises(P.PintError) as e:
            p.get_solution()
        assert e.value.status == P.PINT_ERR_STATE
        p.set_timing(True)
        for _ in range(3):
            p.iterate()
        t = p.get_timing()
        assert t["tpass_launches"] == 3 and t["spass_launches"] == 3
        assert t["tpass_ms"] > 0 and t["spass_ms"] > 0
        it, u, st = p.solve(0.0, 2, raise_on_fail=False)
        assert st == P.PINT_ERR_NOT_CONVERGED and it == 2


@pytest.mark.parametrize("variant", ["fused", "modal", "cq_stream", "cq_modal"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_xmode_slabs_reproduce_single_plan(pint, nranks, variant):
    """The multi-GPU partition on one GPU: each x-mode slab plan iterates independently (the WR
    iteration has no inter-slab exchange), the gathered modal slabs map back to the single-plan
    physical solution (bitwise up to the DST ordering: checked to 1e-14)."""
    from paper_2007_13125_b200 import dist as pdist
    alpha = 0.5 if variant.startswith("cq") else 1.0
    kw = {"modal": True} if variant.endswith("modal") else {}
    prob = inputs.random_complex_problem(63, 31, 128, 4, 0.05, alpha, R=1, seed=12)
    with pint.Plan.from_problem(prob, **kw) as p:
        for _ in range(3):
            p.iterate()
        ref = p.get_solution()
    slabs, bounds, plans = [], [], []
    for r in range(nranks):
        pl = pint.Plan(prob.mx, prob.my, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha,
                       rank=r, nranks=nranks, allreduce_max=lambda x: x, **kw)
        pl.set_problem(prob.v, prob.g, prob.phi, prob.dphi)
        for _ in range(3):
            pl.iterate()
        slabs.append(pl.get_modal_levels(0, prob.N))
        bounds.append(pl.partition())
        plans.append(pl)
    full = pdist.assemble_modal(slabs, bounds, prob.mx)
    phys = plans[0].modal_to_physical(np.ascontiguousarray(full))
    for pl in plans:
        pl.close()
    assert rel(phys, ref) < 1e-14


@pytest.mark.parametrize("N,k,mx,my", [(512, 1, 100, 1), (1024, 3, 63, 20), (2048, 6, 127, 1),
                                       (4096, 2, 31, 9), (2048, 4, 15, 33)])
def test_pruned_tpass_matches_full_fft_and_oracle(pint, N, k, mx, my):
    """Heat with f = 0, reading every iterate: the fused iteration (default), the streaming one
    with the unpruned FFT T-pass (PINT_FLAG_STREAM | PINT_FLAG_FULL_FFT) and the oracle, m = 1..3."""
    prob = inputs.random_complex_problem(mx, my, N, k, 0.02, 1.0, R=0, seed=N + k)
    res = {}
    for name, kw in (("fused", {}), ("full", {"stream_path": True, "full_fft": True})):
        with pint.Plan.from_problem(prob, **kw) as p:
            res[name] = []
            for _ in range(3):
                p.iterate()
                res[name].append(p.get_solution())
    o = wr.wr_naive(prob, 3, dft="fft")
    for m in range(3):
        assert rel(res["fused"][m], res["full"][m]) < 1e-13
        assert rel(res["fused"][m], o[m + 1]) < TOL


UNREAD = [
    # mx, my, N, k, kappa, R: heat cases on the pruned T-pass (N >= 256), with and without
    # dense-in-time sources (R = 1: phi_r(t) dense; R = 0: only v and A v, sparse)
    (200, 1, 256, 2, 0.1, 0),
    (200, 1, 512, 3, 0.1, 0),
    (100, 1, 1024, 1, 0.1, 0),
    (100, 1, 2048, 6, 0.05, 1),
    (31, 40, 256, 4, 0.05, 1),
    (63, 20, 2048, 6, 0.01, 0),
    (33, 1, 4096, 5, 0.02, 0),
]


PATHS = {"fused": {}, "stream": {"stream_path": True}, "stream_full_fft": {"stream_path": True, "full_fft": True}}


@pytest.mark.parametrize("mx,my,N,k,kappa,R", UNREAD)
@pytest.mark.parametrize("path", list(PATHS))
def test_unread_iterations(pint, mx, my, N, k, kappa, R, path):
    """m iterations without reading in between (the production loop: the fused one-kernel
    iteration, the streaming two-pass one with the pruned T-pass, or with the unpruned FFTs), then
    one read: equals the oracle's m-th iterate, and the update norms equal the oracle's window
    updates.  The window levels read before the full array (no materialisation) agree too."""
    prob = inputs.random_complex_problem(mx, my, N, k, kappa, 1.0, R=R, seed=mx + N + k)
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    for m in (1, 3):
        with pint.Plan.from_problem(prob, **PATHS[path]) as p:
            ups = [p.iterate() for _ in range(m)]
            win = p.get_levels(N - k, k)
            err = rel(p.get_solution(), o[m])
            # window error over the full-array norm (the last levels have decayed by ~1e-12)
            assert np.linalg.norm(win - o[m][N - k:]) / np.linalg.norm(o[m]) <= TOL
        assert err <= TOL, (m, err)
        if my == 1:   # 2D monitors the window in the DST-x basis (a different max-norm)
            ref_upd = np.abs(o[m][N - k:] - o[m - 1][N - k:]).max()
            assert abs(ups[-1] - ref_upd) <= 1e-9 * ref_upd + 1e-13, (ups[-1], ref_upd)


def test_c2_unread_matches_read(pint):
    """C2 (k = 3, kappa = 0.01): the unread loop and the read-every-iteration loop agree."""
    prob = inputs.config_c2(k=3, kappa=0.01)
    with pint.Plan.from_problem(prob) as p:
        ub = [p.iterate() for _ in range(3)]
        b = p.get_solution()
    o = wr.wr_naive(prob, 3)
    assert rel(b, o[3]) < TOL
    assert ub[1] > 0.0


@pytest.mark.parametrize("nlev,fused", [(7, True), (12, False)])
def test_forcing_pulse_path_selection(pint, nlev, fused):
    """Forcing supported on the first `nlev` time levels: Gamma F has nk = nlev nonzero leading
    levels.  nk <= 8 runs the fused iteration with nk > k; nk in 9..16 falls back to the streaming
    iteration (pruned T-pass).  Both match the oracle, read every iterate and unread."""
    prob = inputs.random_complex_problem(90, 1, 512, 3, 0.05, 1.0, R=1, seed=nlev)
    phi = prob.phi.copy()
    phi[:, nlev + 1:] = 0.0                 # phi_r(t_n) = 0 for n > nlev (1-based level n)
    prob = prob.with_(phi=phi)
    o = wr.wr_naive(prob, 3, dft="fft")
    with pint.Plan.from_problem(prob) as p:
        assert p.path()["fused"] is fused and p.path()["nk"] == nlev
        errs = []
        for m in range(1, 4):
            p.iterate()
            errs.append(rel(p.get_solution(), o[m]))
    with pint.Plan.from_problem(prob) as p:
        for _ in range(3):
            p.iterate()
        errs.append(rel(p.get_solution(), o[3]))
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("mx,my,N,k,kappa,alpha,R", [
    (31, 40, 64, 3, 0.1, 1.0, 1),        # heat, dense-in-time forcing
    (63, 33, 128, 2, 0.05, 0.5, 1),      # CQ subdiffusion
    (127, 100, 256, 6, 0.01, 1.0, 0),    # heat, BDF6
])
def test_dst_per_iteration_ablation(pint, mx, my, N, k, kappa, alpha, R):
    """the DST-x applied before and after the shifted solves every iteration
    (PINT_FLAG_DST_PER_ITER, physical-x arrays) gives the iterate of the hoisted default, read
    after every m and unread, and both match the oracle."""
    prob = inputs.random_complex_problem(mx, my, N, k, kappa, alpha, R=R, seed=3 * mx + my)
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    hoisted, _ = gpu_iterates(pint, prob, 3)
    per_iter, _ = gpu_iterates(pint, prob, 3, dst_per_iter=True)
    for m in range(3):
        assert rel(per_iter[m], hoisted[m]) < 1e-12
        assert rel(per_iter[m], o[m + 1]) < TOL
    with pint.Plan.from_problem(prob, dst_per_iter=True) as p:
        assert not p.path()["fused"]
        for _ in range(3):
            p.iterate()
        win = p.get_levels(N - k, k)
        assert rel(p.get_solution(), o[3]) < TOL
        assert np.linalg.norm(win - o[3][N - k:]) / np.linalg.norm(o[3]) < TOL


@pytest.mark.parametrize("alpha,k", [(0.25, 1), (0.25, 2), (0.75, 2), (0.75, 3), (1.0, 2)])
def test_newton_wr_allen_cahn(pint, alpha, k):
    """Semilinear extension (Algorithm 3): Example 4 at N = 128 (the library's
    power-of-two N), h = 1/1000.  Each Newton step's iterate U_l matches the oracle's Algorithm 3 and
    the inner WR counts are the oracle's (5, 4, 3, as in Table 4)."""
    from oracle import nonlinear as nl
    G, DG = nl.allen_cahn(1.0)
    prob = inputs.example4_allen_cahn(alpha, k, N=128)
    Us, counts = nl.newton_wr(prob, G, DG, 3)
    with pint.Plan.from_problem(prob) as p:
        p.set_nonlinearity(1.0)
        assert np.array_equal(p.get_solution(), Us[0])      # U_0 = v (= 0 for Example 4)
        with pytest.raises(pint.PintError) as e:
            p.iterate()
        assert e.value.status == pint.PINT_ERR_STATE
        for l in range(1, 4):
            c, u, st = p.newton_solve(1)
            assert c == [counts[l - 1]], (l, c, counts)
            err = rel(p.get_solution(), Us[l])
            print(f"alpha={alpha} k={k} l={l}: inner {c[0]}, rel L2 vs oracle {err:.2e}, update {u[0]:.2e}")
            assert err < TOL, (l, err)
    if alpha < 1.0:
        assert counts == [5, 4, 3]      # Table 4's bracketed counts (alpha = 0.25, 0.75 columns)


def test_newton_wr_rejects_2d(pint):
    prob = inputs.random_complex_problem(15, 9, 64, 2, 0.1, 1.0, R=0, seed=1)
    with pint.Plan.from_problem(prob) as p:
        with pytest.raises(pint.PintError) as e:
            p.set_nonlinearity(1.0)
        assert e.value.status == pint.PINT_ERR_UNSUPPORTED


REAL_CASES = [
    ("C1", lambda: inputs.config_c1()),
    ("C2k6", lambda: inputs.config_c2(k=6, kappa=1e-3)),
    ("C3", lambda: inputs.config_c3()),
    ("2D-real", lambda: inputs.random_complex_problem(63, 40, 256, 4, 0.05, 1.0, R=1, seed=5).real_part()),
    ("1D-N16", lambda: inputs.random_complex_problem(37, 1, 16, 1, 0.3, 1.0, R=2, seed=8).real_part()),
    ("FEM-1D", lambda: inputs.random_complex_problem(127, 1, 256, 3, 0.05, 1.0, R=1, seed=9).real_part().with_(space="fem")),
]


@pytest.mark.parametrize("name,make", REAL_CASES, ids=[c[0] for c in REAL_CASES])
def test_real_data_half_spectrum(pint, name, make):
    """for real data W_{N-p} = conj(W_p), so the fused iteration solves only
    p <= N/2 (PINT_FLAG_REAL_DATA).  Same iterates as the full spectrum and the oracle, read after
    every m and unread."""
    prob = make()
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    half, _ = gpu_iterates(pint, prob, 3, real_data=True)
    full, _ = gpu_iterates(pint, prob, 3)
    for m in range(3):
        assert rel(half[m], full[m]) < 1e-12
        assert rel(half[m], o[m + 1]) < TOL
    with pint.Plan.from_problem(prob, real_data=True) as p:
        for _ in range(3):
            p.iterate()
        assert rel(p.get_solution(), o[3]) < TOL


def test_real_data_rejects_complex(pint):
    prob = inputs.random_complex_problem(31, 1, 64, 2, 0.1, 1.0, R=1, seed=2)
    with pytest.raises(pint.PintError) as e:
        pint.Plan.from_problem(prob, real_data=True)
    assert e.value.status == pint.PINT_ERR_ARG


MODAL_CASES = [
    ("C3", lambda: inputs.config_c3(), {}),
    ("2D-c", lambda: inputs.random_complex_problem(63, 31, 256, 4, 0.05, 1.0, R=1, seed=6), {}),
    ("2D-N2048", lambda: inputs.random_complex_problem(31, 63, 2048, 6, 0.01, 1.0, R=0, seed=7), {}),
    ("2D-real-half", lambda: inputs.random_complex_problem(63, 15, 128, 2, 0.1, 1.0, R=2, seed=9).real_part(),
     {"real_data": True}),
]


@pytest.mark.parametrize("name,make,kw", MODAL_CASES, ids=[c[0] for c in MODAL_CASES])
def test_fully_modal_variant(pint, name, make, kw):
    """SURVEY §8(f) item 2a (PINT_FLAG_MODAL): DST along y too, the shifted solves become divisions
    per (x-mode, y-mode).  Same iterates as the line-solve path and the oracle, read after every m
    and unread; window levels and a user initial guess go through the y-mode space correctly."""
    prob = make()
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    modal, _ = gpu_iterates(pint, prob, 3, modal=True, **kw)
    lines, _ = gpu_iterates(pint, prob, 3, **kw)
    for m in range(3):
        assert rel(modal[m], lines[m]) < 1e-12
        assert rel(modal[m], o[m + 1]) < TOL
    N, k = prob.N, prob.k
    with pint.Plan.from_problem(prob, modal=True, **kw) as p:
        for _ in range(3):
            p.iterate()
        win = p.get_levels(N - k, k)
        assert np.linalg.norm(win - o[3][N - k:]) / np.linalg.norm(o[3]) < TOL
        assert rel(p.get_solution(), o[3]) < TOL
        U0 = o[3].real.astype(np.complex128) if kw.get("real_data") else o[3]   # oracle roundoff in Im
        p.set_initial_guess(np.ascontiguousarray(U0))
        p.iterate()
        assert rel(p.get_solution(), wr.wr_naive(prob, 1, U0=U0, dft="fft", wrap="fft")[1]) < TOL


@pytest.mark.parametrize("mx,my,N,k,kappa,alpha", [
    (63, 1, 64, 2, 0.1, 1.0),
    (100, 1, 256, 6, 0.05, 1.0),     # heat, dense in time: streaming unpruned T-pass
    (15, 9, 32, 4, 0.2, 1.0),        # 2D: DST-x per level of f
    (63, 1, 128, 3, 0.1, 0.5),       # CQ
    (31, 15, 64, 2, 0.05, 0.3),      # 2D CQ
])
def test_dense_forcing(pint, mx, my, N, k, kappa, alpha):
    """pint_set_problem: a non-separable f(t_n, x) with its starting corrections
    a_n f(0) and b_{l,n} tau^l f^(l)(0); iterates match the oracle (which sees the same data as a
    separable record with one source per level), read after every m and unread."""
    prob, f, f0, fd = inputs.random_dense_forcing(mx, my, N, k, kappa, alpha, seed=mx + N)
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    with pint.Plan(prob.mx, prob.my, N, k, kappa, prob.tau, alpha) as p:
        p.set_problem_dense(prob.v, f, f0, fd if fd.size else None)
        assert not p.path()["fused"]
        for m in range(1, 4):
            p.iterate()
            assert rel(p.get_solution(), o[m]) < TOL, m
    with pint.Plan(prob.mx, prob.my, N, k, kappa, prob.tau, alpha) as p:
        p.set_problem_dense(prob.v, f, f0, fd if fd.size else None)
        for _ in range(3):
            p.iterate()
        assert rel(p.get_solution(), o[3]) < TOL


def test_dense_forcing_newton(pint):
    """Newton-WR with the Example-4 forcing passed densely equals the separable run."""
    from oracle import nonlinear as nl
    prob = inputs.example4_allen_cahn(0.75, 2, N=128)
    f = np.ascontiguousarray((prob.phi[:, 1:].T @ prob.g))
    f0 = np.ascontiguousarray(prob.phi[:, 0] @ prob.g)
    res = []
    for dense in (False, True):
        with pint.Plan(prob.mx, 1, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha) as p:
            if dense:
                p.set_problem_dense(prob.v, f, f0)
            else:
                p.set_problem(prob.v, prob.g, prob.phi, prob.dphi)
            p.set_nonlinearity(1.0)
            c, u, st = p.newton_solve(3)
            res.append((c, p.get_solution()))
    assert res[0][0] == res[1][0]
    assert rel(res[1][1], res[0][1]) < 1e-12


def test_wr_solve_divergence_guard(pint, monkeypatch):
    """S:406 / SURVEY §8(b): the WR iteration diverges when kappa R / (1 - kappa R) > 1 (BDF1
    contraction factor) — a scalar problem with a tiny T (R ~ 1) and kappa = 0.9 —
    and pint_wr_solve reports PINT_ERR_DIVERGED after 3 consecutive increases: on the device loop
    (default) after the same number of iterations as on the host loop (PINT_NO_GRAPH=1)."""
    prob = inputs.random_complex_problem(1, 1, 64, 1, 0.9, 1.0, R=0, seed=3, T=1e-3)
    from oracle import theory
    assert theory.bdf1_closed_form(prob.N, prob.kappa, prob.tau, 8.0) > 1.0     # lambda = 2/h^2, h = 1/2
    res = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("PINT_NO_GRAPH", "1")
        with pint.Plan.from_problem(prob) as p:
            it, u, st = p.solve(1e-12, 100, raise_on_fail=False)
            assert st == pint.PINT_ERR_DIVERGED, (it, u, st)
            assert it < 100
            res.append((it, u))
    monkeypatch.delenv("PINT_NO_GRAPH")
    assert res[0] == res[1], res


@pytest.mark.parametrize("mx,my,N,k", [(63, 1, 64, 2), (63, 30, 256, 3), (1023, 1, 1024, 4)])
def test_graph_replay_matches_eager(pint, monkeypatch, mx, my, N, k):
    """The fused iteration replayed as a CUDA graph (default) gives bit-identical iterates and
    update norms to eager launches (PINT_NO_GRAPH=1), also across pint_set_problem calls that
    change the kernel arguments (a forcing with a different nk forces a re-capture) and across
    timing-mode (eager) iterations in between; the reported launch counts agree."""
    prob1 = inputs.random_complex_problem(mx, my, N, k, 0.05, 1.0, R=1, seed=mx + k)
    prob2 = inputs.random_complex_problem(mx, my, N, k, 0.02, 1.0, R=1, seed=mx + k + 1)
    phi = prob2.phi.copy()
    phi[:, 6:] = 0.0                         # forcing on the first 5 levels: nk = 5
    prob2 = prob2.with_(phi=phi)
    monkeypatch.setenv("PINT_NO_GRAPH", "1")
    eager = pint.Plan.from_problem(prob1)
    monkeypatch.delenv("PINT_NO_GRAPH")
    graph = pint.Plan.from_problem(prob1)
    try:
        for p in (eager, graph):
            assert p.path()["fused"]
        l0 = [p.info()["kernel_launches"] for p in (eager, graph)]
        for it in range(4):
            if it == 2:
                graph.set_timing(True)   # event nodes inside the replayed graph
            ue, ug = eager.iterate(), graph.iterate()
            if it == 2:
                tm = graph.get_timing()
                assert tm["spass_launches"] == 1 and tm["tpass_launches"] == 1, tm
                assert tm["spass_ms"] > 0.0 and tm["tpass_ms"] > 0.0, tm
            graph.set_timing(False)
            assert ue == ug, (it, ue, ug)
        assert [p.info()["kernel_launches"] - l for p, l in zip((eager, graph), l0)] == [8, 8]
        assert np.array_equal(eager.get_solution(), graph.get_solution())
        for p in (eager, graph):
            p.set_problem(prob2.v, np.ascontiguousarray(prob2.g), prob2.phi, prob2.dphi)
            assert p.path()["nk"] == 5
        ups = [(eager.iterate(), graph.iterate()) for _ in range(3)]
        assert all(a == b for a, b in ups), ups
        sol = graph.get_solution()
        assert np.array_equal(eager.get_solution(), sol)
        assert rel(sol, wr.wr_naive(prob2, 3, dft="fft")[3]) <= TOL
    finally:
        eager.close()
        graph.close()


FEM_CASES = [
    ("fem_63_bdf2", lambda: inputs.random_complex_problem(63, 1, 64, 2, 0.1, 1.0, R=2, seed=12).with_(space="fem"), 4),
    ("fem_1023_bdf4", lambda: inputs.random_complex_problem(1023, 1, 1024, 4, 0.01, 1.0, R=1, seed=11).with_(space="fem"), 3),
    ("fem_example1_bdf3", lambda: inputs.example1_fem(3, M=1023, N=128), 3),
    ("fd_modal_1d_bdf6", lambda: inputs.random_complex_problem(255, 1, 256, 6, 0.05, 1.0, R=1, seed=13), 3),
    # CQ (streaming path, Step 2 as an elementwise division in the modes)
    ("fem_cq_a05_bdf2", lambda: inputs.random_complex_problem(127, 1, 128, 2, 0.05, 0.5, R=1, seed=14).with_(space="fem"), 3),
    ("fem_example2_cq", lambda: inputs.example2_fd(2, M=255, N=256).with_(space="fem"), 3),
    ("fd_modal_2d_cq", lambda: inputs.random_complex_problem(31, 63, 64, 3, 0.05, 0.3, R=2, seed=15), 3),
]


@pytest.mark.parametrize("name,make,iters", FEM_CASES, ids=[c[0] for c in FEM_CASES])
def test_fem_and_modal_1d(pint, name, make, iters):
    """1D on the fully modal path: P1 FEM (PINT_OP_FEM1D_DIRICHLET) and the FD
    operator with PINT_FLAG_MODAL, against the oracle (FEM: A = M^{-1} K), every iterate; then
    wr_solve converges to the oracle's sequential stepping in the same discretisation."""
    prob = make()
    o = wr.wr_naive(prob, iters, dft="fft")
    kw = {} if prob.space == "fem" else {"modal": True}
    errs = []
    N, k = prob.N, prob.k
    with pint.Plan.from_problem(prob, **kw) as p:
        assert p.path()["fused"] is (prob.alpha == 1.0)
        for m in range(1, iters + 1):
            p.iterate()
            win = p.get_levels(N - k, k)          # window levels before materialisation
            errs.append(float(np.linalg.norm(win - o[m][N - k:]) / np.linalg.norm(o[m])))
            errs.append(rel(p.get_solution(), o[m]))
        it, u, st = p.solve(1e-12, 40, raise_on_fail=False)
        if st != 0:   # diagnostics: the update history of plain iterations from here
            hist = [p.iterate() for _ in range(6)]
            print(name, "solve status", st, "iterations", it, "last update", u, "then", hist)
        seq_err = rel(p.get_solution(), sequential.sequential(prob))
    print(name, errs, it, seq_err)
    assert max(errs) <= TOL, errs
    assert st == 0 and seq_err <= 1e-9, (st, seq_err)


def test_plan_buffers_zero_filled_after_dirty_memory(pint):
    """Device memory left dirty by earlier allocations must not reach the iteration: the fully modal
    plans' physical-window monitor once read never-written pad slots of its window buffers, which gave a
    constant, run-dependent update floor (2.7e-10 on fem_63_bdf2 after other tests) and a solve that
    never reached 1e-12.  Plan allocations are zero-filled since."""
    import torch
    # large-pool and small-pool (2 MB segment) allocations, filled, then handed back to the driver
    junk = [torch.full((1 << 24,), 1e3 * (i + 1), dtype=torch.float64, device="cuda:0") for i in range(8)]
    junk += [torch.full((1 << 15,), 7e2 + i, dtype=torch.float64, device="cuda:0") for i in range(512)]
    torch.cuda.synchronize()
    del junk
    torch.cuda.empty_cache()                      # give the dirty segments back to the driver
    prob = inputs.random_complex_problem(63, 1, 64, 2, 0.1, 1.0, R=2, seed=12).with_(space="fem")
    with pint.Plan.from_problem(prob) as p:
        it, u, st = p.solve(1e-12, 40, raise_on_fail=False)
        assert st == 0 and it <= 8, (st, it, u)
        assert p.iterate() < 1e-14


def test_fem_rejects_unsupported(pint):
    prob = inputs.random_complex_problem(62, 1, 64, 2, 0.1, 1.0, R=0, seed=1).with_(space="fem")   # 2(mx+1) = 126
    with pytest.raises(pint.PintError) as e:
        pint.Plan.from_problem(prob)
    assert e.value.status == pint.PINT_ERR_UNSUPPORTED


@pytest.mark.parametrize("make", [
    lambda: inputs.random_complex_problem(63, 1, 128, 3, 0.05, 1.0, R=1, seed=21),
    lambda: inputs.random_complex_problem(31, 15, 64, 2, 0.1, 0.6, R=1, seed=22),
    lambda: inputs.random_complex_problem(63, 1, 64, 2, 0.1, 1.0, R=1, seed=23).with_(space="fem"),
], ids=["heat1d_stream", "cq2d", "fem_heat_stream"])
def test_streaming_modal_and_initial_guess(pint, make):
    """The streaming modal path (PINT_FLAG_MODAL with PINT_FLAG_STREAM or CQ): iterates vs the
    oracle, and a user initial guess (the sequential solution, DST'd into the modes at
    pint_set_initial_guess) is a fixed point."""
    prob = make()
    o = wr.wr_naive(prob, 2, dft="fft")
    kw = {"modal": True, "stream_path": True} if prob.space == "fd" else {"stream_path": True}
    with pint.Plan.from_problem(prob, **kw) as p:
        assert not p.path()["fused"]
        errs = []
        for m in (1, 2):
            p.iterate()
            errs.append(rel(p.get_solution(), o[m]))
        assert max(errs) <= TOL, errs
        Us = sequential.sequential(prob)
        p.set_initial_guess(np.ascontiguousarray(Us))
        u = p.iterate()
        assert u < 1e-10 * np.abs(Us).max(), u
        assert rel(p.get_solution(), Us) < 1e-10


@pytest.mark.parametrize("make,kw", [
    (lambda: inputs.config_c1(), {}),
    (lambda: inputs.random_complex_problem(63, 40, 128, 4, 0.05, 1.0, R=1, seed=31), {}),
    (lambda: inputs.random_complex_problem(63, 40, 128, 4, 0.05, 1.0, R=1, seed=31), {"stream_path": True}),
    (lambda: inputs.random_complex_problem(100, 1, 256, 6, 0.01, 1.0, R=2, seed=33), {}),
    (lambda: inputs.random_complex_problem(31, 63, 128, 3, 0.05, 1.0, R=1, seed=34), {"modal": True}),
    (lambda: inputs.random_complex_problem(63, 1, 128, 2, 0.05, 1.0, R=1, seed=35).with_(space="fem"), {}),
    (lambda: inputs.random_complex_problem(63, 1, 256, 2, 0.05, 0.5, R=1, seed=36), {}),
    (lambda: inputs.config_c5(m=63), {}),
], ids=["C1", "2d_fused", "2d_stream", "1d_bdf6", "2d_modal", "fem", "cq1d", "c5_63"])
def test_gpu_residual_self_check(pint, make, kw):
    """pint_residual: the GPU's own fixed-point residual of the BDF-k scheme equals
    the oracle residual of the same iterate at m = 1 (far from convergence) and drops to round-off
    at the WR fixed point."""
    from oracle import nonlinear, problem, spatial
    prob = make()
    with pint.Plan.from_problem(prob, **kw) as p:
        p.iterate()
        r1, f1 = p.residual()
        U = p.get_solution()
        # oracle residual of the same iterate in the scheme's own form, eqn:BDF: history
        # U^{<=0} = v on the left and f̄_n on the right (the GPU uses the all-at-once form with the
        # history moved into F_static, so the two agree only if both are right)
        R = nonlinear.dbar(prob, U) + np.stack([spatial.apply_A(U[n], prob.mx, prob.my, prob.space)
                                                for n in range(prob.N)]) - problem.fbar(prob)
        modal_plan = kw.get("modal", False) or prob.space == "fem"
        if prob.my > 1:                                          # the plan works in the DST-x basis
            R = spatial.dst1(R.reshape(prob.N, prob.my, prob.mx), axis=-1)
            if modal_plan:                                       # ... and DST-y on modal plans
                R = spatial.dst1(R, axis=-2)
        elif modal_plan:                                         # 1D modal / FEM: DST along the line
            R = spatial.dst1(R, axis=-1)
        ro = float(np.abs(R).max())
        assert r1 > 1e-8 * f1                                      # not converged after one iteration
        assert abs(r1 - ro) <= 1e-9 * ro, (r1, ro)
        it, u, st = p.solve(1e-13, 60, raise_on_fail=False)
        r, f = p.residual()
        assert r <= 1e-9 * f, (r, f, it, u)


def test_gpu_residual_unsupported(pint):
    """pint_residual is not available for CQ on the modal path and for the DST ablation."""
    cq = inputs.random_complex_problem(31, 15, 64, 2, 0.1, 0.5, R=1, seed=37)
    heat = inputs.random_complex_problem(31, 15, 64, 2, 0.1, 1.0, R=1, seed=38)
    for prob, kw in ((cq, {"modal": True}), (heat, {"dst_per_iter": True})):
        with pint.Plan.from_problem(prob, **kw) as p:
            p.iterate()
            with pytest.raises(pint.PintError) as e:
                p.residual()
            assert e.value.status == pint.PINT_ERR_UNSUPPORTED


def test_api_edge_cases(pint):
    """Empty and out-of-range reads, zero-iteration solves, resets and state errors."""
    P = pint
    prob = inputs.random_complex_problem(31, 9, 64, 3, 0.1, 1.0, R=1, seed=41)
    with P.Plan.from_problem(prob) as p:
        with pytest.raises(P.PintError) as e:
            p.residual()                                      # no iterate yet
        assert e.value.status == P.PINT_ERR_STATE
        it, u, st = p.solve(1e-12, 0, raise_on_fail=False)   # zero iterations allowed
        assert it == 0 and st == P.PINT_ERR_NOT_CONVERGED
        p.iterate()
        assert p.get_levels(5, 0).shape == (0, prob.M)       # empty read
        for n0, cnt in ((-1, 1), (prob.N, 1), (prob.N - 1, 2)):
            with pytest.raises(P.PintError) as e:
                p.get_levels(n0, cnt)
            assert e.value.status == P.PINT_ERR_ARG
        U = p.get_solution()
        assert np.array_equal(p.get_levels(prob.N - 1, 1)[0], U[-1])
        p.set_initial_guess(None)                             # back to U_0^n = v, m = 0
        assert p.info()["m"] == 0
        with pytest.raises(P.PintError) as e:
            p.get_solution()
        assert e.value.status == P.PINT_ERR_STATE
        p.iterate()
        assert rel(p.get_solution(), U) < 1e-14                # the same first iterate again


@pytest.mark.parametrize("make,kw", [
    (lambda: inputs.random_complex_problem(63, 1, 64, 2, 0.1, 1.0, R=1, seed=51).with_(space="fem"), {}),
    (lambda: inputs.random_complex_problem(31, 63, 128, 4, 0.05, 1.0, R=1, seed=52), {"modal": True}),
    (lambda: inputs.random_complex_problem(31, 63, 128, 4, 0.05, 1.0, R=1, seed=53).real_part(), {"modal": True, "real_data": True}),
], ids=["fem_fused", "modal2d_fused", "modal2d_real"])
def test_fused_modal_initial_guess(pint, make, kw):
    """Fused modal plans (P1-FEM, 2D modal): the sequential solution as a user initial guess is a
    fixed point (update at round-off from the first iteration on)."""
    prob = make()
    Us = sequential.sequential(prob)
    with pint.Plan.from_problem(prob, **kw) as p:
        assert p.path()["fused"]
        p.set_initial_guess(np.ascontiguousarray(Us))
        us = [p.iterate() for _ in range(2)]
        assert max(us) < 1e-10 * np.abs(Us).max(), us
        assert rel(p.get_solution(), Us) < 1e-10


@pytest.mark.parametrize("make,tol", [
    (lambda: inputs.config_c1(), 1e-12),
    (lambda: inputs.config_c2(k=3, kappa=1e-2), 1e-12),
    (lambda: inputs.config_c2(k=6, kappa=1e-3), 1e-10),
    (lambda: inputs.random_complex_problem(63, 30, 256, 3, 0.05, 1.0, R=1, seed=41), 1e-11),
])
def test_device_loop_matches_host_loop(pint, monkeypatch, make, tol):
    """pint_wr_solve on the fused path runs its loop on the device (while-conditional graph node, the
    stopping rule in a kernel): same iteration count, update norm and iterate as the host loop
    (PINT_NO_GRAPH=1), in one or several calls, and pint_wr_run(K) equals K pint_wr_iterate calls."""
    prob = make()
    monkeypatch.setenv("PINT_NO_GRAPH", "1")
    host = pint.Plan.from_problem(prob)
    monkeypatch.delenv("PINT_NO_GRAPH")
    dev = pint.Plan.from_problem(prob)
    try:
        assert dev.path()["fused"]
        l0 = dev.info()["kernel_launches"]
        ih, uh, sh = host.solve(tol, 30, raise_on_fail=False)
        idv, ud, sd = dev.solve(tol, 30, raise_on_fail=False)
        print(f"{prob.name}: host loop {ih} it (update {uh:.3e}, status {sh}); device loop {idv} it ({ud:.3e}, {sd})")
        assert (ih, sh) == (idv, sd) and sh == pint.PINT_OK
        assert ud == uh
        # one cooperative kernel per solve (small problems), or fused + finish per iteration (graph loop)
        assert dev.info()["m"] == idv and dev.info()["kernel_launches"] - l0 in (1, 2 * idv)
        assert np.array_equal(host.get_solution(), dev.get_solution())
        # a second solve continues from the converged state (parity and guard state carried over)
        assert host.solve(tol, 5, raise_on_fail=False)[:2] == dev.solve(tol, 5, raise_on_fail=False)[:2]
        # max_iters bound on the device: NOT_CONVERGED after exactly 2 iterations
        it2, _, st2 = dev.solve(0.0, 2, raise_on_fail=False)
        assert (it2, st2) == (2, pint.PINT_ERR_NOT_CONVERGED)
    finally:
        host.close()
        dev.close()
    # pint_wr_run: K iterations with one synchronisation == K pint_wr_iterate calls
    with pint.Plan.from_problem(prob) as a, pint.Plan.from_problem(prob) as b:
        ua = [a.iterate() for _ in range(5)][-1]
        ub = b.run(5)
        assert ua == ub and b.info()["m"] == 5
        assert np.array_equal(a.get_solution(), b.get_solution())
        b.run(1)
        a.iterate()
        assert np.array_equal(a.get_solution(), b.get_solution())


def test_wr_run_streaming_and_args(pint):
    """pint_wr_run on the streaming (CQ) path: K iterations enqueued, one synchronisation; argument checks."""
    prob = inputs.random_complex_problem(31, 20, 256, 2, 0.1, 0.6, R=1, seed=21)
    with pint.Plan.from_problem(prob) as a, pint.Plan.from_problem(prob) as b:
        ua = [a.iterate() for _ in range(3)][-1]
        ub = b.run(3)
        assert ua == ub
        assert np.array_equal(a.get_solution(), b.get_solution())
        with pytest.raises(pint.PintError) as e:
            b.run(0)
        assert e.value.status == pint.PINT_ERR_ARG


@pytest.mark.parametrize("mx,my,N,k,real", [(63, 31, 256, 3, False), (127, 63, 512, 6, True), (255, 1, 256, 2, False)])
def test_modal_window_monitor_is_physical(pint, mx, my, N, k, real):
    """Fully modal heat plans monitor the window update with the line axis back in grid space (DST-y
    every iteration): 1D the grid values, 2D the DST-x basis of the line path (reading R-norm2D) — the
    oracle's max over the window levels in that basis, not the modal-basis norm, which the orthonormal
    DSTs scale by up to sqrt(M)."""
    from oracle import spatial
    prob = inputs.random_complex_problem(mx, my, N, k, 0.05, 1.0, R=1, seed=mx + k)
    if real:
        prob = prob.real_part()
    o = wr.wr_naive(prob, 4, dft="fft")
    basis = (lambda U: U) if my == 1 else \
        (lambda U: spatial.dst1(U.reshape(U.shape[0], my, mx), axis=2).reshape(U.shape[0], -1))
    ou = [float(np.abs(basis(o[m][N - k:]) - basis(o[m - 1][N - k:])).max()) for m in range(1, 5)]
    with pint.Plan.from_problem(prob, modal=True) as p:
        assert p.path()["fused"]
        gu = [p.iterate() for _ in range(4)]
    print(f"modal {mx}x{my}: oracle window updates " + " ".join(f"{u:.3e}" for u in ou) + "; GPU " + " ".join(f"{u:.3e}" for u in gu))
    for g, u in zip(gu, ou):
        assert abs(g - u) <= 1e-6 * u + 1e-13 * ou[0], (g, u)


FEM2D_CASES = [
    ("example3_k3_a0.5", lambda: inputs.example3_fem(k=3, m=31, N=64)),
    ("example3_k2_a0.5_m63", lambda: inputs.example3_fem(k=2, m=63, N=128)),
    ("heat_k4_rand", lambda: inputs.random_complex_problem(31, 31, 64, 4, 0.05, 1.0, R=1, seed=17).with_(space="fem")),
    ("cq_k1_rand", lambda: inputs.random_complex_problem(15, 15, 32, 1, 0.1, 0.7, R=1, seed=18).with_(space="fem")),
]


@pytest.mark.parametrize("name,make", FEM2D_CASES, ids=[c[0] for c in FEM2D_CASES])
def test_fem2d_parity(pint, name, make):
    """2D P1 FEM on the uniform triangulation (the paper's Example 3 setting, reduced grid): every
    iterate against the oracle (sparse LU of s_p M + K per frequency), m = 1..3, and wr_solve's fixed
    point against sequential FEM stepping."""
    prob = make()
    o = wr.wr_naive(prob, 3, dft="fft", wrap="fft")
    with pint.Plan.from_problem(prob) as p:
        assert not p.path()["fused"]
        for m in range(1, 4):
            p.iterate()
            err = rel(p.get_solution(), o[m])
            print(f"{name}: m={m} rel L2 vs oracle {err:.2e}")
            assert err < TOL, (m, err)
        it, u, st = p.solve(1e-12, 30)
        assert st == pint.PINT_OK
        Us = sequential.sequential(prob)
        err = rel(p.get_solution(), Us)
        print(f"{name}: fixed point after {it + 3} iterations vs sequential FEM stepping {err:.2e}")
        assert err < 1e-10
        with pytest.raises(pint.PintError) as e:
            p.residual()
        assert e.value.status == pint.PINT_ERR_UNSUPPORTED
    with pytest.raises(pint.PintError) as e:
        pint.Plan(prob.mx, prob.my, prob.N, prob.k, prob.kappa, prob.tau, prob.alpha, fem=True, rank=0, nranks=2,
                  allreduce_max=lambda x: x)
    assert e.value.status == pint.PINT_ERR_UNSUPPORTED
