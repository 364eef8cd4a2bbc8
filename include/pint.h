/*
 * pint.h — C ABI of the B200-native ParaDiag waveform-relaxation hot path of
 * arXiv 2007.13125 (Wu & Zhou): parallel-in-time BDFk (k = 1..6) for u_t + A u = f and
 * CQ-BDFk for the Caputo subdiffusion problem d_t^alpha u + A u = f, A = -Delta_h (FD,
 * homogeneous Dirichlet, unit interval / unit square, h = 1/(m+1)).
 *
 * One waveform-relaxation (WR) iteration U_{m-1} -> U_m solves the kappa-periodic
 * all-at-once system   (1/tau^a)(B_k(kappa) (x) I) U_m + (I (x) A) U_m = F_{m-1}
 * (PAPER.md:403-430 eq:BDF-k-matrix; PAPER.md:1021-1038 eq:BDF-k-matrix-frac) by
 * Algorithm 1/2:
 *   F_{m-1}  = f̄ + tau^-a (sum_{j<n} w_j) v + kappa-wrap(U_{m-1})   (eqn:BDF-k-F, eq:BDF-subdiff-F)
 *   Step 1   H = V^{-1} Gamma_kappa F         (scale by kappa^{(n-1)/N}, batched time FFT / N)
 *   Step 2   (d_p/tau^a + A) Q_p = H_p, p = 0..N-1   (complex-shifted spatial solves)
 *   Step 3   U_m = Gamma_kappa^{-1} V Q        (inverse time FFT, unscale)
 * Data layout, kernels and readings of the paper: DESIGN.md.
 *
 * Conventions
 *   - All entry points return pint_status; no exception or abort crosses the ABI.  On error
 *     pint_last_error() (thread-local) holds a one-line message naming the bound violated.
 *   - Complex data are complex128: interleaved (re, im) doubles, 16 bytes per value.
 *   - Space index i = iy*mx + ix (x fastest); space-time arrays are time-major [n][i],
 *     n = 1..N stored at rows 0..N-1 (U^n = approximation at t_n = n*tau).
 *   - mem = PINT_HOST: the pointer is host memory (pageable or pinned); PINT_DEVICE: device
 *     memory on the plan's device.  Inputs are copied during the call (the caller may free
 *     them on return); outputs are written into caller buffers before the call returns.
 *   - A plan is bound to one device and one CUDA stream, is not thread-safe, and owns all
 *     its device workspace.  Distinct plans are independent.
 *   - Calls that return host scalars (pint_wr_iterate, pint_wr_solve, getters) synchronise
 *     the plan stream.
 *   - Multi-GPU (2D operators only): each rank creates a plan with the GLOBAL sizes and its
 *     rank/nranks; the plan owns the contiguous x-mode slab [q_begin, q_end) of the hoisted
 *     DST-I basis (pint_get_partition).  The WR iteration needs no data exchange between
 *     slabs (the x-modes decouple exactly); the only collective is the all-reduce(max) of
 *     the update norm, done through the caller-supplied allreduce_max callback.
 *     The collective calls (pint_wr_iterate, pint_wr_solve, pint_residual) make the same
 *     allreduce_max calls on every rank even when the local part fails on one rank: that rank
 *     returns its own error, the others see a non-finite update (wr_solve: DIVERGED) or
 *     PINT_ERR_COMM (residual) instead of blocking in the collective.
 */
#ifndef PINT_H_
#define PINT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pint_plan_s* pint_plan;

typedef enum {
  PINT_OK = 0,
  PINT_ERR_ARG = 1,            /* argument outside its documented range (message names it) */
  PINT_ERR_ALLOC = 2,          /* device/host allocation failed */
  PINT_ERR_CUDA = 3,           /* CUDA runtime error (message holds cudaGetErrorString) */
  PINT_ERR_COMM = 4,           /* allreduce_max callback returned non-zero */
  PINT_ERR_STATE = 5,          /* call out of order (e.g. iterate before set_problem) */
  PINT_ERR_NOT_CONVERGED = 6,  /* pint_wr_solve hit max_iters; solution still retrievable */
  PINT_ERR_DIVERGED = 7,       /* update grew 3 times in a row, or became NaN/Inf */
  PINT_ERR_UNSUPPORTED = 8     /* valid but not implemented on this path (message says what) */
} pint_status;

/* PINT_OP_FEM1D_DIRICHLET: the paper's own discretisation of Examples 1-2 (PAPER.md:1374-1375,
 * SURVEY §8(f) item 4): piecewise-linear Galerkin on the uniform mesh of (0,1), h = 1/(mx+1),
 * stiffness K = (1/h) tridiag(-1,2,-1), mass M = (h/6) tridiag(1,4,1); the plan solves
 * U' + A U = f~ with A = M^{-1} K (v, g_r, U: nodal coefficient vectors; f~ the projected or
 * interpolated forcing).  my must be 1.  It runs on the fully modal path (the DST diagonalises
 * both K and M: lambda_j = K_j / M_j; heat: fused modal kernel, CQ: streaming path with the
 * shifted solves as divisions), so it needs 2(mx+1) a power of two (UNSUPPORTED otherwise);
 * PINT_FLAG_MODAL is implied. */
/* PINT_OP_FEM2D_DIRICHLET: P1 finite elements on the uniform triangulation of the unit square
 * (Example 3), each cell split by its '/' diagonal (DESIGN.md reading
 * R-FEM2D), mx = my interior nodes per axis, h = 1/(mx+1); nodal coefficient vectors as in 1D.  The
 * stiffness is h^2 times the 5-point Laplacian and the mass matrix M = h^2 (M_sym + E) couples the
 * '/' diagonal neighbours, so M is not diagonalised by the DSTs: Step 2, (s_p M + K) W = M H, is
 * solved by a fixed-point iteration preconditioned by the DST-diagonal s_p M_sym + K (fem2d.cuh),
 * iterated to round-off.  Runs on the fully modal streaming path (PINT_FLAG_MODAL | PINT_FLAG_STREAM
 * implied); needs 2(mx+1) a power of two, one rank (UNSUPPORTED otherwise); pint_residual is
 * UNSUPPORTED (A = M^{-1} K is not diagonal in the modes). */
enum { PINT_OP_FD1D_DIRICHLET = 1, PINT_OP_FD2D_DIRICHLET = 2, PINT_OP_FEM1D_DIRICHLET = 3,
       PINT_OP_FEM2D_DIRICHLET = 4 };
enum { PINT_HOST = 0, PINT_DEVICE = 1 };
enum {
  PINT_FLAG_U0_ZERO = 1,       /* WR initial guess U_0 = 0 instead of U_0^n = v */
  PINT_FLAG_FULL_FFT = 2,      /* heat, streaming path: run the unpruned time FFTs every iteration
                                  (A/B, tests); default prunes to the k window outputs / n_k inputs */
  PINT_FLAG_STREAM = 4,        /* heat: use the two-pass streaming iteration (H and W arrays in HBM)
                                  instead of the default fused one-kernel iteration (A/B, tests) */
  PINT_FLAG_DST_PER_ITER = 8,  /* 2D, one rank: ablation of the DST hoisting: keep
                                  the arrays in physical x and apply DST-x before and after the
                                  shifted solves every iteration (streaming path; same iterate) */
  PINT_FLAG_REAL_DATA = 16,    /* heat, fused path: v, g_r (and U_0) are real, so W_{N-p} = conj(W_p)
                                  and only the frequencies p <= N/2 are solved (SURVEY §8(f) item
                                  2b); pint_set_problem_separable returns ARG for complex data */
  PINT_FLAG_MODAL = 32,        /* fully modal variant — the DST is applied
                                  along the line axis as well (2D: y; 1D: x; hoisted), every mode is
                                  a scalar problem and the shifted solves are divisions (heat: the
                                  fused modal kernel; CQ or PINT_FLAG_STREAM: the streaming path with
                                  an elementwise division pass); needs 2(L+1) a power of two, L = my
                                  (2D) or mx (1D) (UNSUPPORTED otherwise); excludes
                                  PINT_FLAG_DST_PER_ITER (ARG) */
  PINT_FLAG_FULL_UPDATE_NORM = 64  /* update monitor over ALL N levels and points: the paper's stopping
                                  rule max_n |U_m^n - U_{m-1}^n|_inf.
                                  Always on for CQ plans (alpha < 1: the kappa-wrap reads every level
                                  of U_{m-1}, so the k-level window does not bound
                                  the update).  Heat: opt-in; selects the streaming path with unpruned
                                  time FFTs.  Costs one more space-time array (U_{m-1}, N*M*16 B) and
                                  32 B of HBM traffic per unknown per iteration; pint_get_levels then
                                  reads U_m from it without re-materialising.  2D: the norm is taken in
                                  the hoisted DST-x basis (orthonormal in x; reading R-norm2D),
                                  fully modal plans in the DST basis of both axes. */
};

typedef struct {
  int32_t kind;                /* PINT_OP_FD1D_DIRICHLET, PINT_OP_FD2D_DIRICHLET, PINT_OP_FEM1D_DIRICHLET or
                                  PINT_OP_FEM2D_DIRICHLET */
  int64_t mx, my;              /* grid points per axis (1D: my = 1); M = mx*my */
} pint_operator;

/* All-reduce(max) over ranks of one double, in place.  Return 0 on success. */
typedef int (*pint_allreduce_max_fn)(double* inout, void* ctx);

typedef struct {
  double alpha;                /* 1.0 = heat (BDFk); (0,1) = Caputo order, CQ-BDFk weights */
  int32_t device;              /* CUDA device ordinal */
  void* stream;                /* cudaStream_t to run on; NULL = plan-owned stream */
  int32_t flags;               /* PINT_FLAG_* */
  int32_t rank, nranks;        /* x-mode slab partition (2D); 0, 1 for one GPU */
  pint_allreduce_max_fn allreduce_max;   /* required when nranks > 1 */
  void* allreduce_ctx;
} pint_options;

/* Create a plan for N time steps of size tau with BDF order k and relaxation parameter kappa
 * (the kappa-wrapped scheme eqn:BDF-iter; CQ: eqn:CQ-iter).
 * Builds the Step-1..3 tables of Algorithm 1 / 2: Gamma, d_p, twiddles.
 * M must equal op->mx * op->my.  Errors (PINT_ERR_ARG): k not in 1..6; kappa not in (0,1);
 * tau <= 0; N < k+1; alpha not in (0,1]; M != mx*my; mx, my < 1; rank/nranks invalid or
 * nranks > mx; nranks > 1 with a 1D operator.  PINT_ERR_UNSUPPORTED: N not a power of two in
 * [16, 4096]; line length (1D: mx, 2D: my) > 1024; 2D with 2(mx+1) not a power of two <= 4096.
 * Validation happens before any CUDA call.  On success *out owns device buffers of about
 * 2*N*M*16 bytes (this rank's slab) plus O((k+R)*M) vectors and O(N) tables. */
pint_status pint_plan_create(int64_t M, int64_t N, int32_t k, double kappa, double tau,
                             const pint_operator* op, const pint_options* opt, pint_plan* out);

/* Problem data with separable forcing f(t, x) = sum_{r<R} phi_r(t) g_r(x):
 *   v    [M] complex: initial value u(0)
 *   g    [R][M] complex (R may be 0, then g/phi/dphi may be NULL)
 *   phi  [R][N+1] double: phi_r(t_n), n = 0..N (host memory always)
 *   dphi [R][max(k-2,0)] double: d^l phi_r / dt^l (0), l = 1..k-2, for the Table-1 starting
 *        corrections b_{l,n} (host memory always)
 * v and g are read from mem (PINT_HOST / PINT_DEVICE; full global arrays on every rank).
 * Builds the static right-hand side coefficients and bootstraps the iteration from U_0
 * (U_0^n = v, or 0 with PINT_FLAG_U0_ZERO): afterwards the iteration count is m = 0. */
pint_status pint_set_problem_separable(pint_plan plan, const void* v, int32_t R, const void* g,
                                       const double* phi, const double* dphi, int32_t mem);

/* Problem data with a dense (non-separable) forcing:
 *   v      [M] complex: u(0)
 *   f      [N][M] complex: f(t_n), n = 1..N (row n-1)
 *   f0     [M] complex: f(0) for the starting correction a_n f(0) (Table 1); NULL = 0
 *   fderiv [max(k-2,0)][M] complex: d^l f/dt^l (0), l = 1..k-2 (b_{l,n} corrections); NULL = 0
 * in memory space mem.  The corrections become separable sources; f(t_n) is stored as a dense
 * right-hand side (16 B per unknown, DST-x applied per level in 2D) that the streaming T-pass adds to
 * F_static, so the plan runs the streaming path (unpruned T-pass) afterwards.  One rank only
 * (UNSUPPORTED otherwise, and with PINT_FLAG_MODAL / PINT_FLAG_DST_PER_ITER).  A plan cannot switch
 * between the separable form with another R and this form (STATE).  Bootstraps like
 * pint_set_problem_separable. */
pint_status pint_set_problem(pint_plan plan, const void* v, const void* f, const void* f0, const void* fderiv,
                             int32_t mem);

/* Replace the WR initial guess by a full space-time array U0 [N][M] (this is U_0^1..U_0^N, the
 * m = 0 iterate of eqn:BDF-iter; the paper starts from U_0^n = v, PAPER.md:173;
 * requires a prior pint_set_problem_separable).  Resets m to 0. */
pint_status pint_set_initial_guess(pint_plan plan, const void* U0, int32_t mem);

/* One WR iteration m-1 -> m.  *update_inf (may be NULL) receives the max over ranks of
 * max |U_m^n(x) - U_{m-1}^n(x)| over the monitored levels: every level n = 1..N for CQ plans and
 * with PINT_FLAG_FULL_UPDATE_NORM, else the window n = N-k+1..N (the wrap
 * state, which determines the next iterate for heat).
 * The fused heat iteration is replayed as a CUDA graph on the plan stream (captured on first use,
 * re-captured when the problem changes; PINT_NO_GRAPH=1 in the environment: eager launches). */
pint_status pint_wr_iterate(pint_plan plan, double* update_inf);

/* Iterate until update < tol (the paper's stopping rule), or max_iters
 * iterations (PINT_ERR_NOT_CONVERGED), or the update
 * grows 3 consecutive times / is not finite (PINT_ERR_DIVERGED).  *iters, *update_inf may be NULL.
 * Fused heat path on one rank: the whole loop runs on the device (a CUDA graph with a while-conditional
 * node; the stopping rule is evaluated by a kernel after every iteration) — one host synchronisation
 * per call; same iterates and stop count as the host loop (other paths, timing mode, several ranks). */
pint_status pint_wr_solve(pint_plan plan, double tol, int32_t max_iters, int32_t* iters,
                          double* update_inf);

/* Run exactly `iters` >= 1 WR iterations (Algorithm 1 / 2 Steps 1-3 each, PAPER.md:468-477,
 * 1053-1061; no stopping rule, no divergence guard) with one host
 * synchronisation at the end; *update_inf (may be NULL) receives the last iteration's update (max over
 * ranks: one all-reduce per call).  The throughput call of bench.py. */
pint_status pint_wr_run(pint_plan plan, int32_t iters, double* update_inf);

/* Copy the current iterate U_m (Step 3's output; the fused heat path materialises
 * it here from the window state), time levels n_begin+1 .. n_begin+n_count (0-based row
 * n_begin .. n_begin+n_count-1 of the [N][M] array), into U [n_count][M] complex in mem.
 * 2D with nranks > 1: returns PINT_ERR_UNSUPPORTED (use the modal-slab calls below). */
pint_status pint_get_levels(pint_plan plan, int64_t n_begin, int64_t n_count, void* U, int32_t mem);
/* = pint_get_levels(plan, 0, N, U, mem) */
pint_status pint_get_solution(pint_plan plan, void* U, int32_t mem);

/* Multi-GPU output path (the p-processor split of PAPER.md:493-508, here over x-modes, which needs
 * no exchange once DST-x is hoisted): this rank's slab of U_m in the DST-x basis, layout
 * [n_count][my][q_end-q_begin] (mode q global index q_begin+j), and the inverse DST-I that
 * maps a gathered full modal array [n_count][my][mx] to physical [n_count][my][mx]. */
pint_status pint_get_modal_levels(pint_plan plan, int64_t n_begin, int64_t n_count, void* Uq, int32_t mem);
pint_status pint_modal_to_physical(pint_plan plan, int64_t n_count, const void* Uq_full, void* U, int32_t mem);

/* Host-only (no CUDA call; partition of the Step-2 systems over p ranks): the
 * contiguous, balanced x-mode slab of `rank` among `nranks`
 * for mx modes: [floor(rank*mx/nranks), floor((rank+1)*mx/nranks)).  PINT_ERR_ARG if
 * nranks < 1, rank outside [0, nranks) or nranks > mx. */
pint_status pint_partition(int64_t mx, int32_t rank, int32_t nranks, int64_t* q_begin, int64_t* q_end);

/* This rank's x-mode slab [q_begin, q_end) (1D: [0, 1)). */
pint_status pint_get_partition(pint_plan plan, int64_t* q_begin, int64_t* q_end);

/* Per-pass timing with CUDA events on the plan stream (bench/profiling):
 * enable != 0 starts accumulating; pint_get_timing returns total milliseconds and launch
 * counts of the T-pass (time-axis kernel) and S-pass (shifted-solve kernel) since enabled.
 * Fused heat path: the S-pass slot holds the fused kernel, the T-pass slot the finish kernel
 * (event nodes inside the replayed graph, which cost a few microseconds per iteration). */
pint_status pint_set_timing(pint_plan plan, int32_t enable);
pint_status pint_get_timing(pint_plan plan, double* tpass_ms, double* spass_ms,
                            int64_t* tpass_launches, int64_t* spass_launches);

/* ---- semilinear extension: Newton's method with WR inner solves ----
 * Problem: dbar^a u + A u + g(u) = f, u(0) = v, with the modified CQ-BDFk / BDFk scheme of
 * eqn:BDF-CQ-m-r, g(u) = (u^3 - u)/eps^2 (Allen-Cahn, Example 4,
 * PAPER.md:1714-1722).  Algorithm 3: U_0^n = v; Newton step l solves
 * (dbar^a + A + g'(Ubar_{l-1})) W = fbar - (dbar^a + A) U_{l-1} - g(U_{l-1}), W^{<=0} = 0, with
 * Ubar the mean over the N levels (reading R-NL-sign: +g'), by the WR
 * iteration (kappa-wrap) until max_n |W_m^n - W_{m-1}^n| < inner_tol, then
 * U_l = U_{l-1} + W.  1D operators on one rank only (g'(Ubar(x)) varies in x, so the line solves
 * are general tridiagonal systems: shift-accurate Thomas); always the streaming path. */
enum { PINT_NL_ALLEN_CAHN = 1 };

/* Make the plan semilinear with nonlinearity `kind` (g of eqn:BDF-CQ-m-r, PAPER.md:1660-1668;
 * Allen-Cahn) and width eps > 0.  The forcing f and v are
 * still given by pint_set_problem_separable (before or after this call); the Newton state is reset
 * to U_0 = v by either call.  Errors: ARG (kind, eps), UNSUPPORTED (2D or nranks > 1).
 * Afterwards pint_wr_iterate / pint_wr_solve return STATE and pint_get_levels returns U_l. */
pint_status pint_set_nonlinearity(pint_plan plan, int32_t kind, double eps);

/* Algorithm 3: run up to max_outer Newton steps from the current U_l (inner WR:
 * at most max_inner iterations, stop when the full-array max-norm update < inner_tol, the rule of
 * PAPER.md:1747-1748).  inner_counts[l] / outer_updates[l]
 * (arrays of max_outer entries, may be NULL) receive the inner iteration count and
 * max |U_l - U_{l-1}| of each step; *outer_done the number of steps run.  Returns OK when the
 * Newton update fell below outer_tol (or outer_tol == 0 and max_outer steps ran),
 * NOT_CONVERGED otherwise, DIVERGED on a non-finite update, STATE before set_problem/
 * set_nonlinearity. */
pint_status pint_newton_solve(pint_plan plan, int32_t max_outer, double outer_tol, double inner_tol,
                              int32_t max_inner, int32_t* inner_counts, double* outer_updates,
                              int32_t* outer_done);

/* Which iteration the plan runs for its current problem: *fused = 1 for the fused one-kernel heat
 * iteration (fused.cuh; no space-time array per iteration), 0 for the two-pass streaming one
 * (CQ, PINT_FLAG_STREAM, or more than 8 nonzero levels of Gamma F).  *chunks = frequency-group
 * chunks per x-mode of the fused kernel (0 when streaming); *nk = number of nonzero leading levels
 * of Gamma F (after pint_set_problem_separable).  Any pointer may be NULL. */
pint_status pint_get_path(pint_plan plan, int32_t* fused, int32_t* chunks, int32_t* nk);

/* Self-check of the current iterate U_m against the scheme it converges to (
 * eqn:BDF P:281-288, CQ eqn:CQ-1 P:946-950): residual_inf = max over all levels and points of
 * |tau^-a sum_j omega_j U^{n-j} + A U^n - F_static_n| (all-at-once form: the v-history is in
 * F_static; in the hoisted DST-x basis),
 * rhs_inf = max |F_static_n|.  At the WR fixed point the ratio is at round-off level; for an
 * unconverged iterate it measures the distance to the sequential BDF-k solution.  Materialises U_m
 * (as pint_get_levels; modal plans and P1-FEM: in the DST modes of both axes, A diagonal).
 * CQ plans: the full history convolution, O(N) per unknown (a check, not a pass).  UNSUPPORTED
 * for CQ on the modal path, semilinear plans, PINT_FLAG_DST_PER_ITER and dense forcing; STATE before
 * the first iteration.  Multi-rank: max over ranks (collective). */
pint_status pint_residual(pint_plan plan, double* residual_inf, double* rhs_inf);

/* Introspection: iteration count m, total kernel launches issued by this plan, device bytes. */
pint_status pint_get_info(pint_plan plan, int64_t* m, int64_t* kernel_launches, int64_t* device_bytes);

pint_status pint_plan_destroy(pint_plan plan);

const char* pint_status_string(pint_status s);
const char* pint_last_error(void);

/* kappa = min(1/ln N, 0.5) (the paper's kappa = O(1/log N) choice for subdiffusion). */
double pint_kappa_log_rule(int64_t N);

#ifdef __cplusplus
}
#endif
#endif /* PINT_H_ */
