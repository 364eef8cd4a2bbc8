// pint.cu — host plan and C ABI (include/pint.h).
//
// Tables (BDFk weights, Table-1 starting corrections, CQ weights, eigenvalues d_p, Gamma,
// twiddles, lambda_q) are built here in 80-bit long double and rounded once to fp64.  This
// file shares no code or tables with oracle/ (test infrastructure); Table 1 is transcribed
// independently below.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pint.h"
#include "kernels.h"

using ld = long double;
using cld = std::complex<long double>;
using namespace pint;

static const ld PI_L = 3.141592653589793238462643383279502884L;

// ------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------
static thread_local std::string g_last_error;
static pint_status fail(pint_status s, const std::string& m) {
  g_last_error = m;
  return s;
}
#define CUDA_TRY(x)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(PINT_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------------------------------
// tables (long double)
// ------------------------------------------------------------------------------------------
// omega_j of delta_k(zeta) = sum_{l=1}^k (1 - zeta)^l / l   (eqn:bdf-gen)
static std::vector<ld> bdf_weights(int k) {
  std::vector<ld> w(k + 1, 0.0L);
  for (int l = 1; l <= k; ++l) {
    ld binom = 1.0L;  // C(l, j)
    for (int j = 0; j <= l; ++j) {
      w[j] += ((j & 1) ? -binom : binom) / (ld)l;
      binom = binom * (ld)(l - j) / (ld)(j + 1);
    }
  }
  return w;
}

// Table 1: a_n^{(k)}, n = 1..k-1, and b_{l,n}^{(k)}; zero for n >= k.
// b^{(5)}_{3,1}: printed +1/720, taken as -1/720 (reading R-Table1).
struct Rat { long num, den; };
static ld table1_a(int k, int n) {
  static const Rat A[7][5] = {
      {}, {},
      {{1, 2}},
      {{11, 12}, {-5, 12}},
      {{31, 24}, {-7, 6}, {3, 8}},
      {{1181, 720}, {-177, 80}, {341, 240}, {-251, 720}},
      {{2837, 1440}, {-2543, 720}, {17, 5}, {-1201, 720}, {95, 288}}};
  if (k < 2 || n < 1 || n > k - 1) return 0.0L;
  return (ld)A[k][n - 1].num / (ld)A[k][n - 1].den;
}
static ld table1_b(int k, int l, int n) {
  // B[k][l][n-1]
  static const Rat B[7][5][5] = {
      {}, {}, {},
      {{}, {{1, 12}, {0, 1}}},
      {{}, {{1, 6}, {-1, 12}, {0, 1}}, {{0, 1}, {0, 1}, {0, 1}}},
      {{}, {{59, 240}, {-29, 120}, {19, 240}, {0, 1}}, {{1, 240}, {-1, 240}, {0, 1}, {0, 1}},
       {{-1, 720}, {0, 1}, {0, 1}, {0, 1}}},
      {{}, {{77, 240}, {-7, 15}, {73, 240}, {-3, 40}, {0, 1}}, {{1, 96}, {-1, 60}, {1, 160}, {0, 1}, {0, 1}},
       {{-1, 360}, {1, 720}, {0, 1}, {0, 1}, {0, 1}}, {{0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}}}};
  if (k < 3 || l < 1 || l > k - 2 || n < 1 || n > k - 1) return 0.0L;
  const Rat r = B[k][l][n - 1];
  if (r.den == 0) return 0.0L;
  return (ld)r.num / (ld)r.den;
}

// CQ weights: power series of delta_k(xi)^alpha by Miller's recurrence
static std::vector<ld> cq_weights(int k, ld alpha, long n) {
  const std::vector<ld> p = bdf_weights(k);
  std::vector<ld> q(n, 0.0L);
  q[0] = powl(p[0], alpha);
  for (long m = 1; m < n; ++m) {
    ld s = 0.0L;
    for (int i = 1; i <= std::min<long>(m, k); ++i) s += ((alpha + 1) * i - (ld)m) * p[i] * q[m - i];
    q[m] = s / ((ld)m * p[0]);
  }
  return q;
}

// ------------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------------
struct pint_plan_s {
  int64_t M, N, mx, my;
  int k, dim, flags, rank, nranks;
  double kappa, tau, alpha, h;  // h = line spacing 1/(L+1)
  pint_allreduce_max_fn allreduce;
  void* actx;
  int64_t q0, Qb, L, NB, ntiles;
  int WB, C, NE;
  int device;
  cudaStream_t stream;
  bool own_stream;
  // device memory
  double2 *A = nullptr, *B = nullptr, *wrap[2] = {nullptr, nullptr};
  double2* src = nullptr;    // [S][ntiles][WB]
  double* coef = nullptr;    // [S][N]
  int* nhi = nullptr;        // [S]
  int S = 0;
  int nmax = 0;               // max_s nhi[s]
  int nk = 0;                 // pruned T-pass: max(k, max sparse nhi)
  int nsparse = 0, ndense = 0;
  int* srclist = nullptr;     // [S]: sparse sources, then dense sources
  double2* chat = nullptr;    // [S][N] DFTs of dense coefficient sequences
  double2* cqhat = nullptr;   // [S][N] CQ split T-pass: DFTs of Gamma h^2/N c_s(n) for every source
  double2* cqwhat = nullptr;  // [N] CQ bootstrap: DFT of Gamma h^2/N times the wrap coefficient of U_0 = v
  double2 *tw = nullptr, *twE = nullptr;
  double *gsf = nullptr, *igs = nullptr, *gsN = nullptr, *wk = nullptr;
  double* cqw = nullptr;      // [N] tau^-a omega_j (CQ plans)
  double2 *dh = nullptr, *dpr = nullptr, *thp = nullptr, *thm = nullptr;
  double2* sig_p = nullptr;
  double* sig_q = nullptr;
  double2 *cq_twi = nullptr, *cq_th = nullptr;   // one-kernel CQ T-pass (cqpass.cuh): pass-A twiddles, theta^n,
  double2* cq_dpr = nullptr;                      // (c_x / N) d'_p
  double cq_gt[32] = {};                                             // kappa^{-N1 t/N}
  double2* phys = nullptr;   // [2][M] physical staging (v, A v)
  double2* wstage = nullptr; // [k][M] staging for window-level reads (lazy)
  unsigned long long* upd = nullptr;
  unsigned long long* updh = nullptr;   // pinned host copy of upd
  char* stage = nullptr;                // pinned staging of the per-problem tables (set_problem)
  size_t stage_cap = 0, stage_off = 0;
  bool upd_queued = false;              // the D2H copy of upd is already on the stream
  // fused heat iteration (fused.cuh): state = X (nk <= 8 levels) + window; no H/W arrays per iteration
  bool dst_iter = false;      // PINT_FLAG_DST_PER_ITER: physical-x arrays, DST-x around every S-pass
  bool half = false;          // PINT_FLAG_REAL_DATA: half-spectrum fused iteration
  bool modal = false;         // PINT_FLAG_MODAL: DST along y too, one warp per (q, j) mode
  bool fem = false;           // PINT_OP_FEM1D_DIRICHLET (modal, mu_j = h^2 K_j / M_j)
  bool fem2d = false;         // PINT_OP_FEM2D_DIRICHLET (modal + streaming, Step 2 by fem2d_solve)
  double *fcx = nullptr, *fcy = nullptr;       // [Qb] cos(q pi h), [L] cos(j pi h)
  double2 *fb = nullptr, *fe = nullptr, *ft = nullptr;   // fem2d_solve: right-hand side, E X, scratch
  unsigned long long* fupd = nullptr;          // [2] fem2d_solve monitors
  int fem_iters = 0;                           // inner iterations of the last fem2d_solve (introspection)
  int NEy = 0;
  double2* twEy = nullptr;    // [NEy] DST-y twiddles
  double* mu = nullptr;       // [my] 4 sin^2(j pi h_y / 2)
  double2* wtmp = nullptr;    // [ntiles][k][WB] modal window -> (q, y) staging
  bool pmon = false;          // fused modal plan, one rank: update monitor on the PHYSICAL window levels
  double2* pwin[2] = {nullptr, nullptr};   // [ntiles][k][WB] window of U_m, line axis in grid space
  unsigned long long* upd_sink = nullptr;  // the finish kernel's (modal-basis) monitor goes here then
  double2* fd = nullptr;      // dense forcing f(t_1..t_N) in the tile layout (pint_set_problem)
  bool full = false;          // full-array update monitor (CQ plans, PINT_FLAG_FULL_UPDATE_NORM)
  double2* ufull = nullptr;   // [ntiles][N][WB]: U_m of every level (tile layout) when `full`
  bool has_fd = false;
  bool fused_ok = false;      // plan-level eligibility (alpha = 1, smem fits, not PINT_FLAG_STREAM)
  bool fused = false;         // active for the current problem (also needs nk <= 8)
  int Cf = 0, Lf = 0, nch = 1, gpc = 1;
  int flanes = 32;            // fused kernel lanes per line (one warp)
  bool ftm = true;            // window partial sums in TMEM
  double2* X[2] = {nullptr, nullptr};   // [Qb][8][Lf]
  int xcur = 0;               // X[xcur] feeds the next iteration; X[1-xcur] produced W_m
  LineConst* lc = nullptr;    // [Qb][N]
  SPassConst* slc = nullptr;  // [Qb][N] line constants of the pair S-pass (streaming path)
  double2* Pp = nullptr;      // [Qb][nch][k][Lf]
  int64_t dev_bytes = 0;
  unsigned long long* prof = nullptr;   // -DPINT_FUSED_PROF builds: phase cycle counters (not owned)
  // semilinear extension (Algorithm 3; newton.cuh): 1D, streaming path
  bool nl = false;
  double nl_eps = 1.0;
  double2 *nlU = nullptr, *nlR = nullptr, *nlC = nullptr, *nlPiv = nullptr, *nlT[2] = {nullptr, nullptr};
  double *nlWt = nullptr, *nlAnl = nullptr;
  std::vector<void*> allocs;
  // state
  bool problem_set = false;
  int stateA = 0;            // 0: A holds H_{m+1} (B holds W_m); 1: A holds U_m (time domain);
                             // 3: U_m read from `ufull` (full-array monitor; A still holds H_{m+1})
  int wcur = 0;              // wrap[wcur] = last-k levels of the current U_m
  int64_t m = 0, launches = 0;
  double last_upd = -1.0;
  int increases = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev, sev;
  double t_ms = 0, s_ms = 0;
  int64_t t_n = 0, s_n = 0;
  // fused iteration replayed as a CUDA graph (memset, fused kernel, [reduce], finish), one per
  // (wcur, xcur) parity; re-captured whenever the kernel arguments differ from the captured ones
  bool graphs = true;
  // slots 4..7: the same with CUDA-event nodes around the fused and finish kernels (timing mode)
  cudaGraphExec_t gexec[8] = {};
  FusedArgs gfa[8];
  FinishArgs gfin[8];
  cudaEvent_t gev[8][4] = {};
  cudaEvent_t* cap_ev = nullptr;   // during a timing capture: the slot's events
  // device-side WR loop (pint_wr_solve on the fused path): a graph with a while-conditional node whose
  // body runs two iterations (both ping-pong parities) each followed by the stopping-rule kernel
  const int* cap_skip = nullptr;   // during its capture: the kernels' early-exit flag (LoopCtl::done)
  LoopCtl* cap_ctl = nullptr;      // during its capture (fused, non-modal-monitor plans): the finish
  unsigned long long cap_hnd = 0;  //   kernel's last block applies the stopping rule
  unsigned int* larrive = nullptr; // its block arrival counter
  GridBar* lbar = nullptr;         // small problems: the whole loop as one cooperative kernel (grid barrier)
  LoopCtl* lctl = nullptr;         // device state of the loop
  LoopCtl* lctl_h = nullptr;       // pinned host copy
  cudaGraphExec_t lexec[4] = {};   // per (wcur, xcur) at loop entry
  FusedArgs lfa[4][2];
  FinishArgs lfin[4][2];
  int64_t llaunch[4] = {};         // kernels per iteration of the loop body (incl. the ctl kernel)
  int gpending = -1;          // slot whose event nodes ran last and are not yet accumulated
  int64_t glaunch = 0;        // kernels per graph replay
};



template <class T>
static pint_status dalloc(pint_plan p, T** ptr, size_t count);

template <class T>
static pint_status dalloc(pint_plan p, T** ptr, size_t count) {
  void* q = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) return fail(PINT_ERR_ALLOC, "cudaMalloc(" + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
  p->allocs.push_back(q);
  p->dev_bytes += (int64_t)bytes;
  *ptr = (T*)q;
  // zero-filled: pad slots (rows y >= L of the window / monitor buffers, tile tails) are never written by
  // the kernels but some are read (the fully modal plans' physical-window monitor took differences over
  // them: an uninitialised allocation left a constant, run-dependent update floor, e.g. 2.7e-10)
  e = cudaMemsetAsync(q, 0, bytes, p->stream);
  if (e != cudaSuccess) return fail(PINT_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  return PINT_OK;
}
#define TRY(x)                        \
  do {                                \
    pint_status s_ = (x);             \
    if (s_ != PINT_OK) return s_;     \
  } while (0)

template <class T>
static pint_status h2d(pint_plan p, T* dst, const std::vector<T>& v) {
  CUDA_TRY(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));   // host vector goes out of scope
  return PINT_OK;
}

static double2 d2(cld z) { return make_double2((double)z.real(), (double)z.imag()); }

// per-problem tables: copied through a plan-owned pinned staging buffer without a synchronisation
// per table (set_problem synchronises once at its end, before the buffer can be reused)
static pint_status stage_reserve(pint_plan p, size_t bytes) {
  if (p->stage_off) CUDA_TRY(cudaStreamSynchronize(p->stream));   // an earlier call returned early
  p->stage_off = 0;
  if (bytes <= p->stage_cap) return PINT_OK;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (p->stage) CUDA_TRY(cudaFreeHost(p->stage));
  p->stage = nullptr;
  p->stage_cap = 0;
  CUDA_TRY(cudaHostAlloc((void**)&p->stage, bytes, cudaHostAllocDefault));
  p->stage_cap = bytes;
  return PINT_OK;
}
template <class T>
static pint_status h2d_async(pint_plan p, T* dst, const std::vector<T>& v) {
  const size_t bytes = v.size() * sizeof(T);
  const size_t off = (p->stage_off + 15) & ~(size_t)15;
  if (off + bytes > p->stage_cap) return h2d(p, dst, v);          // (not reserved: synchronous copy)
  std::memcpy(p->stage + off, v.data(), bytes);
  CUDA_TRY(cudaMemcpyAsync(dst, p->stage + off, bytes, cudaMemcpyHostToDevice, p->stream));
  p->stage_off = off + bytes;
  return PINT_OK;
}

// in-place radix-2 DFT in long double (host plan tables): x_p <- sum_n x_n e^{sign 2 pi i n p / N}
static void fft_ld(std::vector<cld>& x, int sign) {
  const size_t N = x.size();
  for (size_t i = 1, j = 0; i < N; ++i) {   // bit reversal
    size_t bit = N >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(x[i], x[j]);
  }
  for (size_t len = 2; len <= N; len <<= 1) {
    for (size_t i = 0; i < N; i += len)
      for (size_t m = 0; m < len / 2; ++m) {
        const long double ang = (long double)sign * 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)len;
        const cld w(cosl(ang), sinl(ang));
        const cld u = x[i + m], v = x[i + m + len / 2] * w;
        x[i + m] = u + v;
        x[i + m + len / 2] = u - v;
      }
  }
}

static void free_plan(pint_plan p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  if (p->prof) {   // profiling builds: print the phase cycle split of the fused kernel
    unsigned long long h[64];
    cudaMemcpy(h, p->prof, sizeof(h), cudaMemcpyDeviceToHost);
    if (h[44])
      fprintf(stderr, "[pint prof] loop kernel ns per block-iteration: fused %.0f sync1 %.0f finish %.0f sync2 %.0f\n",
              (double)h[40] / h[44], (double)h[41] / h[44], (double)h[42] / h[44], (double)h[43] / h[44]);
    const double tot = (double)(h[0] + h[1] + h[2] + h[3]) + 1e-30;
    fprintf(stderr, "[pint prof] fused phases (warp-cycles share): solve %.3f wait1 %.3f rows %.3f wait2 %.3f\n",
            h[0] / tot, h[1] / tot, h[2] / tot, h[3] / tot);
    if (h[48 + 8]) {
      unsigned long long g[9];
      cudaMemcpy(g, p->prof + 48, sizeof(g), cudaMemcpyDeviceToHost);
      double t = 0; for (int j = 0; j < 9; ++j) t += (double)g[j];
      fprintf(stderr, "[pint prof] solve sub-phases (share): fwd0 %.3f scan1 %.3f fwd1 %.3f bwd0 %.3f scan2 %.3f bwd1 %.3f corr %.3f store %.3f fastP %.3f; cycles per warp-solve %.0f\n",
              g[0] / t, g[1] / t, g[2] / t, g[3] / t, g[4] / t, g[5] / t, g[6] / t, g[7] / t, g[8] / t, t / (double)h[57]);
    }
    for (int w = 0; w < 8; ++w)
      fprintf(stderr, "[pint prof] warp %d: solve %.3e wait1 %.3e rows %.3e wait2 %.3e\n", w, (double)h[4 + 4 * w],
              (double)h[5 + 4 * w], (double)h[6 + 4 * w], (double)h[7 + 4 * w]);
  }
  for (void* q : p->allocs) cudaFree(q);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  for (auto& e : p->tev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (auto& e : p->sev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (cudaGraphExec_t g : p->gexec) if (g) cudaGraphExecDestroy(g);
  for (cudaGraphExec_t g : p->lexec) if (g) cudaGraphExecDestroy(g);
  if (p->lctl_h) cudaFreeHost(p->lctl_h);
  for (auto& ev : p->gev) for (cudaEvent_t e : ev) if (e) cudaEventDestroy(e);
  if (p->updh) cudaFreeHost(p->updh);
  if (p->stage) cudaFreeHost(p->stage);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

extern "C" pint_status pint_partition(int64_t mx, int32_t rank, int32_t nranks, int64_t* q_begin, int64_t* q_end);

static bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

extern "C" pint_status pint_plan_create(int64_t M, int64_t N, int32_t k, double kappa, double tau,
                                        const pint_operator* op, const pint_options* opt, pint_plan* out) {
  if (!out) return fail(PINT_ERR_ARG, "out must not be NULL");
  *out = nullptr;
  if (!op) return fail(PINT_ERR_ARG, "op must not be NULL");
  if (k < 1 || k > 6) return fail(PINT_ERR_ARG, "k must be in 1..6 (BDFk, PAPER.md:278), got " + std::to_string(k));
  if (!(kappa > 0.0 && kappa < 1.0)) return fail(PINT_ERR_ARG, "kappa must be in (0,1)");
  if (!(tau > 0.0) || !std::isfinite(tau)) return fail(PINT_ERR_ARG, "tau must be > 0");
  if (N < k + 1) return fail(PINT_ERR_ARG, "N must be >= k+1 (DESIGN.md reading R-Nk)");
  const double alpha = opt ? opt->alpha : 1.0;
  if (!(alpha > 0.0 && alpha <= 1.0)) return fail(PINT_ERR_ARG, "alpha must be in (0,1]");
  if (op->kind != PINT_OP_FD1D_DIRICHLET && op->kind != PINT_OP_FD2D_DIRICHLET && op->kind != PINT_OP_FEM1D_DIRICHLET &&
      op->kind != PINT_OP_FEM2D_DIRICHLET)
    return fail(PINT_ERR_ARG, "op->kind must be PINT_OP_FD1D_DIRICHLET, PINT_OP_FD2D_DIRICHLET, PINT_OP_FEM1D_DIRICHLET "
                              "or PINT_OP_FEM2D_DIRICHLET");
  if (op->mx < 1 || op->my < 1) return fail(PINT_ERR_ARG, "op->mx, op->my must be >= 1");
  const bool fem = op->kind == PINT_OP_FEM1D_DIRICHLET;
  const bool fem2d = op->kind == PINT_OP_FEM2D_DIRICHLET;
  const bool two_d = op->kind == PINT_OP_FD2D_DIRICHLET || fem2d;
  if (fem2d && op->mx != op->my) return fail(PINT_ERR_UNSUPPORTED, "PINT_OP_FEM2D_DIRICHLET needs mx == my (uniform triangulation, h_x = h_y)");
  if ((op->kind == PINT_OP_FD1D_DIRICHLET || fem) && op->my != 1) return fail(PINT_ERR_ARG, "1D operator needs my == 1");
  if (op->mx * op->my != M) return fail(PINT_ERR_ARG, "M must equal mx*my");
  const int rank = opt ? opt->rank : 0, nranks = opt ? opt->nranks : 1;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PINT_ERR_ARG, "need 0 <= rank < nranks");
  if (nranks > 1 && op->kind != PINT_OP_FD2D_DIRICHLET)
    return fail(fem2d ? PINT_ERR_UNSUPPORTED : PINT_ERR_ARG,
                fem2d ? "2D P1-FEM couples the x-modes (mass matrix): one rank only"
                      : "1D operators do not shard (replicas only): nranks must be 1");
  if (nranks > op->mx) return fail(PINT_ERR_ARG, "nranks must be <= mx");
  if (opt && (opt->flags & PINT_FLAG_DST_PER_ITER) && (op->kind != PINT_OP_FD2D_DIRICHLET || nranks != 1))
    return fail(PINT_ERR_ARG, "PINT_FLAG_DST_PER_ITER needs a 2D operator on one rank");
  // P1-FEM runs modal (1D: diagonal; 2D: the mass matrix's M_sym part is, fem2d.cuh), 2D FEM on the
  // streaming path (its Step 2 is the fem2d fixed-point solve)
  const int32_t flags = (opt ? opt->flags : 0) | ((fem || fem2d) ? PINT_FLAG_MODAL : 0) | (fem2d ? PINT_FLAG_STREAM : 0);
  if (flags & PINT_FLAG_MODAL) {
    const int64_t Lm = two_d ? op->my : op->mx;
    if (flags & PINT_FLAG_DST_PER_ITER) return fail(PINT_ERR_ARG, "PINT_FLAG_MODAL excludes PINT_FLAG_DST_PER_ITER");
    if (!is_pow2(2 * (Lm + 1)) || 2 * (Lm + 1) < 16 || 2 * (Lm + 1) > 4096)
      return fail(PINT_ERR_UNSUPPORTED, "PINT_FLAG_MODAL needs 2(L+1) a power of two in [16, 4096] (L = my in 2D, mx in 1D)");
  }
  if (nranks > 1 && !(opt && opt->allreduce_max)) return fail(PINT_ERR_ARG, "nranks > 1 needs allreduce_max");
  if (!is_pow2(N) || N < 16 || N > 4096) return fail(PINT_ERR_UNSUPPORTED, "N must be a power of two in [16, 4096]");
  const int dim = two_d ? 2 : 1;
  const int64_t L = dim == 1 ? op->mx : op->my;
  if (L > 1024) return fail(PINT_ERR_UNSUPPORTED, "line length (1D: mx, 2D: my) must be <= 1024");
  int NE = 0;
  if (dim == 2) {
    NE = (int)(2 * (op->mx + 1));
    if (!is_pow2(NE) || NE < 16 || NE > 4096) return fail(PINT_ERR_UNSUPPORTED, "2D needs 2(mx+1) a power of two in [16, 4096]");
  }

  pint_plan p = new pint_plan_s();
  p->M = M; p->N = N; p->mx = op->mx; p->my = op->my; p->k = k; p->dim = dim;
  p->flags = flags; p->rank = rank; p->nranks = nranks; p->fem = fem; p->fem2d = fem2d;
  p->kappa = kappa; p->tau = tau; p->alpha = alpha;
  p->allreduce = opt ? opt->allreduce_max : nullptr; p->actx = opt ? opt->allreduce_ctx : nullptr;
  p->L = L; p->h = 1.0 / (double)(L + 1); p->NE = NE;
  if (dim == 2) {
    int64_t qb = 0, qe = 0;
    pint_partition(op->mx, rank, nranks, &qb, &qe);
    p->q0 = qb;
    p->Qb = qe - qb;
  } else {
    p->q0 = 0; p->Qb = 1;
  }
  p->WB = (int)(TILE / N);
  p->NB = (L + p->WB - 1) / p->WB;
  p->ntiles = p->Qb * p->NB;
  int C = 1;
  while (32 * C < L) C *= 2;
  p->C = C;
  p->device = opt ? opt->device : 0;

  auto bail = [&](pint_status s) { free_plan(p); return s; };
  cudaError_t ce = cudaSetDevice(p->device);
  if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce)); }
  if (opt && opt->stream) {
    p->stream = (cudaStream_t)opt->stream;
    p->own_stream = false;
  } else {
    ce = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(ce)); }
    p->own_stream = true;
  }
  // graph replay of the fused iteration (PINT_NO_GRAPH=1: eager launches; the legacy stream cannot capture)
  p->graphs = getenv("PINT_NO_GRAPH") == nullptr && p->stream != cudaStreamLegacy;

  const size_t arr = (size_t)p->ntiles * TILE;
  pint_status st;
  if ((st = dalloc(p, &p->A, arr)) != PINT_OK) return bail(st);   // space-time buffers (H / W, U staging)
  if ((st = dalloc(p, &p->B, arr)) != PINT_OK) return bail(st);
  for (int i = 0; i < 2; ++i)
    if ((st = dalloc(p, &p->wrap[i], (size_t)p->ntiles * k * p->WB)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->tw, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->gsf, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->igs, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->gsN, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->wk, k + 1)) != PINT_OK) return bail(st);
  if (alpha != 1.0 && (st = dalloc(p, &p->cqw, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->dh, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->dpr, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->thp, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->thm, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->sig_p, N)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->sig_q, p->Qb)) != PINT_OK) return bail(st);
  if ((st = dalloc(p, &p->upd, 1)) != PINT_OK) return bail(st);
  ce = cudaHostAlloc((void**)&p->updh, sizeof(unsigned long long), cudaHostAllocDefault);
  if (ce != cudaSuccess) { p->updh = nullptr; return bail(fail(PINT_ERR_ALLOC, std::string("cudaHostAlloc: ") + cudaGetErrorString(ce))); }
  if ((st = dalloc(p, &p->phys, 2 * (size_t)M)) != PINT_OK) return bail(st);
  if (dim == 2 && (st = dalloc(p, &p->twE, NE)) != PINT_OK) return bail(st);
  // fused heat iteration: one warp per line (32 lanes x Cf rows), window sums in TMEM; 8 lines in smem
  {
    p->flanes = 32;
    int Cf = 1;
    while (p->flanes * Cf < L) Cf *= 2;
    p->Cf = Cf;
    p->Lf = p->flanes * Cf;
    p->ftm = true;
  }
  const size_t fsmem = fused_smem_bytes(p->flanes, p->Cf, k, p->ftm);
  p->dst_iter = (p->flags & PINT_FLAG_DST_PER_ITER) != 0;
  // full-array update monitor: the paper's stopping rule; always for CQ plans,
  // whose kappa-wrap reads every level of U_{m-1}
  p->full = alpha != 1.0 || (p->flags & PINT_FLAG_FULL_UPDATE_NORM) != 0;
  if (p->full && (st = dalloc(p, &p->ufull, arr)) != PINT_OK) return bail(st);
  p->fused_ok = alpha == 1.0 && !(p->flags & (PINT_FLAG_STREAM | PINT_FLAG_DST_PER_ITER)) && !p->full &&
                fsmem <= 232448u - 64u;
  p->modal = (p->flags & PINT_FLAG_MODAL) != 0;
  if (p->modal) {
    p->Lf = (int)(p->NB * p->WB);    // X / partials indexed by the y-mode j < my
    p->NEy = (int)(2 * (L + 1));
  }
  if (p->modal) {   // DST along the line axis (fused modal kernel, or division pass of the streaming path)
    if ((st = dalloc(p, &p->twEy, p->NEy)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->mu, (size_t)L)) != PINT_OK) return bail(st);
  }
  if (fem2d) {      // 2D P1-FEM Step 2 (fem2d.cuh): mode cosines, fixed-point buffers
    std::vector<double> cx(p->Qb), cy(L);
    for (int64_t q = 0; q < p->Qb; ++q) cx[q] = (double)cosl((ld)(p->q0 + q + 1) * PI_L / (ld)(op->mx + 1));
    for (int64_t j = 0; j < L; ++j) cy[j] = (double)cosl((ld)(j + 1) * PI_L / (ld)(L + 1));
    if ((st = dalloc(p, &p->fcx, p->Qb)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->fcy, (size_t)L)) != PINT_OK) return bail(st);
    if ((st = h2d(p, p->fcx, cx)) != PINT_OK) return bail(st);
    if ((st = h2d(p, p->fcy, cy)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->fb, arr)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->fe, arr)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->ft, arr)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->fupd, 2)) != PINT_OK) return bail(st);
  }
  if (p->fused_ok && p->modal) {
    // window monitor with the line axis in grid space (DST-y back; reading R-norm2D): the orthonormal
    // DSTs scale the modal coefficients of a smooth field by up to sqrt(M) against the grid values, so
    // a modal-basis max-norm sits ~sqrt(M) above the grid update (its round-off floor 1.7e-12 at C4)
    p->pmon = nranks == 1;
    if (p->pmon) {
      for (int i = 0; i < 2; ++i)
        if ((st = dalloc(p, &p->pwin[i], (size_t)p->ntiles * k * p->WB)) != PINT_OK) return bail(st);
      if ((st = dalloc(p, &p->wtmp, (size_t)p->ntiles * k * p->WB)) != PINT_OK) return bail(st);
      if ((st = dalloc(p, &p->upd_sink, 1)) != PINT_OK) return bail(st);
    }
    p->half = (p->flags & PINT_FLAG_REAL_DATA) != 0;
    p->nch = 1;
    p->gpc = (int)(N / 8);
    for (int i = 0; i < 2; ++i)
      if ((st = dalloc(p, &p->X[i], (size_t)p->Qb * 8 * p->Lf)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->Pp, (size_t)p->Qb * k * p->Lf)) != PINT_OK) return bail(st);
    for (int i = 0; i < 2; ++i) {
      ce = cudaMemsetAsync(p->X[i], 0, (size_t)p->Qb * 8 * p->Lf * sizeof(double2), p->stream);
      if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(ce)); }
    }
  } else if (p->fused_ok) {
    const int per = std::max(fused_ctas_per_sm(p->flanes, p->Cf, k, p->ftm), 1);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
    p->half = (p->flags & PINT_FLAG_REAL_DATA) != 0 && p->ftm;   // the half-spectrum kernel keeps its sums in TMEM
    const long slots = (long)nsm * per, NG = p->half ? N / 16 + 1 : N / 8;
    // chunks of frequency groups per x-mode: smallest power of two giving >= 90% wave efficiency
    long best = 1;
    double beff = 0.0;
    for (long c = 1; c <= NG; c *= 2) {
      const double waves = (double)(p->Qb * c) / (double)slots;
      const double eff = waves / std::ceil(waves);
      if (eff > beff + 1e-9) { beff = eff; best = c; }
      if (eff >= 0.9) { best = c; break; }
    }
    p->nch = (int)best;
    p->gpc = (int)((NG + best - 1) / best);
    for (int i = 0; i < 2; ++i)
      if ((st = dalloc(p, &p->X[i], (size_t)p->Qb * 8 * p->Lf)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->lc, (size_t)p->Qb * N)) != PINT_OK) return bail(st);
    if ((st = dalloc(p, &p->Pp, (size_t)p->Qb * p->nch * k * p->Lf)) != PINT_OK) return bail(st);
    for (int i = 0; i < 2; ++i) {
      ce = cudaMemsetAsync(p->X[i], 0, (size_t)p->Qb * 8 * p->Lf * sizeof(double2), p->stream);
      if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(ce)); }
    }
  }
  ce = cudaMemsetAsync(p->A, 0, arr * sizeof(double2), p->stream);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(p->B, 0, arr * sizeof(double2), p->stream);
  if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(ce)); }

  // ---- tables ----
  const ld kap = kappa, taul = tau, al = alpha, hl = 1.0L / (ld)(L + 1), Nl = (ld)N;
  const ld ta = powl(taul, -al);                      // tau^{-alpha}
  std::vector<ld> w = (alpha == 1.0) ? bdf_weights(k) : cq_weights(k, al, N + 1);
  if (alpha == 1.0) w.resize(N + 1, 0.0L);
  std::vector<double2> tw(N), thp(N), thm(N), dh(N), dpr(N), sigp(N);
  std::vector<cld> dprl(N);
  std::vector<double> gsf(N), igs(N), gsN(N), wk(k + 1), sigq(p->Qb);
  for (int64_t n = 0; n < N; ++n) {
    const ld ang = 2.0L * PI_L * (ld)n / Nl;
    tw[n] = make_double2((double)cosl(ang), (double)-sinl(ang));
    const ld g = powl(kap, (ld)n / Nl);                // Gamma_kappa = diag(kappa^{(n-1)/N}), 1-based n
    gsf[n] = (double)(g * hl * hl / Nl);
    igs[n] = (double)(1.0L / g);
    gsN[n] = (double)(g / Nl);
    const ld th = PI_L * (ld)n / Nl;                   // theta^n = e^{i pi n/N}
    thp[n] = d2(cld(cosl(th), sinl(th)) / Nl);
    thm[n] = d2(cld(cosl(th), -sinl(th)) * (-(hl * hl) * ta / (2.0L * Nl)));
  }
  for (int j = 0; j <= k; ++j) wk[j] = (double)(kap / taul * w[j]);
  // eigenvalues: d_p = sum_j omega_j kappa^{j/N} e^{-2 pi i j p/N}  (Lemma 2.3 / 3.2; CQ:
  // truncated column, reading R-CQeig); d'_p: same for C(-kappa) with (-kappa)^{j/N} = kappa^{j/N} theta^j
  const int64_t jmax = (alpha == 1.0) ? k : N - 1;
  std::vector<ld> cj(jmax + 1);
  for (int64_t j = 0; j <= jmax; ++j) cj[j] = w[j] * powl(kap, (ld)j / Nl);
  std::vector<cld> e2(2 * N);                         // e^{-i pi m/N}, m < 2N
  for (int64_t m = 0; m < 2 * N; ++m) e2[m] = cld(cosl(PI_L * (ld)m / Nl), -sinl(PI_L * (ld)m / Nl));
  for (int64_t pp = 0; pp < N; ++pp) {
    cld d = 0.0L, dq = 0.0L;
    for (int64_t j = 0; j <= jmax; ++j) {
      d += cj[j] * e2[(2 * j * pp) % (2 * N)];
      dq += cj[j] * e2[(j * (2 * pp - 1) % (2 * N) + 2 * N) % (2 * N)];
    }
    sigp[pp] = d2(d * ta * hl * hl);
    dh[pp] = d2(d * (hl * hl) * ta / 2.0L);
    dpr[pp] = d2(dq);
    dprl[pp] = dq;
  }
  for (int64_t ql = 0; ql < p->Qb; ++ql) {
    if (dim == 1) { sigq[ql] = 0.0; continue; }
    const ld hx = 1.0L / (ld)(p->mx + 1);
    const ld sn = sinl((ld)(p->q0 + ql + 1) * PI_L * hx / 2.0L);
    sigq[ql] = (double)(hl * hl * 4.0L / (hx * hx) * sn * sn);   // h_y^2 lambda_q
  }
  if ((st = h2d(p, p->tw, tw)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->gsf, gsf)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->igs, igs)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->gsN, gsN)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->wk, wk)) != PINT_OK) return bail(st);
  if (alpha != 1.0) {   // tau^-a omega_j, j < N (CQ weights; pint_residual's history convolution)
    std::vector<double> cqw(N);
    for (int64_t j = 0; j < N; ++j) cqw[j] = (double)(ta * w[j]);
    if ((st = h2d(p, p->cqw, cqw)) != PINT_OK) return bail(st);
  }
  if ((st = h2d(p, p->dh, dh)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->dpr, dpr)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->thp, thp)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->thm, thm)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->sig_p, sigp)) != PINT_OK) return bail(st);
  if ((st = h2d(p, p->sig_q, sigq)) != PINT_OK) return bail(st);
  if (alpha != 1.0 && (N == 1024 || N == 256)) {
    // one-kernel CQ T-pass (cqpass.cuh): 4-step transforms N = N1 x N1; pass-A tables [i][k2] with the
    // Theta / N and c_x Theta^{-1} factors of the skew-circulant wrap folded in (per-thread part theta^i)
    const int64_t N1 = N == 1024 ? 32 : 16;
    // all four transforms run as inverse 4-step transforms (forward = conj . inverse . conj): one
    // twiddle table w^{+i k2} [i][k2], and theta^n for the skew-circulant rotations
    std::vector<double2> twi(N), thn(N), dps(N);
    for (int64_t i = 0; i < N1; ++i)
      for (int64_t k2 = 0; k2 < N1; ++k2) {
        const ld a = 2.0L * PI_L * (ld)((i * k2) % N) / Nl;
        twi[i * N1 + k2] = d2(cld(cosl(a), sinl(a)));                 // w^{+i k2}
      }
    for (int64_t n = 0; n < N; ++n) thn[n] = d2(cld(cosl(PI_L * (ld)n / Nl), sinl(PI_L * (ld)n / Nl)));
    for (int64_t t = 0; t < N1; ++t) p->cq_gt[t] = (double)powl(kap, -(ld)(N1 * t) / Nl);
    const ld cx = -(hl * hl) * ta / (2.0L * Nl);                     // the chain is linear: 1/N and c_x on D'
    for (int64_t pp = 0; pp < N; ++pp) dps[pp] = d2(dprl[pp] * (cx / Nl));
    double2** tabs[3] = {&p->cq_twi, &p->cq_th, &p->cq_dpr};
    const std::vector<double2>* vals[3] = {&twi, &thn, &dps};
    for (int t = 0; t < 3; ++t) {
      if ((st = dalloc(p, tabs[t], N)) != PINT_OK) return bail(st);
      if ((st = h2d(p, *tabs[t], *vals[t])) != PINT_OK) return bail(st);
    }
  }
  if (p->C >= 4 && p->WB >= 2) {   // the pair S-pass (C/2 rows per lane) reads its line constants
    if ((st = dalloc(p, &p->slc, (size_t)p->Qb * N)) != PINT_OK) return bail(st);
    ce = launch_spass_const(p->slc, p->sig_p, p->sig_q, N, p->Qb, p->C / 2, (int)L, p->stream);
    if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("spass_const: ") + cudaGetErrorString(ce)); }
  }
  if (p->fused_ok && !p->modal) {
    ce = launch_line_const(p->lc, p->sig_p, p->sig_q, N, p->Qb, p->Cf, fused_rows_per_subchain(p->flanes, p->Cf), (int)L,
                           p->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(p->stream);
    if (ce != cudaSuccess) { free_plan(p); return fail(PINT_ERR_CUDA, std::string("line_const: ") + cudaGetErrorString(ce)); }
  }
  if (dim == 2) {
    std::vector<double2> twE(NE);
    for (int m = 0; m < NE; ++m) {
      const ld ang = 2.0L * PI_L * (ld)m / (ld)NE;
      twE[m] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
    if ((st = h2d(p, p->twE, twE)) != PINT_OK) return bail(st);
  }
  if (p->modal) {
    std::vector<double2> twEy(p->NEy);
    for (int m = 0; m < p->NEy; ++m) {
      const ld ang = 2.0L * PI_L * (ld)m / (ld)p->NEy;
      twEy[m] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
    if ((st = h2d(p, p->twEy, twEy)) != PINT_OK) return bail(st);
    // h^2 lambda_j of the line operator: FD 4 s^2 (tridiag(-1,2,-1)); P1 FEM K_j / M_j =
    // 4 s^2 / (1 - (2/3) s^2), s = sin(j pi h / 2) (stiffness and mass share the sine modes)
    std::vector<double> mu(L);
    for (int64_t jj = 0; jj < L; ++jj) {
      const ld sn = sinl((ld)(jj + 1) * PI_L / (2.0L * (ld)(L + 1)));
      mu[jj] = (double)(fem ? 4.0L * sn * sn / (1.0L - 2.0L * sn * sn / 3.0L) : 4.0L * sn * sn);
    }
    if ((st = h2d(p, p->mu, mu)) != PINT_OK) return bail(st);
  }
  *out = p;
  return PINT_OK;
}

// ------------------------------------------------------------------------------------------
// launches
// ------------------------------------------------------------------------------------------
static TPassArgs targs(pint_plan p) {
  TPassArgs a{};
  a.src = p->src; a.coef = p->coef; a.nhi = p->nhi; a.S = p->S;
  a.vsrc = p->src;   // source 0 is v
  a.tw = p->tw; a.gsf = p->gsf; a.igs = p->igs; a.gsN = p->gsN; a.wk = p->wk; a.k = p->k;
  a.dh = p->dh; a.dpr = p->dpr; a.thp = p->thp; a.thm = p->thm; a.gsfq = p->gsf;
  a.upd = p->upd;
  a.nmax = p->nmax;
  a.nk = p->nk;
  a.nsparse = p->nsparse; a.spar = p->srclist;
  a.ndense = p->ndense; a.dsrc = p->srclist ? p->srclist + p->nsparse : nullptr; a.chat = p->chat;
  a.ufull = p->full ? p->ufull : nullptr;
  a.prefetch = 1;
  if (p->has_fd) {   // dense forcing: F_static += f(t_n) at every level (streaming path, unpruned)
    a.fdense = p->fd;
    a.nmax = (int)p->N;
    a.nk = (int)p->N;
  }
  return a;
}

static pint_status tpass(pint_plan p, int mode_in, int mode_out, const double2* in, double2* out,
                         const double2* wold, double2* wnew, bool timed) {
  TPassArgs a = targs(p);
  a.in = in; a.out = out; a.wrap_old = wold; a.wrap_new = wnew;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed && p->timing) {
    CUDA_TRY(cudaEventCreate(&e0)); CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, p->stream));
  }
  const bool pruned = mode_in == IN_FREQ && mode_out == OUT_H && p->alpha == 1.0 && p->N >= 256 &&
                      p->nk <= 16 && p->k <= 8 && !(p->flags & PINT_FLAG_FULL_FFT) && !p->has_fd && !p->full;
  // CQ iteration: one kernel (cqpass.cuh) for N in {256, 1024}, else two kernels of two transforms each
  // (tpass.cuh "CQ T-pass split"); dense right-hand sides keep the four-transform tpass_kernel
  const bool split = p->alpha != 1.0 && mode_in == IN_FREQ && mode_out == OUT_H && !a.fdense && in != out;
  if (pruned) CUDA_TRY(launch_tpass_pruned((int)p->N, a, p->ntiles, p->stream));
  else if (split && p->cq_twi && p->full) {
    // one kernel: W -> U_m (full monitor) -> four on-chip transforms -> H (cqpass.cuh)
    CQArgs c{};
    c.in = in; c.out = out; c.ufull = p->ufull; c.wrap_new = wnew; c.upd = p->upd;
    c.tw = p->cq_twi; c.th = p->cq_th; c.dpr = p->cq_dpr; c.dh = p->dh; c.chat = p->cqhat; c.src = p->src;
    c.igs = p->igs;
    for (int t = 0; t < 32; ++t) c.gt[t] = t < (p->N == 1024 ? 32 : 16) ? p->cq_gt[t] : 0.0;
    c.S = p->S; c.k = p->k; c.ntiles = p->ntiles;
    CUDA_TRY(launch_tpass_cq_fused((int)p->N, c, p->stream));
  } else if (split) {
    CUDA_TRY(launch_tpass_cq_split((int)p->N, 0, a, p->ntiles, p->stream));      // W -> Z (into out)
    TPassArgs b = a;
    b.in = out; b.vsrc = in; b.chat = p->cqhat;                                   // Z, W -> H
    CUDA_TRY(launch_tpass_cq_split((int)p->N, 1, b, p->ntiles, p->stream));
    ++p->launches;
  } else CUDA_TRY(launch_tpass((int)p->N, mode_in, mode_out, p->alpha != 1.0, a, p->ntiles, p->stream));
  ++p->launches;
  if (e0) { CUDA_TRY(cudaEventRecord(e1, p->stream)); p->tev.push_back({e0, e1}); }
  return PINT_OK;
}

static pint_status fem2d_solve(pint_plan p, const double2* H, double2* X, long levels, bool av);

static pint_status spass(pint_plan p, const double2* in, double2* out) {
  if (p->fem2d) {   // 2D P1-FEM: (s_p M + K) W = M H by the DST-preconditioned fixed point (fem2d.cuh)
    cudaEvent_t m0 = nullptr, m1 = nullptr;
    if (p->timing) {
      CUDA_TRY(cudaEventCreate(&m0)); CUDA_TRY(cudaEventCreate(&m1));
      CUDA_TRY(cudaEventRecord(m0, p->stream));
    }
    TRY(fem2d_solve(p, in, out, p->N, false));
    if (m0) { CUDA_TRY(cudaEventRecord(m1, p->stream)); p->sev.push_back({m0, m1}); }
    return PINT_OK;
  }
  SPassArgs a{};
  a.in = in; a.out = out; a.sig_p = p->sig_p; a.sig_q = p->sig_q;
  a.N = p->N; a.NB = p->NB; a.WB = p->WB; a.L = (int)p->L; a.lc = p->slc;
  if (p->modal) {   // streaming modal path: Step 2 is W = H / (sigma_p + sigma_q + mu_j), elementwise
    cudaEvent_t m0 = nullptr, m1 = nullptr;
    if (p->timing) {
      CUDA_TRY(cudaEventCreate(&m0)); CUDA_TRY(cudaEventCreate(&m1));
      CUDA_TRY(cudaEventRecord(m0, p->stream));
    }
    CUDA_TRY(launch_modal_div(a, p->mu, p->Qb, p->stream));
    ++p->launches;
    if (m0) { CUDA_TRY(cudaEventRecord(m1, p->stream)); p->sev.push_back({m0, m1}); }
    return PINT_OK;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->timing) {
    CUDA_TRY(cudaEventCreate(&e0)); CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, p->stream));
  }
  CUDA_TRY(launch_spass(p->C, a, p->Qb, p->stream));
  ++p->launches;
  if (e0) { CUDA_TRY(cudaEventRecord(e1, p->stream)); p->sev.push_back({e0, e1}); }
  return PINT_OK;
}

static FusedArgs fargs(pint_plan p, const double2* X) {
  FusedArgs a{};
  a.X = X; a.lc = p->lc; a.tw = p->tw; a.src = p->src;
  a.dsrc = p->srclist ? p->srclist + p->nsparse : nullptr; a.chat = p->chat; a.ndense = p->ndense;
  a.P = p->Pp; a.W = p->B;
  a.skip = p->cap_skip;
  a.N = p->N; a.Qb = p->Qb; a.L = (int)p->L; a.Lf = p->Lf; a.Lpad = (int)(p->NB * p->WB); a.WB = p->WB;
  a.NB = (int)p->NB; a.k = p->k; a.nk = p->nk; a.nch = p->nch; a.gpc = p->gpc;
  a.half = p->half ? 1 : 0;
  a.mu = p->mu; a.sig_p = p->sig_p; a.sig_q = p->sig_q;
  // X staged in shared memory when it fits next to the lines (TMEM variant: no window sums in smem)
  a.xs = (p->ftm &&
          fused_smem_bytes(p->flanes, p->Cf, p->k, true) + (size_t)p->nk * p->Lf * sizeof(double2) <= 232448u - 64u) ? 1 : 0;
#ifdef PINT_FUSED_PROF
  static unsigned long long* prof = nullptr;
  if (!prof) { cudaMalloc(&prof, 256 * 8); cudaMemset(prof, 0, 256 * 8); }
  a.prof = prof;
  p->prof = prof;
#endif
  return a;
}

static pint_status fused_pass(pint_plan p, const double2* X, bool store_w, bool reset_upd = false) {
  FusedArgs a = fargs(p, X);
  if (reset_upd) a.upd_reset = p->upd;
  if (store_w) {   // materialising variant: shared-memory layout without X, every frequency group
    a.xs = 0;
    a.half = 0;
    a.nch = 1;
    a.gpc = (int)(p->N / 8);
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->cap_ev && !store_w) {                 // graph capture: the slot's own event nodes
    e0 = p->cap_ev[0]; e1 = p->cap_ev[1];
    CUDA_TRY(cudaEventRecordWithFlags(e0, p->stream, cudaEventRecordExternal));
  } else if (p->timing && !store_w) {
    CUDA_TRY(cudaEventCreate(&e0)); CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, p->stream));
  }
  if (p->modal) CUDA_TRY(launch_modal(store_w, a, p->stream));
  else CUDA_TRY(launch_fused(p->flanes, p->Cf, store_w, p->ftm, a, p->stream));
  ++p->launches;
  if (e0) {
    CUDA_TRY(cudaEventRecordWithFlags(e1, p->stream, p->cap_ev ? cudaEventRecordExternal : cudaEventRecordDefault));
    if (!p->cap_ev) p->sev.push_back({e0, e1});
  }
  return PINT_OK;
}

// window of U (mode: FIN_PARTIALS from the fused partial sums, FIN_FROM_WRAP / FIN_FROM_V /
// FIN_ZERO at bootstrap) -> wrap_new, update monitor, and X for the next iteration
static FinishArgs finargs(pint_plan p, const double2* wold, double2* wnew, double2* X) {
  FinishArgs a{};
  a.P = p->Pp; a.wrap_old = wold; a.wrap_new = wnew; a.X = X;
  a.src = p->src; a.coef = p->coef; a.spar = p->srclist; a.nsparse = p->nsparse;
  a.igs = p->igs; a.gsf = p->gsf; a.wk = p->wk; a.upd = p->pmon ? p->upd_sink : p->upd;
  a.N = p->N; a.Qb = p->Qb; a.L = (int)p->L; a.Lf = p->Lf; a.Lpad = (int)(p->NB * p->WB); a.WB = p->WB;
  a.NB = (int)p->NB; a.k = p->k; a.nk = p->nk; a.nch = p->nch; a.pstride = p->nch;
  a.skip = p->cap_skip;
  a.ctl = p->cap_ctl; a.arrive = p->cap_ctl ? p->larrive : nullptr; a.hnd = p->cap_hnd;
  return a;
}

static pint_status finish_pass(pint_plan p, int mode, const double2* wold, double2* wnew, double2* X) {
  const FinishArgs a = finargs(p, wold, wnew, X);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->cap_ev && mode == FIN_PARTIALS) {
    e0 = p->cap_ev[2]; e1 = p->cap_ev[3];
    CUDA_TRY(cudaEventRecordWithFlags(e0, p->stream, cudaEventRecordExternal));
  } else if (p->timing && mode == FIN_PARTIALS) {
    CUDA_TRY(cudaEventCreate(&e0)); CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, p->stream));
  }
  CUDA_TRY(launch_finish(a, mode, p->stream));
  ++p->launches;
  if (e0) {
    CUDA_TRY(cudaEventRecordWithFlags(e1, p->stream, p->cap_ev ? cudaEventRecordExternal : cudaEventRecordDefault));
    if (!p->cap_ev) p->tev.push_back({e0, e1});
  }
  return PINT_OK;
}

static DstArgs dargs(pint_plan p) {
  DstArgs a{};
  a.mx = (int)p->mx; a.my = (int)p->my; a.WB = p->WB; a.NB = p->NB; a.N = p->N;
  a.q0 = p->q0; a.Qb = p->Qb; a.n0 = 0; a.M = p->M;
  a.scale = (double)sqrtl(2.0L / (ld)(p->mx + 1));
  a.tw = p->twE;
  return a;
}

// DST along y inside the tile layout (fully modal path): rows = nq x-modes x `levels` levels
static pint_status dst_y(pint_plan p, const double2* in, double2* out, long levels, long nq) {
  DstArgs a{};
  a.in = in; a.out = out; a.rows = nq * levels;
  a.mx = (int)p->L; a.my = 1; a.WB = p->WB; a.NB = p->NB; a.N = levels; a.n0 = 0;
  a.q0 = 0; a.Qb = nq; a.M = p->M;
  a.scale = (double)sqrtl(2.0L / (ld)(p->L + 1));
  a.tw = p->twEy;
  CUDA_TRY(launch_dst(p->NEy, a, DST_TILE_Y, p->stream));
  ++p->launches;
  return PINT_OK;
}

// physical vector [M] (device) -> source slot s (tile layout [ntiles][WB]; DST-x in 2D)
static pint_status to_source(pint_plan p, const double2* phys_vec, int s) {
  double2* dst = p->src + (size_t)s * p->ntiles * p->WB;
  if (p->dim == 1) {
    CUDA_TRY(cudaMemcpyAsync(dst, phys_vec, p->M * sizeof(double2), cudaMemcpyDeviceToDevice, p->stream));
    return PINT_OK;
  }
  if (p->dst_iter) {   // physical x: plain gather into the tile layout
    RemapArgs r{};
    r.in = phys_vec; r.out = dst; r.count = p->M; r.WB = p->WB; r.my = (int)p->my; r.NB = p->NB;
    r.N = p->N; r.n0 = 0; r.M = p->M; r.Qb = p->Qb;
    CUDA_TRY(launch_remap(r, RM_2D_PHYS_TO_SRC, p->stream));
    ++p->launches;
    return PINT_OK;
  }
  DstArgs a = dargs(p);
  a.in = phys_vec; a.out = dst; a.rows = p->my;
  CUDA_TRY(launch_dst(p->NE, a, DST_PHYS_TO_SRC, p->stream));
  ++p->launches;
  return PINT_OK;
}

// ------------------------------------------------------------------------------------------
// 2D P1-FEM Step 2 (fem2d.cuh): E = Dx Dy / 24 applied in physical space, fixed point in the modes
// ------------------------------------------------------------------------------------------
static pint_status fem2d_applyE(pint_plan p, const double2* Y, double2* Z, long levels) {
  TRY(dst_y(p, Y, p->ft, levels, p->Qb));                           // (q, j) -> (q, y)
  DstArgs d = dargs(p);
  d.rows = levels * p->my; d.N = levels; d.n0 = 0;
  d.in = p->ft; d.out = Z;
  CUDA_TRY(launch_dst(p->NE, d, DST_INT_TO_INT, p->stream));        // (q, y) -> (x, y)
  const long total = p->Qb * p->NB * levels * p->WB;
  CUDA_TRY(launch_fem2d_mixed(Z, p->ft, levels, (int)p->mx, (int)p->my, (int)p->NB, p->WB, total, p->stream));
  d.in = p->ft; d.out = Z;
  CUDA_TRY(launch_dst(p->NE, d, DST_INT_TO_INT, p->stream));        // (x, y) -> (q, y)
  TRY(dst_y(p, Z, Z, levels, p->Qb));                               // (q, y) -> (q, j)
  p->launches += 3;
  return PINT_OK;
}

// X = (s_p M + K)^{-1} M H per level (av: X = M^{-1} K H), modal tile layout with `levels` levels.
// Fixed point X <- P^{-1} (b - s E X), P = s M_sym + K, until max |dX| <= 2^-50 max |X| (at most 300
// steps); one synchronisation per step (the stopping test).
static pint_status fem2d_solve(pint_plan p, const double2* H, double2* X, long levels, bool av) {
  Fem2dArgs f{};
  f.b = p->fb; f.H = H; f.X = X; f.sig_p = p->sig_p; f.sig_q = p->sig_q; f.mu = p->mu; f.cx = p->fcx; f.cy = p->fcy;
  f.levels = levels; f.total = p->Qb * p->NB * levels * p->WB; f.L = (int)p->L; f.NB = (int)p->NB; f.WB = p->WB;
  f.av = av ? 1 : 0; f.kscale = 1.0 / (p->h * p->h); f.upd = p->fupd;
  CUDA_TRY(cudaMemsetAsync(p->fupd, 0, 2 * sizeof(unsigned long long), p->stream));
  if (!av) TRY(fem2d_applyE(p, H, p->fe, levels));
  f.EH = p->fe;
  CUDA_TRY(launch_fem2d(f, true, p->stream));
  ++p->launches;
  unsigned long long bits[2];
  CUDA_TRY(cudaMemcpyAsync(bits, p->fupd, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  double xmax;
  std::memcpy(&xmax, &bits[1], sizeof(double));
  for (int it = 1; it <= 300; ++it) {
    TRY(fem2d_applyE(p, X, p->fe, levels));
    CUDA_TRY(cudaMemsetAsync(p->fupd, 0, sizeof(unsigned long long), p->stream));
    CUDA_TRY(launch_fem2d(f, false, p->stream));
    ++p->launches;
    CUDA_TRY(cudaMemcpyAsync(bits, p->fupd, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    double d;
    std::memcpy(&d, &bits[0], sizeof(double));
    if (!std::isfinite(d)) return fail(PINT_ERR_DIVERGED, "2D FEM inner fixed point: non-finite update");
    if (d <= 0x1p-50 * xmax) { p->fem_iters = it; return PINT_OK; }
  }
  return fail(PINT_ERR_NOT_CONVERGED, "2D FEM inner fixed point: no convergence in 300 steps");
}

// ------------------------------------------------------------------------------------------
// problem setup
// ------------------------------------------------------------------------------------------
static pint_status nl_reset(pint_plan p);
static pint_status modal_window_phys(pint_plan p, const double2* wmodal, double2* out);

static pint_status bootstrap(pint_plan p) {
  // U_0^n = v (default) or 0 (PINT_FLAG_U0_ZERO): A = H_1, wrap = last-k of U_0
  const bool zero = (p->flags & PINT_FLAG_U0_ZERO) != 0;
  if (p->fused) {   // window of U_0 and X_1 only
    TRY(finish_pass(p, zero ? FIN_ZERO : FIN_FROM_V, nullptr, p->wrap[p->wcur], p->X[p->xcur]));
    if (p->pmon) TRY(modal_window_phys(p, p->wrap[p->wcur], p->pwin[p->wcur]));
  } else if (p->alpha != 1.0 && p->cqwhat && !p->has_fd && !p->nl) {
    // CQ: H_1 and the full monitor's U_0 elementwise from the separable sources (no transforms)
    CqBootArgs b{};
    b.H = p->A; b.ufull = p->full ? p->ufull : nullptr; b.wrap = p->wrap[p->wcur]; b.src = p->src;
    b.cqhat = p->cqhat; b.cwhat = p->cqwhat; b.S = p->S; b.zero = zero ? 1 : 0; b.k = p->k;
    b.N = p->N; b.ntiles = p->ntiles; b.WB = p->WB;
    CUDA_TRY(launch_cq_boot(b, p->stream));
    ++p->launches;
  } else {
    TRY(tpass(p, zero ? IN_TIME_ZERO : IN_TIME_V, OUT_H, nullptr, p->A, nullptr, p->wrap[p->wcur], false));
  }
  p->stateA = 0;
  p->m = 0;
  p->last_upd = -1.0;
  p->increases = 0;
  if (p->nl) TRY(nl_reset(p));
  return PINT_OK;
}

static pint_status set_problem_impl(pint_plan p, const void* v, int32_t R, const void* g, const double* phi,
                                    const double* dphi, int32_t mem, bool boot);

extern "C" pint_status pint_set_problem_separable(pint_plan p, const void* v, int32_t R, const void* g,
                                                  const double* phi, const double* dphi, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  p->has_fd = false;
  return set_problem_impl(p, v, R, g, phi, dphi, mem, true);
}

static pint_status set_problem_impl(pint_plan p, const void* v, int32_t R, const void* g, const double* phi,
                                    const double* dphi, int32_t mem, bool boot) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!v) return fail(PINT_ERR_ARG, "v must not be NULL");
  if (R < 0 || R > 64) return fail(PINT_ERR_ARG, "R must be in 0..64");
  if (R > 0 && (!g || !phi)) return fail(PINT_ERR_ARG, "R > 0 needs g and phi");
  if (R > 0 && p->k > 2 && !dphi) return fail(PINT_ERR_ARG, "k > 2 with R > 0 needs dphi (d^l phi/dt^l(0), l=1..k-2)");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  CUDA_TRY(cudaSetDevice(p->device));
  const int64_t M = p->M, N = p->N;
  const int k = p->k;
  const cudaMemcpyKind kind = mem == PINT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;

  // sources: 0 = v, 1 = A v, 2.. = g_r
  const int S = 2 + R;
  TRY(stage_reserve(p, (size_t)S * N * (2 * sizeof(double2) + sizeof(double)) + 2 * (size_t)S * sizeof(int) + 256));
  if (p->S != S) {
    if (p->src) return fail(PINT_ERR_STATE, "set_problem may be called again only with the same R");
    TRY(dalloc(p, &p->src, (size_t)S * p->ntiles * p->WB));
    TRY(dalloc(p, &p->coef, (size_t)S * N));
    TRY(dalloc(p, &p->nhi, S));
    TRY(dalloc(p, &p->srclist, S));
    TRY(dalloc(p, &p->chat, (size_t)S * N));
    if (p->alpha != 1.0) TRY(dalloc(p, &p->cqhat, (size_t)S * N));
    p->S = S;
  }
  CUDA_TRY(cudaMemsetAsync(p->src, 0, (size_t)S * p->ntiles * p->WB * sizeof(double2), p->stream));
  const bool chk_real = (p->flags & PINT_FLAG_REAL_DATA) != 0;
  if (chk_real) CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
  CUDA_TRY(cudaMemcpyAsync(p->phys, v, M * sizeof(double2), kind, p->stream));
  if (chk_real) CUDA_TRY(launch_imag_max(p->phys, M, p->upd, p->stream));
  const double ihx2 = (double)((ld)(p->mx + 1) * (ld)(p->mx + 1));
  const double ihy2 = (double)((ld)(p->my + 1) * (ld)(p->my + 1));
  CUDA_TRY(launch_stencil(p->phys, p->phys + M, (int)p->mx, (int)p->my, ihx2, ihy2, p->stream));
  ++p->launches;
  TRY(to_source(p, p->phys, 0));
  TRY(to_source(p, p->phys + M, 1));
  for (int r = 0; r < R; ++r) {
    CUDA_TRY(cudaMemcpyAsync(p->phys, (const double2*)g + (size_t)r * M, M * sizeof(double2), kind, p->stream));
    if (chk_real) CUDA_TRY(launch_imag_max(p->phys, M, p->upd, p->stream));
    TRY(to_source(p, p->phys, 2 + r));
  }
  if (p->modal) TRY(dst_y(p, p->src, p->src, 1, (long)S * p->Qb));   // sources -> (q, j) modes
  if (p->fem) {   // A v = M^{-1} K v is diagonal in the modes: (A v)_j = (mu_j / h^2) v_j (source 1 <- source 0)
    CUDA_TRY(launch_mode_scale(p->src + (size_t)p->ntiles * p->WB, p->src, p->mu, 1.0 / (p->h * p->h), (int)p->L, p->stream));
    ++p->launches;
  }
  if (p->fem2d) TRY(fem2d_solve(p, p->src, p->src + (size_t)p->ntiles * p->WB, 1, true));   // A v = M^{-1} K v
  if (chk_real) {
    double im = 0.0;
    unsigned long long bits = 0;
    CUDA_TRY(cudaMemcpyAsync(&bits, p->upd, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    std::memcpy(&im, &bits, sizeof(im));
    if (im != 0.0) return fail(PINT_ERR_ARG, "PINT_FLAG_REAL_DATA: v or g has a nonzero imaginary part");
  }

  // time coefficients of F_static_n = f̄_n + tau^-a (sum_{j<n} omega_j) v, 1-based n = row+1:
  //   v   : tau^{-a} sum_{j=0}^{n-1} omega_j
  //   A v : -a_n                                         (a_n (f(0) - A v))
  //   g_r : phi_r(t_n) + a_n phi_r(0) + sum_l b_{l,n} tau^l phi_r^{(l)}(0)
  const ld ta = powl((ld)p->tau, -(ld)p->alpha);
  std::vector<ld> w = (p->alpha == 1.0) ? bdf_weights(k) : cq_weights(k, (ld)p->alpha, N + 1);
  w.resize(N + 1, 0.0L);
  std::vector<double> coef((size_t)S * N, 0.0);
  std::vector<int> nhi(S, 0);
  ld ps = 0.0L;
  for (int64_t n = 1; n <= N; ++n) {
    ps += w[n - 1];
    // heat: sum_{j<n} omega_j vanishes exactly for n > k; keep it exact
    if (p->alpha == 1.0 && n > k) ps = 0.0L;
    coef[0 * N + n - 1] = (double)(ta * ps);
    coef[1 * N + n - 1] = (double)(-table1_a(k, (int)n));
    for (int r = 0; r < R; ++r) {
      ld c = (ld)phi[(size_t)r * (N + 1) + n];
      if (n < k) {
        c += table1_a(k, (int)n) * (ld)phi[(size_t)r * (N + 1)];
        for (int l = 1; l <= k - 2; ++l)
          c += table1_b(k, l, (int)n) * powl((ld)p->tau, (ld)l) * (ld)dphi[(size_t)r * (k - 2) + (l - 1)];
      }
      coef[(size_t)(2 + r) * N + n - 1] = (double)c;
    }
  }
  for (int s = 0; s < S; ++s)
    for (int64_t n = 0; n < N; ++n)
      if (coef[(size_t)s * N + n] != 0.0) nhi[s] = (int)(n + 1);
  p->nmax = *std::max_element(nhi.begin(), nhi.end());
  // pruned heat T-pass: sources whose coefficients vanish for n >= 16 enter X_0..X_15; the others
  // are synthesised from the exact DFT of Gamma h^2/N c_s(n) (long double, once per problem)
  {
    std::vector<int> lst;
    int nk = p->k;
    for (int s = 0; s < S; ++s) if (nhi[s] <= 16) { lst.push_back(s); nk = std::max(nk, nhi[s]); }
    p->nsparse = (int)lst.size();
    std::vector<double2> ch;
    const ld hl = 1.0L / (ld)(p->L + 1), Nl = (ld)N;
    std::vector<cld> eN;                               // e^{-2 pi i m/N}, m < N (long double, built once)
    for (int s = 0; s < S; ++s) {
      if (nhi[s] <= 16) continue;
      lst.push_back(s);
      if (eN.empty()) {
        eN.resize(N);
        for (int64_t m = 0; m < N; ++m) {
          const ld ang = -2.0L * PI_L * (ld)m / Nl;
          eN[m] = cld(cosl(ang), sinl(ang));
        }
      }
      std::vector<ld> cg(N);
      for (int64_t n = 0; n < N; ++n) cg[n] = (ld)coef[(size_t)s * N + n] * powl((ld)p->kappa, (ld)n / Nl) * hl * hl / Nl;
      for (int64_t pp = 0; pp < N; ++pp) {
        cld acc = 0.0L;
        for (int64_t n = 0; n < nhi[s]; ++n) acc += cg[n] * eN[(n * pp) % N];
        ch.push_back(d2(acc));
      }
    }
    p->ndense = S - p->nsparse;
    p->nk = nk;
    p->fused = p->fused_ok && nk <= 8;
    TRY(h2d_async(p, p->srclist, lst));
    if (!ch.empty()) TRY(h2d_async(p, p->chat, ch));
  }
  if (p->cqhat) {
    // CQ split T-pass: H_static = V^{-1} Gamma F_static h^2/N is iteration-invariant and separable,
    // H_static[p] = sum_s chat_s[p] src_s with chat_s the DFT of kappa^{n/N} h^2/N c_s(n): long
    // double, radix-2 FFT (N a power of two), once per problem
    const ld hl = 1.0L / (ld)(p->L + 1), Nl = (ld)N;
    std::vector<double2> ch((size_t)S * N);
    std::vector<cld> x(N);
    for (int s = 0; s < S; ++s) {
      for (int64_t n = 0; n < N; ++n) x[n] = (ld)coef[(size_t)s * N + n] * powl((ld)p->kappa, (ld)n / Nl) * hl * hl / Nl;
      fft_ld(x, -1);
      for (int64_t pp = 0; pp < N; ++pp) ch[(size_t)s * N + pp] = d2(x[pp]);
    }
    TRY(h2d_async(p, p->cqhat, ch));
    // the bootstrap iterate U_0^n = v is constant in time, so its kappa-wrap (kappa/tau^a) sum_{j=n}^{N-1}
    // omega_j U_0^{N+n-j} = c_w(n) v is separable too: H_1 = H_static + cwhat[p] v, cwhat = DFT of
    // kappa^{n/N} h^2/N c_w(n) (eq:BDF-subdiff-F): no transform at bootstrap
    {
      std::vector<ld> wq = cq_weights(k, (ld)p->alpha, N + 1);
      const ld ta = powl((ld)p->tau, -(ld)p->alpha);
      ld tail = 0.0L;                                   // sum_{j=n}^{N-1} omega_j, n = N..1
      std::vector<ld> cw(N);
      for (int64_t n = N; n >= 1; --n) {
        cw[n - 1] = (ld)p->kappa * ta * tail;           // n = N: empty sum
        tail += wq[n - 1];
      }
      // cw[n-1] = kappa tau^-a sum_{j=n}^{N-1} omega_j  (tail before adding omega_{n-1})
      for (int64_t n = 0; n < N; ++n) x[n] = cw[n] * powl((ld)p->kappa, (ld)n / Nl) * hl * hl / Nl;
      fft_ld(x, -1);
      std::vector<double2> cwv(N);
      for (int64_t pp = 0; pp < N; ++pp) cwv[pp] = d2(x[pp]);
      if (!p->cqwhat) TRY(dalloc(p, &p->cqwhat, N));
      TRY(h2d_async(p, p->cqwhat, cwv));
    }
  }
  TRY(h2d_async(p, p->coef, coef));
  TRY(h2d_async(p, p->nhi, nhi));
  p->problem_set = true;
  p->wcur = 0;
  if (boot) TRY(bootstrap(p));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->stage_off = 0;                        // the staged copies have completed
  return PINT_OK;
}

extern "C" pint_status pint_set_problem(pint_plan p, const void* v, const void* f, const void* f0, const void* fderiv,
                                        int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!v || !f) return fail(PINT_ERR_ARG, "v and f must not be NULL");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  if (p->nranks > 1) return fail(PINT_ERR_UNSUPPORTED, "dense forcing on several ranks: use the separable form");
  if (p->modal || p->dst_iter) return fail(PINT_ERR_UNSUPPORTED, "dense forcing with PINT_FLAG_MODAL / DST_PER_ITER");
  CUDA_TRY(cudaSetDevice(p->device));
  const int64_t M = p->M, N = p->N;
  const int k = p->k;
  // the starting corrections a_n f(0) and b_{l,n} tau^l f^(l)(0) are separable sources:
  //   g_0 = f(0) with phi_0(t_n) = [n = 0]  ->  coefficient a_n;   g_l = f^(l)(0), dphi_l = e_l -> b_{l,n} tau^l
  const int32_t R = 1 + std::max(k - 2, 0);
  std::vector<double> phi((size_t)R * (N + 1), 0.0), dphi((size_t)R * std::max(k - 2, 0), 0.0);
  phi[0] = 1.0;
  for (int l = 1; l <= k - 2; ++l) dphi[(size_t)l * (k - 2) + (l - 1)] = 1.0;
  const size_t vb = (size_t)M * sizeof(double2);
  double2* gtmp = nullptr;
  std::vector<double2> gh;
  const void* gptr = nullptr;
  if (mem == PINT_HOST) {
    gh.assign((size_t)R * M, make_double2(0.0, 0.0));
    if (f0) std::memcpy(gh.data(), f0, vb);
    if (fderiv && k > 2) std::memcpy(gh.data() + M, fderiv, (size_t)(k - 2) * vb);
    gptr = gh.data();
  } else {
    CUDA_TRY(cudaMalloc(&gtmp, (size_t)R * vb));
    cudaError_t e = cudaMemsetAsync(gtmp, 0, (size_t)R * vb, p->stream);
    if (e == cudaSuccess && f0) e = cudaMemcpyAsync(gtmp, f0, vb, cudaMemcpyDeviceToDevice, p->stream);
    if (e == cudaSuccess && fderiv && k > 2)
      e = cudaMemcpyAsync(gtmp + M, fderiv, (size_t)(k - 2) * vb, cudaMemcpyDeviceToDevice, p->stream);
    if (e != cudaSuccess) { cudaFree(gtmp); return fail(PINT_ERR_CUDA, std::string("set_problem: ") + cudaGetErrorString(e)); }
    gptr = gtmp;
  }
  pint_status st = set_problem_impl(p, v, R, gptr, phi.data(), k > 2 ? dphi.data() : nullptr, mem, false);
  if (gtmp) { cudaStreamSynchronize(p->stream); cudaFree(gtmp); }
  if (st != PINT_OK) return st;
  // f(t_1..t_N) -> tile layout (DST-x per level in 2D), staged through B
  if (!p->fd) TRY(dalloc(p, &p->fd, (size_t)p->ntiles * TILE));
  CUDA_TRY(cudaMemcpyAsync(p->B, f, (size_t)N * vb, mem == PINT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                           p->stream));
  if (p->dim == 1) {
    RemapArgs r{};
    r.in = p->B; r.out = p->fd; r.count = N * M; r.WB = p->WB; r.my = 1; r.NB = p->NB;
    r.N = N; r.n0 = 0; r.M = M; r.Qb = 1;
    CUDA_TRY(launch_remap(r, RM_1D_LEVELS_TO_INT, p->stream));
  } else {
    DstArgs a = dargs(p);
    a.in = p->B; a.out = p->fd; a.rows = N * p->my; a.n0 = 0;
    CUDA_TRY(launch_dst(p->NE, a, DST_PHYS_LEVELS_TO_INT, p->stream));
  }
  ++p->launches;
  p->has_fd = true;
  p->fused = false;            // X is dense in time: streaming path, unpruned T-pass
  TRY(bootstrap(p));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return PINT_OK;
}

extern "C" pint_status pint_set_initial_guess(pint_plan p, const void* U0, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  CUDA_TRY(cudaSetDevice(p->device));
  if (!U0) return bootstrap(p);
  if (p->nranks > 1) return fail(PINT_ERR_UNSUPPORTED, "user initial guess with nranks > 1");
  const size_t bytes = (size_t)p->N * p->M * sizeof(double2);
  CUDA_TRY(cudaMemcpyAsync(p->B, U0, bytes, mem == PINT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, p->stream));
  if (p->flags & PINT_FLAG_REAL_DATA) {
    CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
    CUDA_TRY(launch_imag_max(p->B, p->N * p->M, p->upd, p->stream));
    unsigned long long bits = 0;
    double im = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&bits, p->upd, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    std::memcpy(&im, &bits, sizeof(im));
    if (im != 0.0) return fail(PINT_ERR_ARG, "PINT_FLAG_REAL_DATA: U0 has a nonzero imaginary part");
  }
  if (p->dim == 1) {
    RemapArgs r{};
    r.in = p->B; r.out = p->A; r.count = p->N * p->M; r.WB = p->WB; r.my = 1; r.NB = p->NB;
    r.N = p->N; r.n0 = 0; r.M = p->M; r.Qb = 1;
    CUDA_TRY(launch_remap(r, RM_1D_LEVELS_TO_INT, p->stream));
  } else if (p->dst_iter) {
    RemapArgs r{};
    r.in = p->B; r.out = p->A; r.count = p->N * p->M; r.WB = p->WB; r.my = (int)p->my; r.NB = p->NB;
    r.N = p->N; r.n0 = 0; r.M = p->M; r.Qb = p->Qb;
    CUDA_TRY(launch_remap(r, RM_2D_LEVELS_TO_INT, p->stream));
  } else {
    DstArgs a = dargs(p);
    a.in = p->B; a.out = p->A; a.rows = p->N * p->my; a.n0 = 0;
    CUDA_TRY(launch_dst(p->NE, a, DST_PHYS_LEVELS_TO_INT, p->stream));
  }
  ++p->launches;
  // H_1 and the wrap state of U_0 from the time-domain array
  if (p->modal) {   // fully modal: the iteration lives in (q, j) space
    // in place: A's pad rows (y >= L) are zero, while B still holds the user's array in the
    // physical layout, whose values would sit in the pad slots the DST does not write
    TRY(dst_y(p, p->A, p->A, p->N, p->Qb));
    TRY(tpass(p, IN_TIME_BUF, OUT_H, p->A, p->A, nullptr, p->wrap[p->wcur], false));
  } else {
    TRY(tpass(p, IN_TIME_BUF, OUT_H, p->A, p->A, nullptr, p->wrap[p->wcur], false));
  }
  if (p->fused) TRY(finish_pass(p, FIN_FROM_WRAP, p->wrap[p->wcur], nullptr, p->X[p->xcur]));
  if (p->pmon) TRY(modal_window_phys(p, p->wrap[p->wcur], p->pwin[p->wcur]));
  p->stateA = 0;
  p->m = 0;
  p->last_upd = -1.0;
  p->increases = 0;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return PINT_OK;
}

// ------------------------------------------------------------------------------------------
// iteration
// ------------------------------------------------------------------------------------------
// one fused iteration: update monitor reset, Steps 1-3 (fused kernel), window / X / monitor (finish)
// fused modal plans: the window levels of U, (q, j) modes -> (q, y): DST-y back, the line axis in
// grid space (1D: the grid values; 2D: the DST-x basis of the line path, reading R-norm2D), tile layout
static pint_status modal_window_phys(pint_plan p, const double2* wmodal, double2* out) {
  TRY(dst_y(p, wmodal, out, p->k, p->Qb));
  return PINT_OK;
}

static pint_status fused_kernels(pint_plan p) {
  TRY(fused_pass(p, p->X[p->xcur], false, true));   // Steps 1-3 (block 0 zeroes the update monitor)
  TRY(finish_pass(p, FIN_PARTIALS, p->wrap[p->wcur], p->wrap[1 - p->wcur], p->X[1 - p->xcur]));
  if (p->pmon) {   // max |U_m - U_{m-1}| on the physical window levels
    TRY(modal_window_phys(p, p->wrap[1 - p->wcur], p->pwin[1 - p->wcur]));
    CUDA_TRY(launch_nl_diffmax(p->pwin[1 - p->wcur], p->pwin[p->wcur], (long)p->ntiles * p->k * p->WB, p->upd, p->stream));
    ++p->launches;
  }
  return PINT_OK;
}

static pint_status fused_step(pint_plan p) {
  TRY(fused_kernels(p));
  CUDA_TRY(cudaMemcpyAsync(p->updh, p->upd, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->stream));
  return PINT_OK;
}

// The device-side WR loop: ONE graph launch and one synchronisation per pint_wr_solve instead of one
// per iteration.  Graph = while node; body = [fused, finish, ctl] for parity (w, x) and again for
// the flipped parity; ctl (wr_loop_ctl_kernel) applies pint_wr_solve's stopping rule and clears the
// condition, and sets `done`, which makes the rest of the body return at once.  Results (iterations,
// last update, divergence-guard state) are read back from the LoopCtl state.
static pint_status fused_loop(pint_plan p, double tol, int32_t max_iters, bool guard, int32_t* iters, double* u_out,
                              int* status) {
  if (!p->lctl) {
    TRY(dalloc(p, &p->lctl, 1));
    TRY(dalloc(p, &p->larrive, 1));
    TRY(dalloc(p, &p->lbar, 1));
    CUDA_TRY(cudaMemsetAsync(p->larrive, 0, sizeof(unsigned int), p->stream));
    CUDA_TRY(cudaMemsetAsync(p->lbar, 0, sizeof(GridBar), p->stream));
    CUDA_TRY(cudaHostAlloc((void**)&p->lctl_h, sizeof(LoopCtl), cudaHostAllocDefault));
  }
  // small problems (every (x-mode, chunk) CTA co-resident): the whole loop as ONE cooperative kernel,
  // grid barriers instead of kernel boundaries (fused.cuh wr_loop_kernel)
  if (!p->pmon && !p->modal && !p->half) {
    LoopKArgs L{};
    int cap = 0;
    CUDA_TRY(launch_loop_kernel(p->Cf, p->nk, L, 0, p->k, p->stream, &cap));
    const long grid = p->Qb * (long)p->nch;
    if (grid <= cap) {
      for (int h = 0; h < 2; ++h) {
        const int w = p->wcur ^ h, x = p->xcur ^ h;
        L.fa[h] = fargs(p, p->X[x]);
        L.fin[h] = finargs(p, p->wrap[w], p->wrap[1 - w], p->X[1 - x]);
      }
      L.ctl = p->lctl;
      L.bar = p->lbar;
      LoopCtl* hs = p->lctl_h;
      *hs = LoopCtl{0, max_iters, 1, 0, p->increases, guard ? 1 : 0, tol, p->last_upd, 0.0};
      CUDA_TRY(cudaMemcpyAsync(p->lctl, hs, sizeof(LoopCtl), cudaMemcpyHostToDevice, p->stream));
      CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
      CUDA_TRY(launch_loop_kernel(p->Cf, p->nk, L, grid, p->k, p->stream, nullptr));
      CUDA_TRY(cudaMemcpyAsync(hs, p->lctl, sizeof(LoopCtl), cudaMemcpyDeviceToHost, p->stream));
      CUDA_TRY(cudaStreamSynchronize(p->stream));
      const int it = hs->it;
      if (it & 1) { p->wcur ^= 1; p->xcur ^= 1; }
      p->m += it;
      p->launches += 1;
      p->stateA = 0;
      p->upd_queued = false;
      if (guard) { p->last_upd = hs->last; p->increases = hs->inc; }
      *iters = it;
      *u_out = it > 0 ? hs->u : INFINITY;
      *status = hs->status;
      return PINT_OK;
    }
  }
  const int key = p->wcur * 2 + p->xcur;
  FusedArgs fa[2];
  FinishArgs fin[2];
  p->cap_skip = &p->lctl->done;
  for (int h = 0; h < 2; ++h) {
    const int w = p->wcur ^ h, x = p->xcur ^ h;
    fa[h] = fargs(p, p->X[x]);
    fa[h].upd_reset = p->upd;
    fin[h] = finargs(p, p->wrap[w], p->wrap[1 - w], p->X[1 - x]);
  }
  p->cap_skip = nullptr;
  if (!p->lexec[key] || memcmp(fa, p->lfa[key], sizeof fa) != 0 || memcmp(fin, p->lfin[key], sizeof fin) != 0) {
    if (p->lexec[key]) { CUDA_TRY(cudaGraphExecDestroy(p->lexec[key])); p->lexec[key] = nullptr; }
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hnd;
    cudaError_t e = cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = hnd;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &np);
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(p->stream, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                           cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) { cudaGraphDestroy(g); return fail(PINT_ERR_CUDA, std::string("loop graph: ") + cudaGetErrorString(e)); }
    const int64_t l0 = p->launches;
    const int w0 = p->wcur, x0 = p->xcur;
    p->cap_skip = &p->lctl->done;
    if (!p->pmon) { p->cap_ctl = p->lctl; p->cap_hnd = (unsigned long long)hnd; }   // ctl in the finish kernel
    pint_status st = PINT_OK;
    for (int h = 0; h < 2 && st == PINT_OK; ++h) {
      p->wcur = w0 ^ h;
      p->xcur = x0 ^ h;
      st = fused_kernels(p);
      if (st == PINT_OK && p->pmon) {
        const cudaError_t ec = launch_loop_ctl(p->lctl, p->upd, hnd, p->stream);
        if (ec != cudaSuccess) st = fail(PINT_ERR_CUDA, std::string("loop ctl: ") + cudaGetErrorString(ec));
      }
    }
    p->cap_skip = nullptr;
    p->cap_ctl = nullptr;
    p->cap_hnd = 0;
    p->wcur = w0;
    p->xcur = x0;
    p->llaunch[key] = (p->launches - l0) / 2 + (p->pmon ? 1 : 0);   // + the ctl kernel (modal monitor)
    p->launches = l0;
    cudaGraph_t body = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(p->stream, &body);
    if (st != PINT_OK) { cudaGraphDestroy(g); return st; }
    if (ec != cudaSuccess) { cudaGraphDestroy(g); return fail(PINT_ERR_CUDA, std::string("loop capture: ") + cudaGetErrorString(ec)); }
    const cudaError_t ei = cudaGraphInstantiate(&p->lexec[key], g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(ei);
    memcpy(p->lfa[key], fa, sizeof fa);
    memcpy(p->lfin[key], fin, sizeof fin);
  }
  LoopCtl* hs = p->lctl_h;
  *hs = LoopCtl{0, max_iters, 1, 0, p->increases, guard ? 1 : 0, tol, p->last_upd, 0.0};
  CUDA_TRY(cudaMemcpyAsync(p->lctl, hs, sizeof(LoopCtl), cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(cudaGraphLaunch(p->lexec[key], p->stream));
  CUDA_TRY(cudaMemcpyAsync(hs, p->lctl, sizeof(LoopCtl), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  const int it = hs->it;
  if (it & 1) { p->wcur ^= 1; p->xcur ^= 1; }
  p->m += it;
  p->launches += p->llaunch[key] * (int64_t)it;   // fused + finish [+ modal monitor] + ctl per iteration
  p->stateA = 0;
  p->upd_queued = false;
  if (guard) { p->last_upd = hs->last; p->increases = hs->inc; }
  *iters = it;
  *u_out = it > 0 ? hs->u : INFINITY;
  *status = hs->status;
  return PINT_OK;
}

// Replay fused_step as a CUDA graph: one host launch per iteration instead of three (small
// problems are launch-bound).  The graph for parity key is (re)captured when the arguments the
// kernels would get now differ from the captured ones (set_problem may move sources, nk, ...).
static pint_status fused_step_graph(pint_plan p) {
  const int key = p->wcur * 2 + p->xcur + (p->timing ? 4 : 0);
  const FusedArgs fa = fargs(p, p->X[p->xcur]);
  const FinishArgs fin = finargs(p, p->wrap[p->wcur], p->wrap[1 - p->wcur], p->X[1 - p->xcur]);
  if (!p->gexec[key] || memcmp(&fa, &p->gfa[key], sizeof fa) != 0 || memcmp(&fin, &p->gfin[key], sizeof fin) != 0) {
    if (p->gexec[key]) { CUDA_TRY(cudaGraphExecDestroy(p->gexec[key])); p->gexec[key] = nullptr; }
    const int64_t l0 = p->launches;
    if (p->timing && !p->gev[key][0])
      for (cudaEvent_t& e : p->gev[key]) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeRelaxed));
    p->cap_ev = p->timing ? p->gev[key] : nullptr;
    const pint_status st = fused_step(p);
    p->cap_ev = nullptr;
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(p->stream, &g);
    if (st != PINT_OK) { if (g) cudaGraphDestroy(g); return st; }
    CUDA_TRY(ec);
    const cudaError_t ei = cudaGraphInstantiate(&p->gexec[key], g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(ei);
    p->glaunch = p->launches - l0;
    p->launches = l0;
    p->gfa[key] = fa;
    p->gfin[key] = fin;
  }
  CUDA_TRY(cudaGraphLaunch(p->gexec[key], p->stream));
  p->launches += p->glaunch;
  if (p->timing) p->gpending = key;
  return PINT_OK;
}

// timing mode with graph replay: add the last replay's fused / finish durations (the event nodes
// are re-recorded by every replay, so they are read after each iteration's synchronisation)
static pint_status graph_timing_collect(pint_plan p) {
  if (p->gpending < 0) return PINT_OK;
  cudaEvent_t* e = p->gev[p->gpending];
  p->gpending = -1;
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, e[0], e[1]));
  p->s_ms += ms; ++p->s_n;
  CUDA_TRY(cudaEventElapsedTime(&ms, e[2], e[3]));
  p->t_ms += ms; ++p->t_n;
  return PINT_OK;
}

static pint_status iterate_async(pint_plan p) {
  if (p->fused) {
    if (p->graphs) TRY(fused_step_graph(p));
    else TRY(fused_step(p));
    p->upd_queued = true;
    p->wcur ^= 1;
    p->xcur ^= 1;
    p->stateA = 0;   // A no longer holds U_m
    ++p->m;
    return PINT_OK;
  }
  if (p->stateA == 1) {   // A holds U_m (after get_levels): re-derive H_{m+1}
    if (p->modal) TRY(dst_y(p, p->A, p->A, p->N, p->Qb));   // physical (q, y) -> (q, j) modes
    TRY(tpass(p, IN_TIME_BUF, OUT_H, p->A, p->A, nullptr, p->wrap[p->wcur], false));
    p->stateA = 0;
  }
  CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
  if (p->dst_iter) {
    // ablation: H (physical x) -DST-> B, solve B -> A, W -DST-> B (physical x again)
    DstArgs d = dargs(p);
    d.rows = p->N * p->my; d.n0 = 0;
    d.in = p->A; d.out = p->B;
    CUDA_TRY(launch_dst(p->NE, d, DST_INT_TO_INT, p->stream));
    TRY(spass(p, p->B, p->A));
    d.in = p->A; d.out = p->B;
    CUDA_TRY(launch_dst(p->NE, d, DST_INT_TO_INT, p->stream));
    p->launches += 2;
  } else {
    TRY(spass(p, p->A, p->B));                                           // W_{m+1} = solve(H_{m+1})
  }
  TRY(tpass(p, IN_FREQ, OUT_H, p->B, p->A, p->wrap[p->wcur], p->wrap[1 - p->wcur], true));  // -> H_{m+2}
  p->wcur ^= 1;
  ++p->m;
  return PINT_OK;
}

static pint_status read_update_local(pint_plan p, double* out) {
  if (!p->upd_queued) CUDA_TRY(cudaMemcpyAsync(p->updh, p->upd, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->stream));
  p->upd_queued = false;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  TRY(graph_timing_collect(p));
  std::memcpy(out, p->updh, sizeof(double));
  return PINT_OK;
}

// One iteration and its update norm, max over ranks.  A local error still takes part in the
// all-reduce (contributing +inf), so the other ranks never block in the collective: they see a
// non-finite update (pint_wr_solve: DIVERGED) while this rank returns its own error.
static pint_status step_collective(pint_plan p, double* out) {
  pint_status st = iterate_async(p);
  double u = INFINITY;
  if (st == PINT_OK) st = read_update_local(p, &u);
  if (p->nranks > 1) {
    double x = st == PINT_OK ? u : INFINITY;
    if (p->allreduce(&x, p->actx) != 0) return st != PINT_OK ? st : fail(PINT_ERR_COMM, "allreduce_max callback failed");
    u = x;
  }
  if (st != PINT_OK) return st;
  *out = u;
  return PINT_OK;
}

extern "C" pint_status pint_wr_iterate(pint_plan p, double* update_inf) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (p->nl) return fail(PINT_ERR_STATE, "semilinear plan: use pint_newton_solve");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  CUDA_TRY(cudaSetDevice(p->device));
  double u;
  TRY(step_collective(p, &u));
  if (update_inf) *update_inf = u;
  return PINT_OK;
}

extern "C" pint_status pint_wr_solve(pint_plan p, double tol, int32_t max_iters, int32_t* iters, double* update_inf) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (p->nl) return fail(PINT_ERR_STATE, "semilinear plan: use pint_newton_solve");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (!(tol >= 0.0) || max_iters < 0) return fail(PINT_ERR_ARG, "need tol >= 0 and max_iters >= 0");
  CUDA_TRY(cudaSetDevice(p->device));
  int it = 0;
  double u = INFINITY;
  pint_status result = PINT_ERR_NOT_CONVERGED;
  if (p->fused && p->graphs && p->nranks == 1 && !p->timing && max_iters > 0) {
    // the same stopping rule on the device: one graph launch, one synchronisation (fused_loop)
    int status = 1;
    TRY(fused_loop(p, tol, max_iters, true, &it, &u, &status));
    result = status == 0 ? PINT_OK : (status == 1 ? PINT_ERR_NOT_CONVERGED : PINT_ERR_DIVERGED);
    if (status == 2) g_last_error = "update is not finite";
    if (status == 3) g_last_error = "update grew 3 consecutive times";
    if (status == 1) g_last_error = "max_iters reached before update < tol";
    if (iters) *iters = it;
    if (update_inf) *update_inf = u;
    return result;
  }
  while (it < max_iters) {
    TRY(step_collective(p, &u));
    ++it;
    if (!std::isfinite(u)) { result = PINT_ERR_DIVERGED; g_last_error = "update is not finite"; break; }
    if (p->last_upd >= 0.0 && u > p->last_upd) {
      if (++p->increases >= 3) { result = PINT_ERR_DIVERGED; g_last_error = "update grew 3 consecutive times"; p->last_upd = u; break; }
    } else {
      p->increases = 0;
    }
    p->last_upd = u;
    if (u < tol) { result = PINT_OK; break; }
  }
  if (result == PINT_ERR_NOT_CONVERGED) g_last_error = "max_iters reached before update < tol";
  if (iters) *iters = it;
  if (update_inf) *update_inf = u;
  return result;
}

extern "C" pint_status pint_wr_run(pint_plan p, int32_t iters, double* update_inf) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (p->nl) return fail(PINT_ERR_STATE, "semilinear plan: use pint_newton_solve");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (iters < 1) return fail(PINT_ERR_ARG, "need iters >= 1");
  CUDA_TRY(cudaSetDevice(p->device));
  if (p->fused && p->graphs && p->nranks == 1 && !p->timing) {   // the device-side loop, no stopping rule
    int it = 0, status = 1;
    double u = INFINITY;
    TRY(fused_loop(p, 0.0, iters, false, &it, &u, &status));
    if (update_inf) *update_inf = u;
    return PINT_OK;
  }
  // enqueue all iterations, read (and all-reduce) the last update only
  for (int32_t i = 0; i < iters - 1; ++i) {
    const pint_status st = iterate_async(p);
    if (st != PINT_OK) {
      if (p->nranks > 1) { double x = INFINITY; p->allreduce(&x, p->actx); }   // keep the collective matched
      return st;
    }
    if (p->timing) {   // timing mode: the replayed graph's event nodes are read after each iteration
      double x;
      TRY(read_update_local(p, &x));
    }
  }
  double u;
  TRY(step_collective(p, &u));
  if (update_inf) *update_inf = u;
  return PINT_OK;
}

// ------------------------------------------------------------------------------------------
// semilinear extension: Newton's method with WR inner solves (Algorithm 3)
// ------------------------------------------------------------------------------------------
static pint_status nl_reset(pint_plan p) {
  // U_0^n = v for all n (Algorithm 3, line 1): source 0 holds v (1D tile layout == physical)
  for (int64_t n = 0; n < p->N; ++n)
    CUDA_TRY(cudaMemcpyAsync(p->nlU + n * p->M, p->src, p->M * sizeof(double2), cudaMemcpyDeviceToDevice, p->stream));
  return PINT_OK;
}

extern "C" pint_status pint_set_nonlinearity(pint_plan p, int32_t kind, double eps) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (kind != PINT_NL_ALLEN_CAHN) return fail(PINT_ERR_ARG, "kind must be PINT_NL_ALLEN_CAHN");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(PINT_ERR_ARG, "eps must be > 0");
  if (p->dim != 1 || p->nranks != 1 || p->fem)
    return fail(PINT_ERR_UNSUPPORTED, "the Newton-WR extension is 1D FD on one rank (g'(Ubar(x)) breaks the DST)");
  CUDA_TRY(cudaSetDevice(p->device));
  p->nl_eps = eps;
  p->fused_ok = false;
  p->fused = false;
  if (!p->nl) {
    const size_t arr = (size_t)p->ntiles * TILE;
    TRY(dalloc(p, &p->nlU, (size_t)p->N * p->M));
    TRY(dalloc(p, &p->nlR, arr));
    TRY(dalloc(p, &p->nlT[0], arr));
    TRY(dalloc(p, &p->nlT[1], arr));
    TRY(dalloc(p, &p->nlC, (size_t)p->L));
    TRY(dalloc(p, &p->nlPiv, (size_t)p->N * p->L));
    TRY(dalloc(p, &p->nlWt, (size_t)p->N));
    TRY(dalloc(p, &p->nlAnl, (size_t)p->N));
    CUDA_TRY(cudaMemsetAsync(p->nlR, 0, arr * sizeof(double2), p->stream));
    // tau^-a omega_j (j < N; heat: zero beyond k) and the Table-1 a_n (n = 1..N -> index n-1)
    const ld ta = powl((ld)p->tau, -(ld)p->alpha);
    std::vector<ld> w = (p->alpha == 1.0) ? bdf_weights(p->k) : cq_weights(p->k, (ld)p->alpha, p->N + 1);
    w.resize(p->N + 1, 0.0L);
    std::vector<double> wt(p->N), anl(p->N);
    for (int64_t j = 0; j < p->N; ++j) wt[j] = (double)(ta * w[j]);
    for (int64_t n = 1; n <= p->N; ++n) anl[n - 1] = (double)table1_a(p->k, (int)n);
    TRY(h2d(p, p->nlWt, wt));
    TRY(h2d(p, p->nlAnl, anl));
  }
  p->nl = true;
  if (p->problem_set) {
    TRY(bootstrap(p));   // streaming state + U_0 = v
    CUDA_TRY(cudaStreamSynchronize(p->stream));
  }
  return PINT_OK;
}

// T-pass of the inner linear problem: W^{<=0} = 0 (no v terms), F_static = R (dense), never pruned
static pint_status tpass_nl(pint_plan p, int mode_in, int mode_out, const double2* in, double2* out,
                            const double2* wold, double2* wnew) {
  TPassArgs a = targs(p);
  a.in = in; a.out = out; a.wrap_old = wold; a.wrap_new = wnew;
  a.S = 0; a.nmax = (int)p->N; a.nsparse = 0; a.ndense = 0;
  a.fdense = p->nlR;
  a.ufull = nullptr;   // the inner WR has its own full-array monitor (nl_diffmax)
  CUDA_TRY(launch_tpass((int)p->N, mode_in, mode_out, p->alpha != 1.0, a, p->ntiles, p->stream));
  ++p->launches;
  return PINT_OK;
}

static pint_status read_upd(pint_plan p, double* out) {
  unsigned long long bits = 0;
  CUDA_TRY(cudaMemcpyAsync(&bits, p->upd, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  std::memcpy(out, &bits, sizeof(double));
  return PINT_OK;
}

extern "C" pint_status pint_newton_solve(pint_plan p, int32_t max_outer, double outer_tol, double inner_tol,
                                         int32_t max_inner, int32_t* inner_counts, double* outer_updates,
                                         int32_t* outer_done) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!p->nl) return fail(PINT_ERR_STATE, "call pint_set_nonlinearity first");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (max_outer < 0 || max_inner < 1 || !(inner_tol >= 0.0) || !(outer_tol >= 0.0))
    return fail(PINT_ERR_ARG, "need max_outer >= 0, max_inner >= 1, tolerances >= 0");
  CUDA_TRY(cudaSetDevice(p->device));
  NewtonArgs na{};
  na.U = p->nlU; na.R = p->nlR; na.c = p->nlC; na.src = p->src; na.coef = p->coef; na.wt = p->nlWt; na.anl = p->nlAnl;
  na.fd = p->has_fd ? p->fd : nullptr;
  na.S = p->S; na.L = (int)p->L; na.Lpad = (int)(p->NB * p->WB); na.WB = p->WB; na.N = p->N;
  const ld hl = 1.0L / (ld)(p->L + 1);
  na.ih2 = (double)(1.0L / (hl * hl)); na.h2 = (double)(hl * hl); na.ieps2 = 1.0 / (p->nl_eps * p->nl_eps);
  VcArgs va{};
  va.piv = p->nlPiv; va.sig_p = p->sig_p; va.c = p->nlC; va.N = p->N; va.L = (int)p->L;
  va.Lpad = (int)(p->NB * p->WB); va.WB = p->WB;
  const long count = p->ntiles * TILE;
  pint_status result = PINT_ERR_NOT_CONVERGED;
  int32_t done = 0;
  for (int32_t l = 0; l < max_outer; ++l) {
    CUDA_TRY(launch_nl_coeff(na, p->stream));
    CUDA_TRY(launch_nl_residual(na, p->stream));
    p->launches += 2;
    // inner WR on W: W_0 = 0 -> H_1 into A, window 0
    TRY(tpass_nl(p, IN_TIME_ZERO, OUT_H, nullptr, p->A, nullptr, p->wrap[p->wcur]));
    CUDA_TRY(cudaMemsetAsync(p->nlT[0], 0, count * sizeof(double2), p->stream));
    int cur = 1, m = 0;
    double upd = INFINITY;
    while (m < max_inner) {
      va.in = p->A; va.out = p->B;
      CUDA_TRY(launch_spass_vc(va, p->stream));                                             // W_m (freq)
      TRY(tpass_nl(p, IN_FREQ, OUT_H, p->B, p->A, p->wrap[p->wcur], p->wrap[1 - p->wcur]));  // H_{m+1}
      p->wcur ^= 1;
      TRY(tpass_nl(p, IN_FREQ, OUT_U, p->B, p->nlT[cur], nullptr, nullptr));                // W_m (time)
      CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
      CUDA_TRY(launch_nl_diffmax(p->nlT[cur], p->nlT[1 - cur], count, p->upd, p->stream));
      p->launches += 2;
      ++m;
      TRY(read_upd(p, &upd));
      cur ^= 1;
      if (!std::isfinite(upd)) { g_last_error = "inner update is not finite"; return PINT_ERR_DIVERGED; }
      if (upd < inner_tol) break;
    }
    // U_l = U_{l-1} + W (latest W_m is nlT[1 - cur])
    CUDA_TRY(cudaMemsetAsync(p->upd, 0, sizeof(unsigned long long), p->stream));
    CUDA_TRY(launch_nl_update(p->nlU, p->nlT[1 - cur], p->N, (int)p->L, p->WB, p->upd, p->stream));
    ++p->launches;
    double ou = 0.0;
    TRY(read_upd(p, &ou));
    if (inner_counts) inner_counts[l] = m;
    if (outer_updates) outer_updates[l] = ou;
    ++done;
    ++p->m;
    if (!std::isfinite(ou)) { g_last_error = "Newton update is not finite"; result = PINT_ERR_DIVERGED; break; }
    if (ou < outer_tol) { result = PINT_OK; break; }
  }
  if (result == PINT_ERR_NOT_CONVERGED && done == max_outer && outer_tol == 0.0) result = PINT_OK;
  if (result == PINT_ERR_NOT_CONVERGED) g_last_error = "max_outer reached before the Newton update < outer_tol";
  if (outer_done) *outer_done = done;
  p->stateA = 2;   // A/B hold inner-WR data: pint_get_levels reads U_l
  return result;
}

// ------------------------------------------------------------------------------------------
// output
// ------------------------------------------------------------------------------------------
static pint_status materialize(pint_plan p) {
  if (p->stateA == 1 || p->stateA == 3) return PINT_OK;
  if (p->full && !p->fused && !p->nl) {
    // the full-array monitor keeps U_m of every level in `ufull` (tile layout): no Step-3 pass
    if (p->modal) {                          // (q, j) modes -> (q, y) into A (H is re-derived later)
      TRY(dst_y(p, p->ufull, p->A, p->N, p->Qb));
      p->stateA = 1;
    } else {
      p->stateA = 3;
    }
    return PINT_OK;
  }
  if (p->fused && p->modal) {
    // W_m per (q, j) mode into A, U_m = Gamma^{-1} V W_m into B, DST-y back to (q, y) into A
    FusedArgs a = fargs(p, p->X[1 - p->xcur]);
    a.W = p->A; a.half = 0;
    CUDA_TRY(launch_modal(true, a, p->stream));
    ++p->launches;
    TRY(tpass(p, IN_FREQ, OUT_U, p->A, p->B, nullptr, nullptr, false));
    TRY(dst_y(p, p->B, p->A, p->N, p->Qb));
    p->stateA = 1;
    return PINT_OK;
  }
  // fused: W_m = solve(H_m) with H_m synthesised from the X that produced it, into B
  if (p->fused) TRY(fused_pass(p, p->X[1 - p->xcur], true));
  // U_m = Gamma^{-1} V W_m (Step 3) from B into A (time domain)
  TRY(tpass(p, IN_FREQ, OUT_U, p->B, p->A, nullptr, nullptr, false));
  if (p->modal) TRY(dst_y(p, p->A, p->A, p->N, p->Qb));   // streaming modal: (q, j) -> (q, y), B keeps W_m
  p->stateA = 1;
  return PINT_OK;
}

// the materialised U_m (tile layout): A, or the full-array monitor's copy
static const double2* ucur(pint_plan p) { return p->stateA == 3 ? p->ufull : p->A; }

extern "C" pint_status pint_get_levels(pint_plan p, int64_t n_begin, int64_t n_count, void* U, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (n_begin < 0 || n_count < 0 || n_begin + n_count > p->N) return fail(PINT_ERR_ARG, "levels out of range [0, N)");
  if (!U && n_count > 0) return fail(PINT_ERR_ARG, "U must not be NULL");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  if (p->nranks > 1) return fail(PINT_ERR_UNSUPPORTED, "nranks > 1: use pint_get_modal_levels + pint_modal_to_physical");
  CUDA_TRY(cudaSetDevice(p->device));
  if (p->nl) {   // semilinear plans: the Newton iterate U_l (physical [N][M]; l = 0 gives v)
    if (n_count == 0) return PINT_OK;
    CUDA_TRY(cudaMemcpyAsync(U, p->nlU + n_begin * p->M, n_count * p->M * sizeof(double2),
                             mem == PINT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PINT_OK;
  }
  if (p->m == 0) return fail(PINT_ERR_STATE, "no WR iterate computed yet (m = 0)");
  if (n_count == 0) return PINT_OK;
  if (n_begin >= p->N - p->k && p->stateA != 1) {
    // levels inside the window n = N-k..N-1: read from the wrap state (no materialisation)
    if (!p->wstage) TRY(dalloc(p, &p->wstage, (size_t)p->k * p->M));
    double2* wdst = mem == PINT_DEVICE ? (double2*)U : p->wstage;
    const double2* wsrc = p->wrap[p->wcur];
    if (p->modal) {   // window levels are (q, j)-modal: DST-y back first
      if (!p->wtmp) TRY(dalloc(p, &p->wtmp, (size_t)p->ntiles * p->k * p->WB));
      TRY(dst_y(p, p->wrap[p->wcur], p->wtmp, p->k, p->Qb));
      wsrc = p->wtmp;
    }
    if (p->dim == 1) {
      RemapArgs r{};
      r.in = wsrc; r.out = wdst; r.count = n_count * p->M; r.WB = p->WB; r.my = 1; r.NB = p->NB;
      r.N = p->k; r.n0 = n_begin - (p->N - p->k); r.M = p->M; r.Qb = 1;
      CUDA_TRY(launch_remap(r, RM_INT_TO_1D_LEVELS, p->stream));
    } else if (p->dst_iter) {
      RemapArgs r{};
      r.in = p->wrap[p->wcur]; r.out = wdst; r.count = n_count * p->M; r.WB = p->WB; r.my = (int)p->my;
      r.NB = p->NB; r.N = p->k; r.n0 = n_begin - (p->N - p->k); r.M = p->M; r.Qb = p->Qb;
      CUDA_TRY(launch_remap(r, RM_INT_TO_2D_LEVELS, p->stream));
    } else {
      DstArgs a = dargs(p);
      a.in = wsrc; a.out = wdst; a.rows = n_count * p->my; a.N = p->k; a.n0 = n_begin - (p->N - p->k);
      CUDA_TRY(launch_dst(p->NE, a, DST_INT_TO_PHYS_LEVELS, p->stream));
    }
    ++p->launches;
    if (mem == PINT_HOST)
      CUDA_TRY(cudaMemcpyAsync(U, wdst, n_count * p->M * sizeof(double2), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PINT_OK;
  }
  TRY(materialize(p));
  const double2* usrc = ucur(p);
  double2* dst = mem == PINT_DEVICE ? (double2*)U : p->B;   // B is free once U_m is in A (or ufull)
  if (p->dim == 1) {
    RemapArgs r{};
    r.in = usrc; r.out = dst; r.count = n_count * p->M; r.WB = p->WB; r.my = 1; r.NB = p->NB;
    r.N = p->N; r.n0 = n_begin; r.M = p->M; r.Qb = 1;
    CUDA_TRY(launch_remap(r, RM_INT_TO_1D_LEVELS, p->stream));
  } else if (p->dst_iter) {
    RemapArgs r{};
    r.in = usrc; r.out = dst; r.count = n_count * p->M; r.WB = p->WB; r.my = (int)p->my; r.NB = p->NB;
    r.N = p->N; r.n0 = n_begin; r.M = p->M; r.Qb = p->Qb;
    CUDA_TRY(launch_remap(r, RM_INT_TO_2D_LEVELS, p->stream));
  } else {
    DstArgs a = dargs(p);
    a.in = usrc; a.out = dst; a.rows = n_count * p->my; a.n0 = n_begin;
    CUDA_TRY(launch_dst(p->NE, a, DST_INT_TO_PHYS_LEVELS, p->stream));
  }
  ++p->launches;
  if (mem == PINT_HOST)
    CUDA_TRY(cudaMemcpyAsync(U, dst, n_count * p->M * sizeof(double2), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return PINT_OK;
}

extern "C" pint_status pint_get_solution(pint_plan p, void* U, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  return pint_get_levels(p, 0, p->N, U, mem);
}

extern "C" pint_status pint_get_modal_levels(pint_plan p, int64_t n_begin, int64_t n_count, void* Uq, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (p->dim != 2) return fail(PINT_ERR_ARG, "modal levels exist for 2D operators only");
  if (p->dst_iter) return fail(PINT_ERR_UNSUPPORTED, "PINT_FLAG_DST_PER_ITER keeps physical x: use pint_get_levels");
  if (n_begin < 0 || n_count < 0 || n_begin + n_count > p->N) return fail(PINT_ERR_ARG, "levels out of range [0, N)");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  if (p->m == 0) return fail(PINT_ERR_STATE, "no WR iterate computed yet (m = 0)");
  CUDA_TRY(cudaSetDevice(p->device));
  TRY(materialize(p));
  double2* dst = mem == PINT_DEVICE ? (double2*)Uq : p->B;
  RemapArgs r{};
  r.in = ucur(p); r.out = dst; r.count = n_count * p->my * p->Qb; r.WB = p->WB; r.my = (int)p->my;
  r.NB = p->NB; r.N = p->N; r.n0 = n_begin; r.M = p->M; r.Qb = p->Qb;
  CUDA_TRY(launch_remap(r, RM_INT_TO_MODAL, p->stream));
  ++p->launches;
  if (mem == PINT_HOST)
    CUDA_TRY(cudaMemcpyAsync(Uq, dst, r.count * sizeof(double2), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return PINT_OK;
}

extern "C" pint_status pint_modal_to_physical(pint_plan p, int64_t n_count, const void* Uq_full, void* U, int32_t mem) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (p->dim != 2) return fail(PINT_ERR_ARG, "2D operators only");
  if (n_count < 0 || !Uq_full || !U) return fail(PINT_ERR_ARG, "bad n_count or NULL buffers");
  if (mem != PINT_HOST && mem != PINT_DEVICE) return fail(PINT_ERR_ARG, "mem must be PINT_HOST or PINT_DEVICE");
  CUDA_TRY(cudaSetDevice(p->device));
  const size_t elems = (size_t)n_count * p->M, bytes = elems * sizeof(double2);
  DstArgs a = dargs(p);
  a.rows = n_count * p->my;
  if (mem == PINT_DEVICE) {
    a.in = (const double2*)Uq_full; a.out = (double2*)U;
    CUDA_TRY(launch_dst(p->NE, a, DST_ROWS, p->stream));
    ++p->launches;
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PINT_OK;
  }
  // host arrays: stage through B when it is free and large enough, else temporaries
  double2* stage = nullptr;
  bool tmp = false;
  if (p->stateA == 1 && 2 * elems <= (size_t)p->ntiles * TILE) {
    stage = p->B;                                    // U_m already materialised in A
  } else {
    CUDA_TRY(cudaMalloc(&stage, 2 * bytes));
    tmp = true;
  }
  cudaError_t e = cudaMemcpyAsync(stage, Uq_full, bytes, cudaMemcpyHostToDevice, p->stream);
  a.in = stage; a.out = stage + elems;
  if (e == cudaSuccess) e = launch_dst(p->NE, a, DST_ROWS, p->stream);
  ++p->launches;
  if (e == cudaSuccess) e = cudaMemcpyAsync(U, stage + elems, bytes, cudaMemcpyDeviceToHost, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  if (tmp) cudaFree(stage);
  if (e != cudaSuccess) return fail(PINT_ERR_CUDA, std::string("modal_to_physical: ") + cudaGetErrorString(e));
  return PINT_OK;
}

extern "C" pint_status pint_partition(int64_t mx, int32_t rank, int32_t nranks, int64_t* q_begin, int64_t* q_end) {
  if (nranks < 1 || rank < 0 || rank >= nranks || mx < 1 || nranks > mx)
    return fail(PINT_ERR_ARG, "need 1 <= nranks <= mx and 0 <= rank < nranks");
  if (q_begin) *q_begin = (rank * mx) / nranks;
  if (q_end) *q_end = ((rank + 1) * mx) / nranks;
  return PINT_OK;
}

extern "C" pint_status pint_get_partition(pint_plan p, int64_t* q_begin, int64_t* q_end) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (q_begin) *q_begin = p->q0;
  if (q_end) *q_end = p->q0 + p->Qb;
  return PINT_OK;
}

extern "C" pint_status pint_set_timing(pint_plan p, int32_t enable) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  for (auto& e : p->tev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (auto& e : p->sev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  p->tev.clear(); p->sev.clear();
  p->t_ms = p->s_ms = 0; p->t_n = p->s_n = 0;
  p->gpending = -1;
  p->timing = enable != 0;
  return PINT_OK;
}

extern "C" pint_status pint_get_timing(pint_plan p, double* tpass_ms, double* spass_ms, int64_t* tn, int64_t* sn) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  TRY(graph_timing_collect(p));
  for (auto& e : p->tev) {
    float ms = 0; CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    p->t_ms += ms; ++p->t_n; cudaEventDestroy(e.first); cudaEventDestroy(e.second);
  }
  for (auto& e : p->sev) {
    float ms = 0; CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    p->s_ms += ms; ++p->s_n; cudaEventDestroy(e.first); cudaEventDestroy(e.second);
  }
  p->tev.clear(); p->sev.clear();
  if (tpass_ms) *tpass_ms = p->t_ms;
  if (spass_ms) *spass_ms = p->s_ms;
  if (tn) *tn = p->t_n;
  if (sn) *sn = p->s_n;
  return PINT_OK;
}

static pint_status residual_local(pint_plan p, double* r_out, double* f_out);

extern "C" pint_status pint_residual(pint_plan p, double* residual_inf, double* rhs_inf) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  double r = 0.0, f = 0.0;
  const pint_status st = residual_local(p, &r, &f);
  if (p->nranks > 1) {
    // collective: every rank makes the same all-reduce calls even when its local part failed
    double bad = st == PINT_OK ? 0.0 : 1.0;
    if (p->allreduce(&bad, p->actx) != 0) return st != PINT_OK ? st : fail(PINT_ERR_COMM, "allreduce_max callback failed");
    if (st != PINT_OK) return st;
    if (bad != 0.0) return fail(PINT_ERR_COMM, "pint_residual failed on another rank");
    if (p->allreduce(&r, p->actx) != 0 || p->allreduce(&f, p->actx) != 0) return fail(PINT_ERR_COMM, "allreduce_max callback failed");
  }
  if (st != PINT_OK) return st;
  if (residual_inf) *residual_inf = r;
  if (rhs_inf) *rhs_inf = f;
  return PINT_OK;
}

static pint_status residual_local(pint_plan p, double* r_out, double* f_out) {
  if (!p->problem_set) return fail(PINT_ERR_STATE, "call pint_set_problem_separable first");
  if (p->m == 0) return fail(PINT_ERR_STATE, "no WR iterate computed yet (m = 0)");
  if (p->nl || p->dst_iter || p->has_fd || (p->alpha != 1.0 && p->modal) || p->fem2d)
    return fail(PINT_ERR_UNSUPPORTED, "pint_residual: separable data; CQ on the line-solve path; not 2D P1-FEM");
  CUDA_TRY(cudaSetDevice(p->device));
  TRY(materialize(p));                     // U_m, x in DST modes, y physical (tile layout)
  const double2* U = ucur(p);
  if (p->modal) {                          // back to (q, j) modes, where the sources live; B is free
    TRY(dst_y(p, p->A, p->B, p->N, p->Qb));   // here (A keeps U_m, the next iteration re-derives from it)
    U = p->B;
  }
  if (!p->wstage) TRY(dalloc(p, &p->wstage, (size_t)p->k * p->M));
  unsigned long long* acc = (unsigned long long*)p->wstage;   // 2 words of scratch
  CUDA_TRY(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), p->stream));
  ResidArgs a{};
  a.U = U; a.src = p->src; a.coef = p->coef; a.wk = p->wk; a.sig_q = p->sig_q; a.out = acc;
  a.mu = p->modal ? p->mu : nullptr;
  if (p->alpha != 1.0) {   // CQ: the full history convolution per column, tile by tile into B (free here)
    CUDA_TRY(launch_resid_cq_time(U, p->B, p->cqw, p->N, p->ntiles, p->stream));
    ++p->launches;
    a.tconv = p->B;
  }
  a.N = p->N; a.NB = p->NB; a.Qb = p->Qb; a.WB = p->WB; a.L = (int)p->L; a.S = p->S; a.k = p->k;
  a.ikappa = 1.0 / p->kappa; a.ih2 = 1.0 / (p->h * p->h);
  CUDA_TRY(launch_resid(a, p->stream));
  ++p->launches;
  unsigned long long bits[2];
  CUDA_TRY(cudaMemcpyAsync(bits, acc, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  std::memcpy(r_out, &bits[0], sizeof(double));
  std::memcpy(f_out, &bits[1], sizeof(double));
  return PINT_OK;
}

extern "C" pint_status pint_get_info(pint_plan p, int64_t* m, int64_t* launches, int64_t* dev_bytes) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (m) *m = p->m;
  if (launches) *launches = p->launches;
  if (dev_bytes) *dev_bytes = p->dev_bytes;
  return PINT_OK;
}

extern "C" pint_status pint_get_path(pint_plan p, int32_t* fused, int32_t* chunks, int32_t* nk) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  if (fused) *fused = p->fused ? 1 : 0;
  if (chunks) *chunks = p->fused ? p->nch : 0;
  if (nk) *nk = p->nk;
  return PINT_OK;
}

extern "C" pint_status pint_plan_destroy(pint_plan p) {
  if (!p) return fail(PINT_ERR_ARG, "plan is NULL");
  free_plan(p);
  return PINT_OK;
}

extern "C" const char* pint_status_string(pint_status s) {
  switch (s) {
    case PINT_OK: return "PINT_OK";
    case PINT_ERR_ARG: return "PINT_ERR_ARG";
    case PINT_ERR_ALLOC: return "PINT_ERR_ALLOC";
    case PINT_ERR_CUDA: return "PINT_ERR_CUDA";
    case PINT_ERR_COMM: return "PINT_ERR_COMM";
    case PINT_ERR_STATE: return "PINT_ERR_STATE";
    case PINT_ERR_NOT_CONVERGED: return "PINT_ERR_NOT_CONVERGED";
    case PINT_ERR_DIVERGED: return "PINT_ERR_DIVERGED";
    case PINT_ERR_UNSUPPORTED: return "PINT_ERR_UNSUPPORTED";
  }
  return "PINT_ERR_UNKNOWN";
}

extern "C" const char* pint_last_error(void) { return g_last_error.c_str(); }

extern "C" double pint_kappa_log_rule(int64_t N) {
  if (N < 2) return 0.5;
  return std::min(1.0 / std::log((double)N), 0.5);
}
