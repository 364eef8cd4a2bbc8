// fused.cuh — the whole heat (alpha = 1) WR iteration in one kernel per x-mode, with no
// space-time array in HBM ("window-state" ParaDiag, DESIGN.md §5 "Fused iteration").
//
// The next iterate depends on U_m only through its last k levels (the kappa-wrap, PAPER.md:388,
// 416-428), and for heat X = Gamma F h^2/N vanishes beyond the first nk <= 8 levels (F_static
// has k-1 nonzero levels plus dense-in-time sources, which enter through their exact DFTs).  So
// per x-mode q the state of the iteration is X_t[y] (t < nk) and the window U^{N-k+j}[y] (j < k),
// and one iteration is, for every frequency p and every line y (Algorithm 1):
//   Step 1  H_p[y]  = sum_{t<nk} X_t[y] e^{-2 pi i t p/N}  (+ sum_d chat_d[p] src_d[y])
//   Step 2  W_p     = (sigma_p + sigma_q + A_y)^{-1} H_p           (tridiagonal line solve)
//   Step 3  U^n[y]  = kappa^{-n/N} sum_p e^{+2 pi i n p/N} W_p[y],   n = N-k .. N-1 only
// The frequencies are processed in groups of FG = 8, p = i + (N/8) s (s < 8): Step 1 for a group
// is one twiddle per input and a DFT8 per row, Step 3 one DFT8 per row and k twiddled
// accumulations (FFT pruning: only nk inputs, only k outputs).  The group's 8 lines live in shared
// memory (H in, W out, in place); the k window partial sums of the CTA live in shared memory.
// Every one of the N*M space-time unknowns is synthesised, solved and transformed each iteration;
// only H and W are never written to HBM.  A finish kernel sums the partials, monitors the update,
// stores the new window and forms X for the next iteration.
#pragma once
#include "spass.cuh"
#include "tpass.cuh"

namespace pint {

constexpr int FG = 8;      // lines per group (radix of the Step-1 / Step-3 DFTs)

// Per line (q, p): the iteration-invariant constants of the Toeplitz factorisation (spass.cuh),
// computed once at plan time (line_const_kernel).
struct LineConst {
  double2 u;        // 1 - a,  a = 1/r, r + 1/r = 2 + sigma, |r| > 1
  double2 uh;       // u-form of a^{CS}, CS = rows per sub-chain
  double2 uE;       // u-form of a^{(2L+2) mod C}
  double2 ru2L;     // 1 / (1 - a^{2L+2})
  double2 rr;       // r
  double2 rrh;      // r^{CS}
  double2 uc[8];    // u-forms of a^{C 2^i}
  double2 ap[5];    // a^{2^i} (value form), i < 5: per-lane powers of the boundary fix-up
  double tl;        // log(1e-18 |1 - a^{2L+2}|) / log|a|: |a^e / (1 - a^{2L+2})| > 1e-18 iff e < tl
  int nlev;         // lane-scan levels i < nlev have |a^{C 2^i}| >= 2^-64 (the others add nothing: skipped)
  int pad1;
};                  // 320 bytes
constexpr int LC_CHUNKS = 20;   // 16-byte cp.async chunks per LineConst
static_assert(sizeof(LineConst) == 16 * LC_CHUNKS, "LineConst is staged in 16-byte chunks");

struct FusedArgs {
  const double2* X;        // [Qb][8][Lf]  X_t[y], zero for t >= nk and y >= L
  const LineConst* lc;     // [Qb][N]
  const double2* tw;       // [N] e^{-2 pi i m/N}
  const double2* src;      // [S][Qb][Lpad] source vectors (tile layout, DST-x applied)
  const int* dsrc;         // [ndense] source indices with dense time coefficients
  const double2* chat;     // [ndense][N]
  double2* P;              // [Qb][nch][k][Lf] partial sums sum_p e^{2 pi i n p/N} W_p
  double2* W;              // STORE_W: W_m in the tile layout [q][yb][N][WB]
  long N, Qb;
  int L, Lf, Lpad, WB, NB, k, nk, ndense, nch, gpc;
  unsigned long long* prof; // profiling builds (-DPINT_FUSED_PROF): cycles per phase, total + per warp
  int xs;                  // 1: X of the CTA's x-mode staged once into shared memory (TMEM variant, nk small)
  int half;                // 1: real data (PINT_FLAG_REAL_DATA): W_{N-p} = conj(W_p), so only the groups
                           //    i <= N/16 are solved and the others enter the window as conjugates
  const double* mu;        // fully modal path (PINT_FLAG_MODAL): [L] mu_j = 4 sin^2(j pi h_y / 2)
  const double2* sig_p;    // modal path: [N] h^2 d_p / tau^a
  const double* sig_q;     // modal path: [Qb] h^2 lambda_q
  const int* skip;         // device-side WR loop (pint_wr_solve / pint_wr_run graphs): the kernel returns
                           // at once when *skip != 0 (the loop stopped inside an unrolled pair)
  unsigned long long* upd_reset;   // iteration launches: the update monitor, zeroed by block 0 before
                                   // the finish kernel accumulates into it (replaces a memset)
};
static_assert(sizeof(FusedArgs) == 176, "FusedArgs must stay padding-free");

// smem row swizzle: lane l of the solve owns rows [lC, lC + C); XOR-ing the low bits with the
// chunk index keeps its 16-byte accesses bank-conflict free, and consecutive rows (row phases)
// stay within their aligned 8-row block.
template <int C> __device__ __forceinline__ int swz(int y) {
  constexpr int CM = C < 8 ? C : 8;
  constexpr int SH = C >= 8 ? 0 : (C == 4 ? 1 : (C == 2 ? 2 : 3));
  return y ^ (((y / C) >> SH) & (CM - 1));
}

// Row addressing of lane gl's chunk in a swizzled line (swz): y0 + (r ^ m), m constant per lane,
// so the 8 (or C) distinct low parts are precomputed once and every row is pointer + immediate.
template <int C> struct SwzRows {
  static constexpr int CM = C < 8 ? C : 8;
  double2* p[CM];
  __device__ __forceinline__ SwzRows(double2* Hl, int gl) {
    constexpr int SH = C >= 8 ? 0 : (C == 4 ? 1 : (C == 2 ? 2 : 3));
    const int m = (gl >> SH) & (CM - 1);
#pragma unroll
    for (int i = 0; i < CM; ++i) p[i] = Hl + gl * C + (i ^ m);
  }
  __device__ __forceinline__ double2& operator[](int r) const { return p[r & (CM - 1)][r & ~(CM - 1)]; }
};

__device__ __forceinline__ double2 one_minus(double2 u) { return make_double2(1.0 - u.x, -u.y); }

// Recurrence multipliers.  AF = false: the shift-accurate u-form (c = 1 - multiplier, every
// product z - c z); AF = true: the plain value form, used for lines with |u| >= 1e-3,
// where the rounding of a = 1 - u perturbs u (hence the shift) by at most 2e-13 relatively.
template <bool AF> __device__ __forceinline__ double2 mstep(double2 c, double2 z, double2 d) {   // d + m z
  if constexpr (AF) return cfma(c, z, d);
  else return cadd(d, amul(c, z));
}
// the backward sweep on v = a w: v_y = a (f_y + v_{y+1}) — the final x = a (w - w_0 phi) then needs no
// multiplication by a per row (the chunked scan combines exactly as for w: a chunk's value is its
// zero-carry total plus a^len times the carry)
template <bool AF> __device__ __forceinline__ double2 vstep(double2 c, double2 z, double2 f);
template <bool AF> __device__ __forceinline__ double2 mmul(double2 c, double2 z) {
  if constexpr (AF) return cmul(c, z);
  else return amul(c, z);
}
template <bool AF> __device__ __forceinline__ double2 mconv(double2 uform) { return AF ? one_minus(uform) : uform; }
template <bool AF> __device__ __forceinline__ double2 vstep(double2 c, double2 z, double2 f) { return mmul<AF>(c, cadd(f, z)); }
// value form: the forward carry sweep stores g_y = a f_y, so that the backward sweeps are v_y = g_y + a v_{y+1}
// (one complex FMA, two dependent DFMAs per step instead of an add and a multiply: three); u-form: g = f
template <bool AF> __device__ __forceinline__ double2 gform(double2 c, double2 f) {
  if constexpr (AF) return cmul(c, f);
  else return f;
}
template <bool AF> __device__ __forceinline__ double2 bstep(double2 c, double2 z, double2 g) {
  if constexpr (AF) return cfma(c, z, g);
  else return vstep<false>(c, z, g);
}
constexpr double FUSED_AF_U2 = 1e-6;   // |u|^2 threshold of the value form

// LANES lanes per line: 32 (one warp; default) or 64 (two warps, pair-scoped named barriers);
// threads per CTA = 8 LANES; LF = LANES C rows per line; NS interleaved sub-chains per lane chunk.
#ifndef PINT_FUSED_NS
#define PINT_FUSED_NS 2   // A/B r2 (C4 10.17 -> 10.07 ms, C3 0.418 -> 0.402 ms; 8: 10.63 ms)
#endif
#ifndef PINT_TM_BATCH
#define PINT_TM_BATCH 4   // rows per TMEM load batch in the window phase
#endif
#ifndef PINT_FUSED_MINB16
#define PINT_FUSED_MINB16 2   // resident CTAs per SM for lines of <= 512 rows (C <= 16)
#endif
template <int LANES> struct FCfg {
  static constexpr int THREADS = FG * LANES;
  static constexpr int NSMAX = LANES == 32 ? PINT_FUSED_NS : 2;
  // C <= 16 (L <= 512): half the line registers, 64 KB of lines, <= 256 TMEM columns: two CTAs
  // per SM interleave their solve and row phases
  static constexpr int minb(int C) { return (LANES == 32 && C <= 16) ? PINT_FUSED_MINB16 : 1; }
};
template <int C, int LANES> constexpr int fused_ns() { return C < FCfg<LANES>::NSMAX ? C : FCfg<LANES>::NSMAX; }

__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Step 2 for line (q, p): rows gl*C .. gl*C + C - 1 of lane gl (chunked scan, spass.cuh), each chunk
// as NS interleaved sub-chains of CS rows (independent dependency chains).
template <int C, int LANES, bool STORE_W, bool AF>
__device__ __forceinline__ void fused_solve(const FusedArgs& a, double2* Hl, const LineConst& lc, double2* xch,
                                            long q, long p, int half, int bar, unsigned long long* sp = nullptr) {
  constexpr bool PAIR = LANES == 64;
#ifdef PINT_SOLVE_PROF
  long long tp_ = clock64();
#define PINT_SP(j) do { const long long t_ = clock64(); if (sp) sp[j] += t_ - tp_; tp_ = t_; } while (0)
#else
#define PINT_SP(j) do { } while (0)
#endif
  constexpr int NS = fused_ns<C, LANES>();
  constexpr int CS = C / NS;
  const int lane = threadIdx.x & 31;
  const int gl = PAIR ? half * 32 + lane : lane;
  const int L = a.L;
  const double2 u = mconv<AF>(lc.u);                        // a
  const double2 uh = mconv<AF>(lc.uh);                      // a^{CS}
  double2 uc[5];                                            // a^{C 2^i}
#pragma unroll
  for (int i = 0; i < 5; ++i) uc[i] = mconv<AF>(lc.uc[i]);
  const int y0 = gl * C;
  const int nv = min(max(L - y0, 0), C);
  double2 d[C];
  // pad rows y >= L of Hl hold exact zeros (X and the sources vanish there): no load masking
  const SwzRows<C> rows(Hl, gl);
  // loads in the order the forward sweep consumes them (row r of every sub-chain, then r + 1; neutral in
  // an A/B on C4 and C3, kept: the sweep may start before the whole chunk has landed)
#pragma unroll
  for (int r = 0; r < CS; ++r)
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) d[s2 * CS + r] = rows[s2 * CS + r];

  // ---- forward recurrence f_y = d_y + a f_{y-1} ----
  double2 fs[NS];
  // zero carry: the first step of each sub-chain is its first row (no multiplication of the zero state)
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2) fs[s2] = d[s2 * CS];
#pragma unroll
  for (int r = 1; r < CS; ++r)
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) fs[s2] = mstep<AF>(u, fs[s2], d[s2 * CS + r]);
  PINT_SP(0);
  double2 f = fs[0];
#pragma unroll
  for (int s2 = 1; s2 < NS; ++s2) f = mstep<AF>(uh, f, fs[s2]);          // chunk total (zero carry)
  if (PAIR && half == 1) {                                                 // inject warp 0's total
    pair_sync(bar);
    if (lane == 0) f = mstep<AF>(uc[0], xch[0], f);
  }
  const int nlev = PAIR ? 5 : lc.nlev;                                     // warp-uniform
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i >= nlev) break;
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_up_sync(0xffffffffu, f.x, o);
    x.y = __shfl_up_sync(0xffffffffu, f.y, o);
    if (lane >= o) f = mstep<AF>(uc[i], x, f);
  }
  if (PAIR && half == 0) {
    if (lane == 31) xch[0] = f;
    pair_sync(bar);
  }
  double2 carry;
  carry.x = __shfl_up_sync(0xffffffffu, f.x, 1);
  carry.y = __shfl_up_sync(0xffffffffu, f.y, 1);
  if (lane == 0) carry = (PAIR && half) ? xch[0] : make_double2(0.0, 0.0);
  PINT_SP(1);
  double2 st[NS];
  st[0] = carry;
#pragma unroll
  for (int s2 = 1; s2 < NS; ++s2) st[s2] = mstep<AF>(uh, st[s2 - 1], fs[s2 - 1]);
#pragma unroll
  for (int r = 0; r < CS; ++r)
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
      st[s2] = mstep<AF>(u, st[s2], d[s2 * CS + r]);
      d[s2 * CS + r] = gform<AF>(u, st[s2]);
    }
  PINT_SP(2);
  // the lane holding row L-1: the backward sweep starts from zero at row L.  L = LF - 1 (the
  // 2^n - 1 grids) has one pad row: a warp-uniform branch avoids C predicated selects per lane.
  if (L >= LANES * C - 1) {
    if (nv < C) d[C - 1] = make_double2(0.0, 0.0);
  } else if (nv < C) {
#pragma unroll
    for (int r = 0; r < C; ++r)
      if (r >= nv) d[r] = make_double2(0.0, 0.0);
  }

  // ---- backward recurrence w_y = f_y + a w_{y+1}, carried as v = a w: v_y = a (f_y + v_{y+1}) ----
  // (value form: v_y = g_y + a v_{y+1}, so the zero-carry start is the last row's g itself)
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2) fs[s2] = AF ? d[s2 * CS + CS - 1] : make_double2(0.0, 0.0);
#pragma unroll
  for (int r = AF ? CS - 2 : CS - 1; r >= 0; --r)
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) fs[s2] = bstep<AF>(u, fs[s2], d[s2 * CS + r]);
  PINT_SP(3);
  double2 w = fs[NS - 1];
#pragma unroll
  for (int s2 = NS - 2; s2 >= 0; --s2) w = mstep<AF>(uh, w, fs[s2]);
  if (PAIR && half == 0) {                                                 // inject warp 1's total
    pair_sync(bar);
    if (lane == 31) w = mstep<AF>(uc[0], xch[1], w);
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i >= nlev) break;
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_down_sync(0xffffffffu, w.x, o);
    x.y = __shfl_down_sync(0xffffffffu, w.y, o);
    if (lane + o < 32) w = mstep<AF>(uc[i], x, w);
  }
  if (PAIR && half == 1) {
    if (lane == 0) xch[1] = w;
    pair_sync(bar);
  }
  carry.x = __shfl_down_sync(0xffffffffu, w.x, 1);
  carry.y = __shfl_down_sync(0xffffffffu, w.y, 1);
  if (lane == 31) carry = (PAIR && !half) ? xch[1] : make_double2(0.0, 0.0);
  st[NS - 1] = carry;
#pragma unroll
  for (int s2 = NS - 2; s2 >= 0; --s2) st[s2] = mstep<AF>(uh, st[s2 + 1], fs[s2 + 1]);
  PINT_SP(4);
  if constexpr (!STORE_W && !PAIR) {
    // Large-shift lines (the P correction reaches < 256 rows, the Q correction none): the rows are
    // stored as the carry sweep produces them, and the warp fixes rows y < rP up afterwards, one row
    // per lane.  v_0 is lane 0's inclusive backward total (the scan above), known before the sweep.
    if (lc.tl <= 258.0 && (double)L + 3.0 >= lc.tl) {                     // warp-uniform
      double2 w0;
      w0.x = __shfl_sync(0xffffffffu, w.x, 0);
      w0.y = __shfl_sync(0xffffffffu, w.y, 0);
      double2 al = lc.ap[1];                                               // a^{lane + 2}
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if ((lane >> i) & 1) al = cmul(al, lc.ap[i]);
#pragma unroll
      for (int r = CS - 1; r >= 0; --r)
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          st[s2] = bstep<AF>(u, st[s2], d[s2 * CS + r]);
          rows[s2 * CS + r] = st[s2];
        }
      PINT_SP(5);
      const int rP = min((int)ceil(lc.tl - 2.0), L);
      double2 Ka = cmul(cmul(w0, lc.ru2L), al);                            // K a^{y+2}, y = lane
      const double2 a32 = cmul(lc.ap[4], lc.ap[4]);
      __syncwarp();
      for (int yy = lane; yy < rP; yy += 32) {
        double2& xr = Hl[swz<C>(yy)];
        xr = csub(xr, Ka);
        Ka = cmul(Ka, a32);
      }
      PINT_SP(8);
      return;
    }
  }
#pragma unroll
  for (int r = CS - 1; r >= 0; --r)
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
      st[s2] = bstep<AF>(u, st[s2], d[s2 * CS + r]);
      d[s2 * CS + r] = st[s2];
    }

  PINT_SP(5);
  // ---- rank-1 Dirichlet correction x = v - v_0 phi (v = a w), phi_y = (a^{y+2} - a^{2L+2-y}) / (1 - a^{2L+2}) ----
  double2 w0;
  if constexpr (PAIR) {
    if (half == 0 && lane == 0) xch[2] = d[0];
    pair_sync(bar);
    w0 = xch[2];
  } else {
    w0.x = __shfl_sync(0xffffffffu, d[0].x, 0);
    w0.y = __shfl_sync(0xffffffffu, d[0].y, 0);
  }
  const double2 K = cmul(w0, lc.ru2L);
  // rows y < rP carry a P term K a^{y+2} above the 1e-18 threshold: y + 2 < tl.  When they are
  // few (rP <= 256: the large-shift lines) the warp fixes them up after the store, one row per lane,
  // instead of every lane running the C-row correction loop for lane 0's sake.
  const double rPd = lc.tl - 2.0;
  const bool fastP = !STORE_W && !PAIR && rPd <= 256.0;
  if (nv > 0) {
    const double tl = lc.tl;
    if (!fastP && y0 + 2 < tl) {                                           // |a^{y+2}| is largest at y0
      double2 ul = uprod(lc.u, lc.u);                                      // a^2
#pragma unroll
      for (int i = 0; i < (PAIR ? 6 : 5); ++i)
        if ((gl >> i) & 1) ul = uprod(ul, lc.uc[i]);                      // a^{C gl + 2}
      double2 KP[NS];
      KP[0] = cmul(K, one_minus(ul));
#pragma unroll
      for (int s2 = 1; s2 < NS; ++s2) KP[s2] = cmul(KP[s2 - 1], one_minus(lc.uh));
      const double2 a1 = one_minus(lc.u);
#pragma unroll
      for (int r = 0; r < CS; ++r)
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) { d[s2 * CS + r] = csub(d[s2 * CS + r], KP[s2]); KP[s2] = cmul(KP[s2], a1); }
    }
    if (2.0 * L + 2 - (y0 + nv - 1) < tl) {                                // |a^{2L+2-y}| largest at the chunk end
      const int m = (2 * L + 2) / C - gl;                                  // 2L+2-y0 = e + C m, e = (2L+2) mod C
      double2 uq = lc.uE;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((m >> i) & 1) uq = uprod(uq, lc.uc[i]);
      double2 KQ[NS];
      KQ[0] = cmul(K, one_minus(uq));
#pragma unroll
      for (int s2 = 1; s2 < NS; ++s2) KQ[s2] = cmul(KQ[s2 - 1], lc.rrh);
      const double2 rr = lc.rr;
#pragma unroll
      for (int r = 0; r < CS; ++r)
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) { d[s2 * CS + r] = cadd(d[s2 * CS + r], KQ[s2]); KQ[s2] = cmul(KQ[s2], rr); }
    }
  }
  PINT_SP(6);
  if constexpr (STORE_W) {
    double2* Wq = a.W + (q * a.NB * a.N + p) * a.WB;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int y = y0 + r;
      if (y < a.Lpad) Wq[((long)(y / a.WB) * a.N) * a.WB + (y % a.WB)] = (r < nv) ? d[r] : make_double2(0.0, 0.0);
    }
  } else {
#pragma unroll
    for (int r = 0; r < C; ++r) rows[r] = d[r];   // pad rows: never read (finish uses y < L)
    PINT_SP(7);
    if (fastP) {
      // x_y -= K a^{y+2} for y < rP, K = v_0 / (1 - a^{2L+2}) (value-form powers: |a| < 0.85 here)
      __syncwarp();
      const int rP = min((int)ceil(rPd), L);
      double2 al = make_double2(1.0, 0.0);                                 // a^{lane}
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if ((lane >> i) & 1) al = cmul(al, lc.ap[i]);
      double2 Ka = cmul(K, lc.ap[1]);                                      // K a^2
      Ka = cmul(Ka, al);
      const double2 a32 = cmul(lc.ap[4], lc.ap[4]);
      for (int yy = lane; yy < rP; yy += 32) {
        double2& xr = Hl[swz<C>(yy)];
        xr = csub(xr, Ka);
        Ka = cmul(Ka, a32);
      }
    }
    PINT_SP(8);
  }
}

// ---- Tensor memory (TMEM) for the window partial sums --------------------------------------
// Each row thread keeps its acc[rr][r] (window slots r = 2..7 <-> level n = N - 8 + r) in its TMEM
// lane: warp w reads/writes lanes 32 (w % 4) .. + 31; column block (w / 4) * RPT * 24 + rr * 24.
// 24 32-bit columns per row = 6 complex doubles.  This frees 96 KB of shared memory bandwidth per
// group (the RMW of 6 partial sums per row) onto the otherwise idle TMEM datapath.
__device__ __forceinline__ void tmem_ld24_async(uint32_t addr, uint32_t (&w)[24]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                 "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
               : "r"(addr));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23])
               : "r"(addr + 16));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld24(uint32_t addr, uint32_t (&w)[24]) {
  tmem_ld24_async(addr, w);
  tmem_wait_ld();
}
__device__ __forceinline__ void tmem_st24(uint32_t addr, const uint32_t (&w)[24]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
               :: "r"(addr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                  "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]) : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
               :: "r"(addr + 16), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]),
                  "r"(w[23]) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// NW (16, 24 or 32) columns of this thread's TMEM lane, in chunks of 16 and 8 (X levels, 4 per level)
template <int O, int NW> __device__ __forceinline__ void tmem_ld16_at(uint32_t addr, uint32_t (&w)[NW]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(w[O + 0]), "=r"(w[O + 1]), "=r"(w[O + 2]), "=r"(w[O + 3]), "=r"(w[O + 4]), "=r"(w[O + 5]),
                 "=r"(w[O + 6]), "=r"(w[O + 7]), "=r"(w[O + 8]), "=r"(w[O + 9]), "=r"(w[O + 10]), "=r"(w[O + 11]),
                 "=r"(w[O + 12]), "=r"(w[O + 13]), "=r"(w[O + 14]), "=r"(w[O + 15])
               : "r"(addr + O));
}
template <int O, int NW> __device__ __forceinline__ void tmem_ld8_at(uint32_t addr, uint32_t (&w)[NW]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(w[O + 0]), "=r"(w[O + 1]), "=r"(w[O + 2]), "=r"(w[O + 3]), "=r"(w[O + 4]), "=r"(w[O + 5]),
                 "=r"(w[O + 6]), "=r"(w[O + 7])
               : "r"(addr + O));
}
template <int O, int NW> __device__ __forceinline__ void tmem_st16_at(uint32_t addr, const uint32_t (&w)[NW]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
               :: "r"(addr + O), "r"(w[O + 0]), "r"(w[O + 1]), "r"(w[O + 2]), "r"(w[O + 3]), "r"(w[O + 4]),
                  "r"(w[O + 5]), "r"(w[O + 6]), "r"(w[O + 7]), "r"(w[O + 8]), "r"(w[O + 9]), "r"(w[O + 10]),
                  "r"(w[O + 11]), "r"(w[O + 12]), "r"(w[O + 13]), "r"(w[O + 14]), "r"(w[O + 15]) : "memory");
}
template <int O, int NW> __device__ __forceinline__ void tmem_st8_at(uint32_t addr, const uint32_t (&w)[NW]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
               :: "r"(addr + O), "r"(w[O + 0]), "r"(w[O + 1]), "r"(w[O + 2]), "r"(w[O + 3]), "r"(w[O + 4]),
                  "r"(w[O + 5]), "r"(w[O + 6]), "r"(w[O + 7]) : "memory");
}
template <int NW> __device__ __forceinline__ void tmem_ldn_async(uint32_t addr, uint32_t (&w)[NW]) {
  static_assert(NW == 16 || NW == 24 || NW == 32, "16, 24 or 32 columns");
  tmem_ld16_at<0>(addr, w);
  if constexpr (NW == 24) tmem_ld8_at<16>(addr, w);
  if constexpr (NW == 32) tmem_ld16_at<16>(addr, w);
}
template <int NW> __device__ __forceinline__ void tmem_stn(uint32_t addr, const uint32_t (&w)[NW]) {
  static_assert(NW == 16 || NW == 24 || NW == 32, "16, 24 or 32 columns");
  tmem_st16_at<0>(addr, w);
  if constexpr (NW == 24) tmem_st8_at<16>(addr, w);
  if constexpr (NW == 32) tmem_st16_at<16>(addr, w);
}
template <int NW> __device__ __forceinline__ double2 tw_getn(const uint32_t (&w)[NW], int s) {
  return make_double2(__hiloint2double((int)w[4 * s + 1], (int)w[4 * s]), __hiloint2double((int)w[4 * s + 3], (int)w[4 * s + 2]));
}
template <int NW> __device__ __forceinline__ void tw_putn(uint32_t (&w)[NW], int s, double2 v) {
  const unsigned long long a = (unsigned long long)__double_as_longlong(v.x), b = (unsigned long long)__double_as_longlong(v.y);
  w[4 * s] = (uint32_t)a; w[4 * s + 1] = (uint32_t)(a >> 32); w[4 * s + 2] = (uint32_t)b; w[4 * s + 3] = (uint32_t)(b >> 32);
}
__device__ __forceinline__ double2 tw_get(const uint32_t (&w)[24], int s) {
  return make_double2(__hiloint2double((int)w[4 * s + 1], (int)w[4 * s]), __hiloint2double((int)w[4 * s + 3], (int)w[4 * s + 2]));
}
__device__ __forceinline__ void tw_put(uint32_t (&w)[24], int s, double2 v) {
  const unsigned long long a = (unsigned long long)__double_as_longlong(v.x), b = (unsigned long long)__double_as_longlong(v.y);
  w[4 * s] = (uint32_t)a; w[4 * s + 1] = (uint32_t)(a >> 32); w[4 * s + 2] = (uint32_t)b; w[4 * s + 3] = (uint32_t)(b >> 32);
}

// Window contribution of group i: c = e^{2 pi i n i/N} Y.  Real data (half spectrum): the group's
// conjugate partner N/8 - i (lines p <-> N - p) adds conj(c), so a pair contributes 2 Re(c); the
// self-conjugate groups 0 and N/16 contribute Re(c).
__device__ __forceinline__ double2 wcontrib(double2 Y, double2 w, int half, double hw) {
  const double2 c = cmul(Y, w);
  return half ? make_double2(hw * c.x, 0.0) : c;
}

// Row phase between two solves, thread per row (rows y = tid + THREADS r): all X loads of the
// next synthesis and the group's twiddles are issued first (one memory round trip), then each row
// reduces group i into the window (Step 3) and synthesises group i + 1 in place (Step 1).
// XT: X of this x-mode read from tensor memory (txs: this thread's X columns, 4 NKC per row)
template <int C, int LANES, bool WINDOW, bool TM = false, bool HALF = false, int NKC = 8, bool XT = false>
__device__ __forceinline__ void fused_rows(const FusedArgs& a, double2* Hs, double2* acc, const double2* Xq,
                                           long q, int i, bool next, uint32_t tacc = 0, uint32_t txs = 0) {
  constexpr int LF = LANES * C, T = FCfg<LANES>::THREADS;
  constexpr int RPT = LF >= T ? LF / T : 1;
  const int N = (int)a.N, k = a.k, nk = a.nk;
  const int NG = N / FG;
  const int i1 = i + 1;
  // ---- Step 3 (window of group i) for all rows of this thread ----
  if (WINDOW) {
    const double hw = (i == 0 || 16 * i == N) ? 1.0 : 2.0;      // half spectrum: pair weight
    double2 tww[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = t - 8 + k;                                                               // level n = N - 8 + t
      double2 w = (t >= 8 - NKC && j >= 0) ? __ldg(&a.tw[((N - 8 + t) * i) & (N - 1)]) : make_double2(0.0, 0.0);
      w.y = -w.y;                                                                            // e^{+2 pi i n i/N}
      tww[t] = w;
    }
    if constexpr (TM) {
      // slots r = 2..7 of each row; TMEM loads in batches of TMB rows (one round trip per batch)
      constexpr int TMB = PINT_TM_BATCH < RPT ? PINT_TM_BATCH : RPT;
      uint32_t w[RPT][24];
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        if (rr % TMB == 0) {
#pragma unroll
          for (int b = rr; b < rr + TMB && b < RPT; ++b)
            if (!(LF < T && threadIdx.x + T * b >= LF)) tmem_ld24_async(tacc + 24 * b, w[b]);
          tmem_wait_ld();
        }
        const int y = threadIdx.x + T * rr;
        if (LF < T && y >= LF) break;                    // warp-uniform (LF % 32 == 0)
        double2 x[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) x[s2] = Hs[s2 * LF + swz<C>(y)];
        dft8<+1>(x);                                     // Y_r = sum_s e^{+2 pi i rs/8} W_{i + (N/8) s}
#pragma unroll
        for (int r = 2; r < 8; ++r)
          if (r >= 8 - NKC && r - 8 + k >= 0)
            tw_put(w[rr], r - 2, HALF ? cadd(tw_get(w[rr], r - 2), wcontrib(x[r], tww[r], 1, hw))
                                        : cfma(x[r], tww[r], tw_get(w[rr], r - 2)));
        tmem_st24(tacc + 24 * rr, w[rr]);
      }
    } else {
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int y = threadIdx.x + T * rr;
        if (LF < T && y >= LF) break;
        double2 x[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) x[s2] = Hs[s2 * LF + swz<C>(y)];
        dft8<+1>(x);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int j = r - 8 + k;
          if (r >= 8 - NKC && j >= 0)
            acc[j * LF + y] = HALF ? cadd(acc[j * LF + y], wcontrib(x[r], tww[r], 1, hw))
                                     : cfma(x[r], tww[r], acc[j * LF + y]);
        }
      }
    }
  }
  // ---- Step 1 (synthesis of group i + 1) in place ----
  if (next) {
    double2 xv[RPT][8];
    if constexpr (XT) {
      constexpr int XC = 4 * NKC;
      uint32_t xw[RPT][XC];
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr)
        if (!(LF < T && threadIdx.x + T * rr >= LF)) tmem_ldn_async<XC>(txs + XC * rr, xw[rr]);
      tmem_wait_ld();
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr)
#pragma unroll
        for (int t = 0; t < 8; ++t) xv[rr][t] = t < NKC ? tw_getn<XC>(xw[rr], t) : make_double2(0.0, 0.0);
    } else {
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int y = threadIdx.x + T * rr;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          xv[rr][t] = (t < NKC && t < nk && y < LF) ? Xq[t * LF + y] : make_double2(0.0, 0.0);
      }
    }
    double2 tws[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) tws[t] = (t > 0 && t < NKC && t < nk) ? __ldg(&a.tw[t * i1]) : make_double2(1.0, 0.0);   // w_N^{t (i+1)}
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) {
      const int y = threadIdx.x + T * rr;
      if (LF < T && y >= LF) break;
      double2* z = xv[rr];
#pragma unroll
      for (int t = 1; t < NKC; ++t) z[t] = cmul(z[t], tws[t]);                   // X_t w_N^{t (i+1)}
      dft8z<-1, NKC>(z);                                 // H_{i+1 + (N/8) s} = sum_t (.) e^{-2 pi i ts/8}
      for (int dd = 0; dd < a.ndense; ++dd) {
        const double2 g = y < a.L ? __ldg(&a.src[((long)__ldg(&a.dsrc[dd]) * a.Qb + q) * a.Lpad + y])
                                  : make_double2(0.0, 0.0);
        const double2* ch = a.chat + (long)dd * N + i1;
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) z[s2] = cfma(__ldg(&ch[s2 * NG]), g, z[s2]);
      }
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) Hs[s2 * LF + swz<C>(y)] = z[s2];
    }
  }
}

// line constants of group i (8 lines x 240 B) -> shared memory, 16-byte cp.async chunks
__device__ __forceinline__ void fused_stage_lc(const FusedArgs& a, LineConst* slc, long q, int i) {
  const int NG = (int)(a.N / FG);
  const int t = threadIdx.x;
  if (t < 8 * LC_CHUNKS) {
    const int line = t / LC_CHUNKS, c = t % LC_CHUNKS;
    const char* src = (const char*)(a.lc + q * a.N + i + (long)NG * line) + 16 * c;
    cp_async16((char*)(slc + line) + 16 * c, src);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}


// ---- finish: window of U_{m+1}, update monitor, X for the next iteration ----
enum { FIN_PARTIALS = 0, FIN_FROM_WRAP = 1, FIN_FROM_V = 2, FIN_ZERO = 3 };

struct FinishArgs {
  const double2* P;        // [Qb][nch][k][Lf]
  const double2* wrap_old; // [q*NB + yb][k][WB]
  double2* wrap_new;
  double2* X;              // [Qb][8][Lf]
  const double2* src;      // [S][Qb][Lpad]
  const double* coef;      // [S][N]
  const int* spar;         // [nsparse]
  const double* igs;       // [N] kappa^{-n/N}
  const double* gsf;       // [N] kappa^{n/N} h^2 / N
  const double* wk;        // [k+1] (kappa/tau) omega_j
  unsigned long long* upd;
  long N, Qb;
  int L, Lf, Lpad, WB, NB, k, nk, nsparse, nch;
  int pstride;             // chunks per x-mode in the memory layout of P; nch = how many are summed
  const int* skip;         // device-side WR loop: return at once when *skip != 0 (see FusedArgs)
  struct LoopCtl* ctl;     // device-side WR loop: the LAST block to finish applies the stopping rule
  unsigned int* arrive;    //   (block arrival counter, reset by that block)
  unsigned long long hnd;  //   while-node condition handle (cudaGraphConditionalHandle)
};
static_assert(sizeof(FinishArgs) == 176, "FinishArgs must stay padding-free");

// Device-side WR loop (pint_wr_solve without a host round trip per iteration): the state of the
// stopping rule of pint_wr_solve (update < tol, max_iters, 3 consecutive increases or a non-finite
// update: PAPER.md:1747-1748), advanced after every iteration by the last block of the finish
// kernel (or by wr_loop_ctl_kernel when the monitor comes later: fully modal plans).
struct LoopCtl {
  int it, max_it, status, done, inc, guard;   // status: 0 OK, 1 max_iters, 2 non-finite, 3 three increases
  double tol, last, u;                        // last < 0: no previous update
};

// the host loop's stopping rule (pint.cu, pint_wr_solve) for update u: advances the state, returns
// true (and sets done) when the loop stops
__device__ __forceinline__ bool loop_ctl_eval(LoopCtl* s, double u) {
  if (s->done) return true;
  s->u = u;
  s->it += 1;
  int stop = 0;
  if (s->guard) {
    if (!(u <= 1.7976931348623157e308)) {
      s->status = 2;
      stop = 1;
    } else {
      if (s->last >= 0.0 && u > s->last) {
        if (++s->inc >= 3) {
          s->status = 3;
          stop = 1;
        }
      } else {
        s->inc = 0;
      }
      s->last = u;
      if (!stop && u < s->tol) {
        s->status = 0;
        stop = 1;
      }
    }
  }
  if (!stop && s->it >= s->max_it) {
    s->status = 1;
    stop = 1;
  }
  if (stop) s->done = 1;
  return stop != 0;
}
// the rule on a register copy of the state: one batch of loads and one of stores (field by field on
// global memory it was ~10 dependent L2 round trips inside the grid barrier's critical section)
__device__ __forceinline__ bool loop_ctl_apply(LoopCtl* s, double u) {
  LoopCtl c = *s;
  const bool stop = loop_ctl_eval(&c, u);
  *s = c;
  return stop;
}
// ... and clears the while-node condition of the device-loop graph
__device__ __forceinline__ void loop_ctl_step(LoopCtl* s, double u, cudaGraphConditionalHandle h) {
  if (loop_ctl_apply(s, u)) cudaGraphSetConditional(h, 0);
}

#ifndef PINT_BAR_SLEEP
#define PINT_BAR_SLEEP 0    // ns between polls of the grid barrier's generation word (0: spin; 40 measured no better)
#endif
// the whole WR loop as one cooperative kernel (wr_loop_kernel below)
struct GridBar { unsigned int count, gen; };
struct LoopKArgs {
  FusedArgs fa[2];           // the two ping-pong parities (X in, window in/out)
  FinishArgs fin[2];
  LoopCtl* ctl;
  GridBar* bar;
};

// grid-wide barrier of a co-resident (cooperatively launched) grid; the last block to arrive runs
// the stopping rule on the iteration's update (and resets the monitor) before releasing the others
__device__ __forceinline__ void grid_sync(GridBar* b, LoopCtl* ctl, unsigned long long* upd) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &b->gen;
    const unsigned int g = *vgen;
    __threadfence();                                   // this block's writes before its arrival
    const unsigned int arrived = atomicAdd(&b->count, 1u);
    PINT_ASSERT(arrived < gridDim.x);                  // a barrier generation never overflows
    if (arrived == gridDim.x - 1) {
      if (ctl) {
        const double u = __longlong_as_double((long long)*(volatile unsigned long long*)upd);
        *upd = 0ull;
        loop_ctl_apply(ctl, u);
      }
      b->count = 0u;
      __threadfence();
      atomicExch(&b->gen, g + 1u);
    } else {
      while (*vgen == g) {
#if PINT_BAR_SLEEP > 0
        __nanosleep(PINT_BAR_SLEEP);
#endif
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// after this block's atomicMax into *upd: the last block to arrive reads the final update and
// advances the loop (device-scope fence + arrival counter: every block's maximum is in before)
__device__ __forceinline__ void finish_loop_tail(LoopCtl* ctl, unsigned int* arrive, unsigned long long hnd,
                                                 const unsigned long long* upd) {
  if (!ctl || threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
    *arrive = 0u;
    __threadfence();
    const double u = __longlong_as_double((long long)*(volatile const unsigned long long*)upd);
    loop_ctl_step(ctl, u, (cudaGraphConditionalHandle)hnd);
  }
}

#ifdef PINT_DEFINE_FUSED_KERNELS

// TMEM columns per lane quadrant: the window sums (24 per row) and X (4 NKC per row) of the
// (T / 128) threads sharing the quadrant
template <int C, int LANES, int NKC = 8> struct FTmem {
  static constexpr int LF = LANES * C, T = FCfg<LANES>::THREADS;
  static constexpr int RPT = LF >= T ? LF / T : 1;
  static constexpr int WCOLS = (T / 128) * RPT * 24;
  static constexpr int NEED = WCOLS + (T / 128) * RPT * 4 * NKC;   // columns
  static constexpr int COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
};

// TM: window partial sums in tensor memory (default) instead of shared memory.
// HALF: real-data half spectrum (PINT_FLAG_REAL_DATA; instantiated with TM only).
// NKC: compile-time bound on nk (and k): X_t = 0 for t >= NKC and window slots r < 8 - NKC are
// unused, so the synthesis twiddles and the DFT8 butterflies on those zeros/outputs are pruned.
// One fused iteration of this CTA's (x-mode, chunk): Steps 1-3 for its frequency groups, window partial
// sums -> P.  TMEM (when TM && !STORE_W) is allocated by the caller: tbase.
template <int C, int LANES, bool STORE_W, bool TM, bool HALF, int NKC>
__device__ __forceinline__ void fused_iteration(const FusedArgs& a, double2* fsm, uint32_t tbase) {
  constexpr int LF = LANES * C;
  constexpr bool TMA = TM && !STORE_W;                  // TMEM accumulators in use
  double2* Hs = fsm;                                   // [8][LF]  H (in) / W (out) of the group's lines
  double2* acc = fsm + 8 * LF;                         // [k][LF]  window partial sums (shared-memory variant)
  LineConst* slc = (LineConst*)(acc + (TMA ? 0 : a.k * LF));   // [8] line constants of the group
  double2* xch = (double2*)(slc + 8);                  // [8][4]   pair exchange (LANES = 64 only)
  double2* Xs = xch + (LANES == 64 ? 32 : 0);          // [nk][LF] X of this x-mode (a.xs)
  const long q = blockIdx.x / a.nch;
  const int ch = blockIdx.x % a.nch;
  PINT_ASSERT(q < a.Qb && a.L <= LF && a.k <= 8 && a.nk <= NKC && blockDim.x == FCfg<LANES>::THREADS);
  static_assert(!TMA || FTmem<C, LANES, NKC>::NEED <= FTmem<C, LANES, NKC>::COLS, "TMEM columns");
  const int NG = (int)(a.N / FG);                      // line stride of a group
  const int NGL = HALF ? NG / 2 + 1 : NG;               // groups solved (half spectrum: i <= N/16)
  const int g0 = ch * a.gpc, g1 = min(g0 + a.gpc, NGL);
  const int warp = threadIdx.x >> 5;
  const int line = LANES == 64 ? warp >> 1 : warp, half = LANES == 64 ? warp & 1 : 0;
  const double2* Xg = a.X + q * 8 * LF;
  const double2* Xq = Xg;
  if (!TMA && a.xs) {   // X is the same for every frequency group of this x-mode: stage it once
    for (int e = threadIdx.x; e < a.nk * LF; e += FCfg<LANES>::THREADS) cp_async16(&Xs[e], &Xg[e]);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    cp_async_wait0();
    __syncthreads();
    Xq = Xs;
  }
  uint32_t tacc = 0, txs = 0;
  if constexpr (TMA) {
    tacc = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * FTmem<C, LANES, NKC>::RPT * 24);
    uint32_t z[24];
#pragma unroll
    for (int j = 0; j < 24; ++j) z[j] = 0u;
#pragma unroll
    for (int rr = 0; rr < FTmem<C, LANES, NKC>::RPT; ++rr) tmem_st24(tacc + 24 * rr, z);
    // X of this x-mode (the same for every frequency group) into this thread's TMEM columns
    constexpr int XC = 4 * NKC, RPTX = FTmem<C, LANES, NKC>::RPT;
    txs = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)FTmem<C, LANES, NKC>::WCOLS + (uint32_t)((warp >> 2) * RPTX * XC);
#pragma unroll
    for (int rr = 0; rr < RPTX; ++rr) {
      const int y = threadIdx.x + FCfg<LANES>::THREADS * rr;
      if (LF < FCfg<LANES>::THREADS && y >= LF) break;          // warp-uniform
      uint32_t xw[XC];
#pragma unroll
      for (int t = 0; t < NKC; ++t) tw_putn<XC>(xw, t, Xg[t * LF + y]);
      tmem_stn<XC>(txs + XC * rr, xw);
    }
    tmem_wait_st();
  }
  fused_stage_lc(a, slc, q, g0);
  if (!STORE_W && !TMA)
    for (int y = threadIdx.x; y < LF; y += FCfg<LANES>::THREADS)
      for (int j = 0; j < a.k; ++j) acc[j * LF + y] = make_double2(0.0, 0.0);
  fused_rows<C, LANES, false, false, false, NKC>(a, Hs, acc, Xq, q, g0 - 1, true);   // synthesise group g0
  cp_async_wait0();
  __syncthreads();
  unsigned long long sp[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // PINT_SOLVE_PROF: cycles per solve sub-phase
#ifdef PINT_FUSED_PROF
  unsigned long long pt[4] = {0, 0, 0, 0};
#define PINT_TS(v) long long v = clock64()
#else
#define PINT_TS(v)
#endif
  for (int i = g0; i < g1; ++i) {
    PINT_TS(t0);
    {
      const LineConst& lcl = slc[line];
      if (cabs2(lcl.u) >= FUSED_AF_U2)
        fused_solve<C, LANES, STORE_W, true>(a, Hs + line * LF, lcl, xch + 4 * line, q, i + (long)NG * line, half, 1 + line, sp);
      else
        fused_solve<C, LANES, STORE_W, false>(a, Hs + line * LF, lcl, xch + 4 * line, q, i + (long)NG * line, half, 1 + line, sp);
    }
    PINT_TS(t1);
    __syncthreads();
    PINT_TS(t2);
    const bool next = i + 1 < g1;
    if (next) fused_stage_lc(a, slc, q, i + 1);
    fused_rows<C, LANES, !STORE_W, TMA, HALF, NKC, TMA>(a, Hs, acc, Xq, q, i, next, tacc, txs);
    if constexpr (TMA) tmem_wait_st();
    cp_async_wait0();
    PINT_TS(t3);
    __syncthreads();
#ifdef PINT_FUSED_PROF
    const long long t4 = clock64();
    pt[0] += t1 - t0; pt[1] += t2 - t1; pt[2] += t3 - t2; pt[3] += t4 - t3;
#endif
  }
#ifdef PINT_FUSED_PROF
  if ((threadIdx.x & 31) == 0 && a.prof) {
    const int w = threadIdx.x >> 5;
    for (int j = 0; j < 4; ++j) {
      atomicAdd(&a.prof[j], pt[j]);
      atomicAdd(&a.prof[4 + 4 * w + j], pt[j]);
    }
#ifdef PINT_SOLVE_PROF
    for (int j = 0; j < 9; ++j) atomicAdd(&a.prof[48 + j], sp[j]);
    atomicAdd(&a.prof[57], (unsigned long long)(g1 - g0));
#endif
  }
#endif
  (void)sp;
  if (!STORE_W) {
    double2* P = a.P + ((q * a.nch + ch) * a.k) * LF;
    if constexpr (TMA) {
#pragma unroll
      for (int rr = 0; rr < FTmem<C, LANES, NKC>::RPT; ++rr) {
        const int y = threadIdx.x + FCfg<LANES>::THREADS * rr;
        if (LF < FCfg<LANES>::THREADS && y >= LF) break;          // warp-uniform (LF % 32 == 0)
        uint32_t w[24];
        tmem_ld24(tacc + 24 * rr, w);
#pragma unroll
        for (int r = 2; r < 8; ++r) {
          const int j = r - 8 + a.k;
          if (j >= 0) P[j * LF + y] = tw_get(w, r - 2);
        }
      }
    } else {
      for (int y = threadIdx.x; y < LF; y += FCfg<LANES>::THREADS)
        for (int j = 0; j < a.k; ++j) P[j * LF + y] = acc[j * LF + y];
    }
  }
}

template <int C, int LANES, int NKC>
__device__ __forceinline__ uint32_t fused_tmem_alloc(uint32_t* tbase_smem) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(tbase_smem)), "n"(FTmem<C, LANES, NKC>::COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  return *tbase_smem;
}
template <int C, int LANES, int NKC>
__device__ __forceinline__ void fused_tmem_free(uint32_t tbase) {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n"
                 :: "r"(tbase), "n"(FTmem<C, LANES, NKC>::COLS) : "memory");
}

template <int C, int LANES, bool STORE_W, bool TM, bool HALF = false, int NKC = 8>
__global__ void __launch_bounds__(FCfg<LANES>::THREADS, FCfg<LANES>::minb(C)) wr_fused_kernel(const FusedArgs a) {
  extern __shared__ double2 fsm[];
  constexpr bool TMA = TM && !STORE_W;
  if (a.skip && *(volatile const int*)a.skip) return;   // device-side loop already stopped
  if (a.upd_reset && blockIdx.x == 0 && threadIdx.x == 0) *a.upd_reset = 0ull;
  __shared__ uint32_t tbase_s;
  uint32_t tbase = 0;
  if constexpr (TMA) tbase = fused_tmem_alloc<C, LANES, NKC>(&tbase_s);
  fused_iteration<C, LANES, STORE_W, TM, HALF, NKC>(a, fsm, tbase);
  if constexpr (TMA) fused_tmem_free<C, LANES, NKC>(tbase);
}


// ---------------------------------------------------------------------------------------------
// Fully modal variant (PINT_FLAG_MODAL): with the DST applied along y as well
// (hoisted like the DST-x), every (x-mode q, y-mode j) is a scalar problem and Step 2 is a division,
// W_p = H_p / (sigma_{p,q} + mu_j), mu_j = 2 - 2 cos(j pi h_y) (eigenvalues of tridiag(-1, 2, -1)):
// the shift is never added to 2, so the division is shift-accurate by construction.  One warp per
// mode; lane l takes the frequency groups i = l, l + 32, ...: synthesis (twiddle + DFT8), division,
// window (DFT8 + k twiddled accumulations) in registers; a warp reduction of the k window sums.
// No shared memory, no barriers; the finish kernel is the line path's (y index = mode j).
// STORE_W: write W (every p) into the tile layout [q][jb][N][WB] for materialisation.
#ifndef PINT_MODAL_MINB
#define PINT_MODAL_MINB 2
#endif
// z / b with 1/|b|^2 from the hardware reciprocal estimate and two Newton steps (quadratic: the
// estimate's ~2^-23 relative error becomes ~2^-92, below the final rounding), without the IEEE
// division's special-case path; |b|^2 is a normal number here (sigma_p + c is bounded away from 0)
__device__ __forceinline__ double2 cdiv_nr(double2 z, double2 b) {
  const double m = fma(b.x, b.x, b.y * b.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m));
  r = fma(r, fma(-m, r, 1.0), r);
  r = fma(r, fma(-m, r, 1.0), r);
  return make_double2(fma(z.x, b.x, z.y * b.y) * r, fma(z.y, b.x, -z.x * b.y) * r);
}

template <bool STORE_W>
__global__ void __launch_bounds__(256, PINT_MODAL_MINB) wr_modal_kernel(const FusedArgs a) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (a.skip && *(volatile const int*)a.skip) return;   // device-side loop already stopped
  if (a.upd_reset && blockIdx.x == 0 && threadIdx.x == 0) *a.upd_reset = 0ull;
  if (gw >= a.Qb * (long)a.L) return;                       // warp-uniform
  const long q = gw / a.L;
  const int j = (int)(gw % a.L);
  const int N = (int)a.N, k = a.k, nk = a.nk;
  const int NG = N / FG;
  const int NGL = (a.half && !STORE_W) ? NG / 2 + 1 : NG;
  double2 X[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) X[t] = (t < nk) ? a.X[(q * 8 + t) * a.Lf + j] : make_double2(0.0, 0.0);
  const double cm = __ldg(&a.sig_q[q]) + __ldg(&a.mu[j]);
  double2 acc[6];
#pragma unroll
  for (int l = 0; l < 6; ++l) acc[l] = make_double2(0.0, 0.0);
  for (int i = lane; i < NGL; i += 32) {
    double2 z[8];
    z[0] = X[0];
#pragma unroll
    for (int t = 1; t < 8; ++t) z[t] = (t < nk) ? cmul(X[t], __ldg(&a.tw[t * i])) : make_double2(0.0, 0.0);
    dft8<-1>(z);                                            // H_{i + (N/8) s}
    for (int dd = 0; dd < a.ndense; ++dd) {
      const double2 g = __ldg(&a.src[((long)__ldg(&a.dsrc[dd]) * a.Qb + q) * a.Lpad + j]);
      const double2* ch = a.chat + (long)dd * N + i;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) z[s2] = cfma(__ldg(&ch[s2 * NG]), g, z[s2]);
    }
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) {                        // Step 2: W_p = H_p / (sigma_p + c)
      const double2 sp = __ldg(&a.sig_p[i + s2 * NG]);
      z[s2] = cdiv_nr(z[s2], make_double2(sp.x + cm, sp.y));
    }
    if constexpr (STORE_W) {
      double2* Wq = a.W + ((q * a.NB + j / a.WB) * a.N) * a.WB + j % a.WB;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) Wq[(long)(i + s2 * NG) * a.WB] = z[s2];
    } else {
      dft8<+1>(z);                                          // Y_r = sum_s e^{+2 pi i rs/8} W_{i + (N/8) s}
      const double hw = (i == 0 || 16 * i == N) ? 1.0 : 2.0;
#pragma unroll
      for (int r = 2; r < 8; ++r) {
        const int l = r - 8 + k;                            // window level N - 8 + r = N - k + l
        if (l >= 0) {
          double2 w = __ldg(&a.tw[((N - 8 + r) * i) & (N - 1)]);
          w.y = -w.y;
          acc[r - 2] = cadd(acc[r - 2], wcontrib(z[r], w, a.half, hw));
        }
      }
    }
  }
  if constexpr (!STORE_W) {
#pragma unroll
    for (int r = 2; r < 8; ++r)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[r - 2].x += __shfl_xor_sync(0xffffffffu, acc[r - 2].x, o);
        acc[r - 2].y += __shfl_xor_sync(0xffffffffu, acc[r - 2].y, o);
      }
    if (lane == 0) {
#pragma unroll
      for (int r = 2; r < 8; ++r) {
        const int l = r - 8 + k;
        if (l >= 0) a.P[(q * k + l) * a.Lf + j] = acc[r - 2];
      }
    }
  }
}

// many chunks (nch > 16, 1D problems): one warp per row sums the chunks' window sums (lanes over
// chunks, a shuffle tree per window level j < k), then the warp runs the finish step of the row with
// lane j on window level j (U_j, its update, the new wrap state) and lane t on X_t (the U_j reach it
// by shuffles): every load of the step is issued by some lane at once (lane 0 alone serialised ~8 L2
// round trips per row: the finish phase of C2 took 12 us of a 30 us iteration)
__device__ __forceinline__ void reduce_finish_rows(const FinishArgs& a) {
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  double updl = 0.0;
  bool nonfinite = false;
  for (long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5; gw < a.Qb * (long)a.Lf;
       gw += ((long)gridDim.x * blockDim.x) >> 5) {
    const long q = gw / a.Lf;
    const int y = (int)(gw % a.Lf);
    const bool live = y < a.L;
    // ---- window sums S_j (all lanes hold all S_j after the xor trees) ----
    double2 S[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      S[j] = make_double2(0.0, 0.0);
      if (j < k) {                                           // warp-uniform
        const double2* Pj = a.P + (q * a.pstride * k + j) * a.Lf + y;
        const long cs = (long)k * a.Lf;                      // chunk stride
        double2 s0 = make_double2(0.0, 0.0), s1 = s0;
        int c = lane;
        for (; c + 32 < a.nch; c += 64) { s0 = cadd(s0, Pj[c * cs]); s1 = cadd(s1, Pj[(c + 32) * cs]); }
        if (c < a.nch) s0 = cadd(s0, Pj[c * cs]);
        double2 sv = cadd(s0, s1);
        for (int o = 16; o > 0; o >>= 1) {
          sv.x += __shfl_xor_sync(0xffffffffu, sv.x, o);
          sv.y += __shfl_xor_sync(0xffffffffu, sv.y, o);
        }
        S[j] = sv;
      }
    }
    // ---- lane j < k: U_j = kappa^{-n/N} S_j (n = N - k + j), update, new wrap state ----
    const long wb = (q * a.NB + y / a.WB) * k * a.WB + (y % a.WB);
    double2 Uj = make_double2(0.0, 0.0);
    if (lane < k && live) {
      double2 Sj = S[0];
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (lane == j) Sj = S[j];
      Uj = cscale(Sj, __ldg(&a.igs[a.N - k + lane]));
      const double dd = sqrt(cabs2(csub(Uj, a.wrap_old[wb + lane * a.WB])));
      if (!(dd <= 1.7976931348623157e308)) nonfinite = true;
      updl = fmax(updl, dd);
      a.wrap_new[wb + lane * a.WB] = Uj;
    }
    double2 U[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      U[j].x = __shfl_sync(0xffffffffu, Uj.x, j);
      U[j].y = __shfl_sync(0xffffffffu, Uj.y, j);
    }
    // ---- lane t < 8: X_t = Gamma_t h^2/N [ F_static(t) + (kappa/tau) sum_jw omega_jw U^{N+t-jw} ] ----
    if (lane < 8) {
      const int t = lane;
      double2 F = make_double2(0.0, 0.0);
      if (t < a.nk && live) {
        for (int i = 0; i < a.nsparse; ++i) {
          const int sidx = __ldg(&a.spar[i]);
          F = cfmar(__ldg(&a.src[((long)sidx * a.Qb + q) * a.Lpad + y]), __ldg(&a.coef[(long)sidx * a.N + t]), F);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)                          // window entry j = level N-k+j, jw = k+t-j
          if (j >= t && j < k) F = cfmar(U[j], __ldg(&a.wk[k + t - j]), F);
        F = cscale(F, __ldg(&a.gsf[t]));
      }
      a.X[(q * 8 + t) * a.Lf + y] = F;
    }
  }
  if (nonfinite) updl = __longlong_as_double(0x7ff0000000000000LL);
  block_max_atomic(updl, a.upd);
}
__global__ void __launch_bounds__(TPB) wr_reduce_finish_kernel(const FinishArgs a) {
  if (a.skip && *(volatile const int*)a.skip) return;
  reduce_finish_rows(a);
  finish_loop_tail(a.ctl, a.arrive, a.hnd, a.upd);
}


__device__ __forceinline__ void finish_rows(const FinishArgs& a, int mode) {
  double updl = 0.0;
  bool nonfinite = false;
  const long total = a.Qb * a.Lf;
  const int k = a.k;
  for (long e = blockIdx.x * (long)TPB + threadIdx.x; e < total; e += (long)gridDim.x * TPB) {
    const long q = e / a.Lf;
    const int y = (int)(e % a.Lf);
    const bool live = y < a.L;
    const long wb = (q * a.NB + y / a.WB) * k * a.WB + (y % a.WB);   // + j * WB
    double2 U[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      U[j] = make_double2(0.0, 0.0);
      if (j < k && live) {
        if (mode == FIN_PARTIALS) {
          double2 s = make_double2(0.0, 0.0);
          for (int c = 0; c < a.nch; ++c) s = cadd(s, a.P[((q * a.pstride + c) * k + j) * a.Lf + y]);
          U[j] = cscale(s, __ldg(&a.igs[a.N - k + j]));
          const double2 o = a.wrap_old[wb + j * a.WB];
          const double dd = sqrt(cabs2(csub(U[j], o)));
          if (!(dd <= 1.7976931348623157e308)) nonfinite = true;
          updl = fmax(updl, dd);
        } else if (mode == FIN_FROM_WRAP) {
          U[j] = a.wrap_old[wb + j * a.WB];
        } else if (mode == FIN_FROM_V) {
          U[j] = __ldg(&a.src[q * a.Lpad + y]);             // source 0 is v
        }
        if (mode != FIN_FROM_WRAP) a.wrap_new[wb + j * a.WB] = U[j];
      }
    }
    // X_t = Gamma_t h^2/N [ F_static(t) + (kappa/tau) sum_{jw=t+1}^{k} omega_jw U^{N+t-jw} ]
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      double2 F = make_double2(0.0, 0.0);
      if (t < a.nk && live) {
        for (int i = 0; i < a.nsparse; ++i) {
          const int s = __ldg(&a.spar[i]);
          F = cfmar(__ldg(&a.src[((long)s * a.Qb + q) * a.Lpad + y]), __ldg(&a.coef[(long)s * a.N + t]), F);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)                          // window entry j = level N-k+j, jw = k+t-j
          if (j >= t && j < k) F = cfmar(U[j], __ldg(&a.wk[k + t - j]), F);
        F = cscale(F, __ldg(&a.gsf[t]));
      }
      a.X[(q * 8 + t) * a.Lf + y] = F;
    }
  }
  if (mode == FIN_PARTIALS) {
    if (nonfinite) updl = __longlong_as_double(0x7ff0000000000000LL);
    block_max_atomic(updl, a.upd);
  }
}
__global__ void __launch_bounds__(TPB) wr_finish_kernel(const FinishArgs a, int mode) {
  if (a.skip && *(volatile const int*)a.skip) return;
  finish_rows(a, mode);
  if (mode == FIN_PARTIALS) finish_loop_tail(a.ctl, a.arrive, a.hnd, a.upd);
}

// ---- the whole WR loop as ONE cooperative kernel (small problems: every (x-mode, chunk) CTA resident) ----
// Per iteration: the fused iteration of this CTA (Steps 1-3, window partial sums -> P), a grid barrier,
// the finish step distributed over all CTAs (window of U_m, monitor, X of the next iteration), a grid
// barrier whose last block applies pint_wr_solve's stopping rule.  No kernel launch, no graph node
// and no host round trip per iteration.
template <int C, int NKC>
__global__ void __launch_bounds__(FG * 32, 1) wr_loop_kernel(const LoopKArgs L) {
  extern __shared__ double2 fsm[];
  __shared__ uint32_t tbase_s;
  const uint32_t tbase = fused_tmem_alloc<C, 32, NKC>(&tbase_s);
#ifdef PINT_FUSED_PROF
#define PINT_GT(v) unsigned long long v; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#else
#define PINT_GT(v)
#endif
  for (int h = 0;; h ^= 1) {
    PINT_GT(g0);
    fused_iteration<C, 32, false, true, false, NKC>(L.fa[h], fsm, tbase);
    PINT_GT(g1);
    grid_sync(L.bar, nullptr, nullptr);
    PINT_GT(g2);
    // warp per row when the chunks are many or every row gets its own warp (thread per row left the
    // C1 finish to block 0 alone: 8 sequential partial loads per level while 7 blocks waited)
    if (L.fin[h].nch > 16 || L.fin[h].Qb * (long)L.fin[h].Lf <= (long)gridDim.x * (blockDim.x / 32))
      reduce_finish_rows(L.fin[h]);
    else
      finish_rows(L.fin[h], FIN_PARTIALS);
    PINT_GT(g3);
    grid_sync(L.bar, L.ctl, L.fin[h].upd);
    PINT_GT(g4);
#ifdef PINT_FUSED_PROF
    if (threadIdx.x == 0 && L.fa[h].prof) {   // ns per phase, summed over blocks and iterations
      unsigned long long* pr = L.fa[h].prof + 40;
      atomicAdd(&pr[0], g1 - g0); atomicAdd(&pr[1], g2 - g1); atomicAdd(&pr[2], g3 - g2);
      atomicAdd(&pr[3], g4 - g3); atomicAdd(&pr[4], 1ull);
    }
#endif
    if (*(volatile int*)&L.ctl->done) break;
  }
  fused_tmem_free<C, 32, NKC>(tbase);
}

// ---- plan time: per-line constants ----
// C = rows per lane, CS = rows per sub-chain
__global__ void line_const_kernel(LineConst* lc, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int CS,
                                  int L) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < N * Qb; e += (long)gridDim.x * blockDim.x) {
    const long q = e / N, p = e % N;
    const double2 sp = sig_p[p];
    const double2 sig = make_double2(sp.x + sig_q[q], sp.y);
    const double2 s = csqrt_(cmul(sig, make_double2(4.0 + sig.x, sig.y)));
    const double2 t1 = cscale(cadd(sig, s), 0.5), t2 = cscale(csub(sig, s), 0.5);
    const double2 tb = cabs2(t1) >= cabs2(t2) ? t1 : t2;
    const double2 ts = cdiv(make_double2(-sig.x, -sig.y), tb);          // tb * ts = -sigma
    const double2 rb = make_double2(1.0 + tb.x, tb.y), rs = make_double2(1.0 + ts.x, ts.y);
    const double2 tt = cabs2(rb) > cabs2(rs) ? tb : ts;
    LineConst c;
    c.rr = make_double2(1.0 + tt.x, tt.y);                              // r = 1/a, |r| > 1
    c.u = cdiv(tt, c.rr);                                               // u = 1 - a
    c.uc[0] = upow(c.u, C);
    for (int i = 1; i < 8; ++i) c.uc[i] = uprod(c.uc[i - 1], c.uc[i - 1]);
    c.uh = upow(c.u, CS);
    c.rrh = make_double2(1.0, 0.0);
    for (int i = 0; i < CS; ++i) c.rrh = cmul(c.rrh, c.rr);
    const double2 u2L = upow(c.u, 2L * L + 2);
    c.ru2L = cdiv(make_double2(1.0, 0.0), u2L);
    c.uE = upow(c.u, (2L * L + 2) % C);
    c.ap[0] = one_minus(c.u);
    for (int i = 1; i < 5; ++i) c.ap[i] = cmul(c.ap[i - 1], c.ap[i - 1]);
    const double la = 0.5 * log(cabs2(one_minus(c.u)));                // log|a| < 0
    const double thr = -41.44653167389282 + 0.5 * log(cabs2(u2L));      // log(1e-18 |1 - a^{2L+2}|)
    c.tl = la < 0.0 ? thr / la : INFINITY;
    c.nlev = 0;
    while (c.nlev < 5 && cabs2(one_minus(c.uc[c.nlev])) >= 0x1p-128) ++c.nlev;
    c.pad1 = 0;
    lc[e] = c;
  }
}
#endif  // PINT_DEFINE_FUSED_KERNELS

}  // namespace pint
