// tpass.cuh — the time-axis pass ("T-pass") of one WR iteration, fused per spatial tile.
//
// One CTA owns one tile: all N time levels of WB = 4096/N contiguous spatial columns
// (64 KB complex128, contiguous in the blocked layout [q][yb][n][WB]).  Per iteration
// (mode FREQ -> H):
//   W_m --(inverse time FFT, unscale: Step 3)--> U_m            [registers]
//   update |U_m - U_{m-1}| on the wrap window n = N-k+1..N; store the new wrap state
//   F_m = f̄ + tau^-a (sum_{j<n} w_j) v + kappa-wrap(U_m)   (eqn:BDF-k-F / eq:BDF-subdiff-F)
//   H_{m+1} = (h^2/N) FFT(Gamma F_m)                           (Step 1)
// HBM traffic: read 16 B + write 16 B per space-time unknown.
//
// CQ (subdiffusion) wrap: kappa Wup U = (C(kappa) U - C(-kappa) U) / 2 with C(c) the
// c-circulant of omega_0..omega_{N-1} (B_k(kappa) = C(kappa)), both
// diagonalised by scaled DFTs (Lemma 3.2); in the frequency domain
//   H = (h^2/N) FFT(Gamma F_static) + (h^2/2 tau^a) [ D W - V^{-1} Theta^{-1} V D' V^{-1} Theta V W ],
//   Theta = diag(e^{i pi n/N}), D' = eigenvalues of C(-kappa).  DESIGN.md "CQ wrap".
#pragma once
#include "fft.cuh"

namespace pint {

#ifndef PINT_PRUNED_MINB
#define PINT_PRUNED_MINB 3
#endif
#ifndef PINT_CQ_MINB
#define PINT_CQ_MINB 2
#endif
#ifndef PINT_TPASS_MINB
#define PINT_TPASS_MINB 2
#endif
#ifndef CQ_SV
#define CQ_SV 2   // CQ T-pass: sources whose column values stay in registers for the whole tile
#endif

enum { IN_FREQ = 0, IN_TIME_V = 1, IN_TIME_ZERO = 2, IN_TIME_BUF = 3 };
enum { OUT_H = 0, OUT_U = 1 };

struct TPassArgs {
  const double2* in;        // W (FREQ) or U (TIME_BUF), tile-blocked layout
  double2* out;             // H (OUT_H) or U (OUT_U); may alias `in` (tile-local in place)
  const double2* wrap_old;  // [ntiles][k][WB] last-k levels of U_{m-1} (FREQ mode monitor)
  double2* wrap_new;        // [ntiles][k][WB] last-k levels of U_m
  const double2* src;       // [S][ntiles][WB] spatial source vectors (g_r, Av, v) in tile layout
  const double* coef;       // [S][N] time coefficients of F_static
  const int* nhi;           // [S] coef[s][n] == 0 for n >= nhi[s]
  int S;
  const double2* vsrc;      // the v source (for IN_TIME_V), tile layout [ntiles][WB]
  const double2* tw;        // [N] exp(-2 pi i m/N)
  const double* gsf;        // [N] kappa^{n/N} h^2/N      (forward scale, heat)
  const double* igs;        // [N] kappa^{-n/N}           (unscale)
  const double* gsN;        // [N] kappa^{n/N} / N        (CQ time-mode bootstrap)
  const double* wk;         // [k+1] (kappa/tau) omega_j  (heat wrap)
  int k;
  // CQ tables
  const double2* dh;        // [N] (h^2 / (2 tau^a)) d_p
  const double2* dpr;       // [N] d'_p (eigenvalues of C(-kappa))
  const double2* thp;       // [N] theta^n / N
  const double2* thm;       // [N] -(h^2/(2 N tau^a)) theta^{-n}
  const double* gsfq;       // [N] kappa^{n/N} h^2/N (CQ static part)
  unsigned long long* upd;  // max |update| as ordered bits
  int nmax;                 // max_s nhi[s]: F_static(n) == 0 for n >= nmax
  int prefetch;             // 1: bulk-prefetch the next tile into L2
  // pruned heat T-pass: sources with coefficients beyond n = 15 ("dense") are synthesised in the
  // frequency domain: H += sum_d chat[d][p] * src[dsrc[d]]; sparse sources enter X_0..X_15
  int nsparse;              // number of sparse sources (listed first in spar[])
  const int* spar;          // [nsparse] source indices with nhi <= 16
  int ndense;
  const int* dsrc;          // [ndense] source indices with nhi > 16
  const double2* chat;      // [ndense][N]  sum_n gsf[n] coef[s][n] e^{-2 pi i n p / N}
  int nk;                   // X_n = 0 for n >= nk (nk = max(k, max sparse nhi) <= 16)
  const double2* fdense;    // optional dense right-hand side [N][M] in the tile layout, added to
                            // F_static (Newton inner solves: the residual R; set nmax = N)
  double2* ufull;           // full-array update monitor (PINT_FLAG_FULL_UPDATE_NORM, CQ plans): U_{m-1}
                            // of every level in the tile layout; FREQ mode compares U_m with it and
                            // overwrites it with U_m, time-domain (bootstrap) modes store U_0
};

// |U - ufull[e]| into (upd, nonfinite) and ufull[e] = U (FREQ mode); store only (bootstrap modes)
template <bool CMP>
__device__ __forceinline__ void full_monitor(double2* ufull, long e, double2 U, double& upd, bool& nonfinite) {
  if constexpr (CMP) {
    const double d = sqrt(cabs2(csub(U, ufull[e])));
    if (!(d <= 1.7976931348623157e308)) nonfinite = true;
    upd = fmax(upd, d);
  }
  ufull[e] = U;
}

// table load that the compiler may not hoist above barriers (bounds live ranges in the CQ path)
template <class T> __device__ __forceinline__ T ldt(const T* p) { return *(volatile const T*)p; }
__device__ __forceinline__ double2 ldt(const double2* p) {
  double2 r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double ldt(const double* p) {
  double r;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// L2 eviction-priority policies (createpolicy) for loads/stores with an explicit cache hint
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_hint(const double2* ptr, unsigned long long pol) {
  double2 r;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_hint(double2* ptr, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void prefetch_l2_t(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void block_max_atomic(double x, unsigned long long* dst) {
  __shared__ double red[TPB / 32];
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  // NaN must survive: fmax drops NaN, so track it separately
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int i = 1; i < TPB / 32; ++i) m = fmax(m, red[i]);
    atomicMax(dst, (unsigned long long)__double_as_longlong(m));
  }
}

// F_static(n, c) = sum_s coef[s][n] * src[s][tile][c]; zero for n >= nmax.
// srcp = src + tile*WB + c, sstride = ntiles*WB (one spatial vector per source).
// FD: a.fdense is set (a template switch: the runtime test and the element index cost the CQ T-pass
// 15 % through register pressure, 8.3 -> 9.5 ms on C5)
template <bool FD>
__device__ __forceinline__ double2 static_rhs(const TPassArgs& a, const double2* srcp, long sstride, int N, int n,
                                              long e) {
  double2 f = make_double2(0.0, 0.0);
  if (n >= a.nmax) return f;
  for (int s = 0; s < a.S; ++s) f = cfmar(ldt(&srcp[s * sstride]), ldt(&a.coef[(long)s * N + n]), f);
  if constexpr (FD) f = cadd(f, ldt(&a.fdense[e]));
  return f;
}

template <int N, int MODE_IN, int MODE_OUT, bool CQ, bool FD = false>
__global__ void __launch_bounds__(TPB, CQ ? PINT_CQ_MINB : PINT_TPASS_MINB) tpass_kernel(const TPassArgs a, long ntiles) {
  using TM = TimeMap<N>;
  using FM = FreqMap<N>;
  constexpr int WB = TILE / N;
  extern __shared__ double2 sm[];

  const int k = a.k;
  const double2* tw = a.tw;
  const bool dense = a.nmax > TM::PL;   // F_static nonzero beyond the first PL levels
  double upd = 0.0;
  bool nonfinite = false;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  // tid re-read per tile through volatile asm: keeps the per-element table addresses (which
  // depend only on tid) from being hoisted out of the tile loop and spilled
  int tid;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const long base = tile * (long)TILE;
  if ((MODE_IN == IN_FREQ || MODE_IN == IN_TIME_BUF) && a.prefetch) {
    const long nt = tile + gridDim.x;
    if (tid < 4 && nt < ntiles) prefetch_l2_t(a.in + nt * (long)TILE + tid * (TILE / 4), TILE / 4 * 16);
  }
  double2 v[16];
  // D W term: kept in registers only for the time-domain bootstrap (W computed in-kernel);
  // in FREQ mode W is re-read from the (untouched, L2-resident) input tile at the end.
  constexpr bool KEEP_DW = CQ && (MODE_IN != IN_FREQ);
  double2 dw[KEEP_DW ? 16 : 1];

  // ---------------- input ----------------
  if constexpr (MODE_IN == IN_FREQ) {
    if constexpr (CQ && MODE_OUT == OUT_H) {
      // W is re-read for the D W term at the end of the tile: keep it in L2 until then
      const unsigned long long keep = l2_evict_last();
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = ld_hint(&a.in[base + FM::e(t, tid)], keep);
    } else {
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = a.in[base + FM::e(t, tid)];
    }
    run_passes<N, +1, false>(v, sm, tw, tid);        // u = V W  (unnormalised inverse DFT)
  } else {
    // time-domain input U (registers in TimeMap)
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) {
        const int r = j * TM::RL + s;
        if constexpr (MODE_IN == IN_TIME_V) v[r] = __ldg(&a.vsrc[tile * WB + TM::c(j, tid)]);
        else if constexpr (MODE_IN == IN_TIME_ZERO) v[r] = make_double2(0.0, 0.0);
        else v[r] = a.in[base + TM::e(j, s, tid)];
      }
    if constexpr (CQ) {
      // W = FFT(Gamma U)/N, then u = V W (recomputed) so the frequency-domain path is shared
#pragma unroll
      for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
        for (int s = 0; s < TM::RL; ++s) v[j * TM::RL + s] = cscale(v[j * TM::RL + s], ldt(&a.gsN[TM::n(j, s, tid)]));
      run_passes<N, -1, true>(v, sm, tw, tid);
      if constexpr (KEEP_DW) {
#pragma unroll
        for (int t = 0; t < 16; ++t) dw[t] = cmul(v[t], ldt(&a.dh[FM::p(t, tid)]));
      }
      run_passes<N, +1, false>(v, sm, tw, tid);
    }
    // heat time modes: v holds U itself (HAVE_U_DIRECT below)
  }

  // ---------------- U_m = Gamma^{-1} u ; wrap window ----------------
  // v holds u (FREQ or CQ time modes) or U (heat time modes).
  constexpr bool HAVE_U_DIRECT = (MODE_IN != IN_FREQ) && !CQ;
  if constexpr (MODE_OUT == OUT_U) {
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) {
        const int r = j * TM::RL + s;
        const double2 U = HAVE_U_DIRECT ? v[r] : cscale(v[r], ldt(&a.igs[TM::n(j, s, tid)]));
        a.out[base + TM::e(j, s, tid)] = U;
      }
    continue;
  }

  if (a.ufull) {   // full-array monitor: every level of U_m
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) {
        const int r = j * TM::RL + s;
        const double2 U = HAVE_U_DIRECT ? v[r] : cscale(v[r], ldt(&a.igs[TM::n(j, s, tid)]));
        full_monitor<MODE_IN == IN_FREQ>(a.ufull, base + TM::e(j, s, tid), U, upd, nonfinite);
      }
  }

  __syncthreads();   // sm free: all readers of the last exchange are done
  double2* sW = sm;  // [k][WB] wrap window values of U_m
#pragma unroll
  for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
    for (int s = 0; s < TM::RL; ++s) {
      const int n = TM::n(j, s, tid);
      if ((s == TM::RL - 1 || TM::PL < 8) && n >= N - k) {
        const int r = j * TM::RL + s, c = TM::c(j, tid), jj = n - (N - k);
        const double2 U = HAVE_U_DIRECT ? v[r] : cscale(v[r], ldt(&a.igs[n]));
        const long wi = (tile * k + jj) * WB + c;
        if constexpr (MODE_IN == IN_FREQ) {
          const double2 o = a.wrap_old[wi];
          const double d = sqrt(cabs2(csub(U, o)));
          if (!(d <= 1.7976931348623157e308)) nonfinite = true;
          upd = fmax(upd, d);
        }
        a.wrap_new[wi] = U;
        sW[jj * WB + c] = U;
      }
    }
  __syncthreads();

  if constexpr (!CQ) {
    // ---------------- heat: F = F_static + wrap ; X = Gamma F h^2/N ----------------
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) {
        const int n = TM::n(j, s, tid), c = TM::c(j, tid);
        const int r = j * TM::RL + s;
        // F_static is zero for n >= nmax; with nmax <= PL only s == 0 slots can be nonzero
        const bool live = (s == 0) || dense || (TM::PL < 8);
        double2 F = make_double2(0.0, 0.0);
        if (live) F = static_rhs<FD>(a, a.src + tile * WB + c, ntiles * WB, N, n, base + TM::e(j, s, tid));
        if ((s == 0 || TM::PL < 8) && n < k) {
          // (kappa/tau) sum_{j=n+1}^{k} omega_j U_m^{N+n-j} (0-based levels), window index k+n-j
          for (int jw = n + 1; jw <= k; ++jw) F = cfmar(sW[(k + n - jw) * WB + c], __ldg(&a.wk[jw]), F);
        }
        v[r] = live ? cscale(F, __ldg(&a.gsf[n])) : F;
      }
    run_passes<N, -1, true>(v, sm, tw, tid);   // H = (h^2/N) FFT(Gamma F)
  } else {
    // ---------------- CQ ----------------
    // z = V^{-1} Theta u
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) v[j * TM::RL + s] = cmul(v[j * TM::RL + s], ldt(&a.thp[TM::n(j, s, tid)]));
    run_passes<N, -1, true>(v, sm, tw, tid);
    // s = V (D' z)
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = cmul(v[t], ldt(&a.dpr[FM::p(t, tid)]));
    run_passes<N, +1, false>(v, sm, tw, tid);
    // X = Gamma F_static h^2/N - (h^2/(2 N tau^a)) Theta^{-1} s.  A thread's column is the same for
    // every element (TPB % WB == 0): the first CQ_SV source values are loaded once per tile.
    static_assert(TPB % WB == 0, "fixed column per thread");
    const int cc = tid % WB;
    double2 sv[CQ_SV];
#pragma unroll
    for (int q = 0; q < CQ_SV; ++q) sv[q] = q < a.S ? ldt(&a.src[(long)q * ntiles * WB + tile * WB + cc]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s = 0; s < TM::RL; ++s) {
        const int n = TM::n(j, s, tid);
        double2 F = make_double2(0.0, 0.0);
        if (n < a.nmax) {
#pragma unroll
          for (int q = 0; q < CQ_SV; ++q)
            if (q < a.S) F = cfmar(sv[q], ldt(&a.coef[(long)q * N + n]), F);
          for (int q = CQ_SV; q < a.S; ++q)
            F = cfmar(ldt(&a.src[(long)q * ntiles * WB + tile * WB + cc]), ldt(&a.coef[(long)q * N + n]), F);
          if constexpr (FD) F = cadd(F, ldt(&a.fdense[base + TM::e(j, s, tid)]));
        }
        const int r = j * TM::RL + s;
        v[r] = cfmar(F, ldt(&a.gsfq[n]), cmul(v[r], ldt(&a.thm[n])));
      }
    run_passes<N, -1, true>(v, sm, tw, tid);
    if constexpr (KEEP_DW) {
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = cadd(v[t], dw[t]);
    } else {
      const unsigned long long last = l2_evict_first();   // W's last use
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = cfma(ld_hint(&a.in[base + FM::e(t, tid)], last), ldt(&a.dh[FM::p(t, tid)]), v[t]);
    }
  }

  if constexpr (CQ) {
    // H is next read by the S-pass after the whole T-pass: do not let it displace the W tiles
    const unsigned long long stream = l2_evict_first();
#pragma unroll
    for (int t = 0; t < 16; ++t) st_hint(&a.out[base + FM::e(t, tid)], v[t], stream);
  } else {
#pragma unroll
    for (int t = 0; t < 16; ++t) a.out[base + FM::e(t, tid)] = v[t];
  }
  __syncthreads();   // smem reused by the next tile
  }  // tile loop

  if constexpr (MODE_IN == IN_FREQ) {
    // fmax drops NaN: report any non-finite update as +inf (orders above all finite bits)
    if (nonfinite) upd = __longlong_as_double(0x7ff0000000000000LL);
    block_max_atomic(upd, a.upd);
  }
}

// ---------------------------------------------------------------------------------------------
// CQ T-pass split in two kernels of two transforms each (mode FREQ -> H, no dense RHS).  The
// monolithic kernel above holds a tile through four transforms and the table applications and
// spills at the 128-register bound; each half below has the register shape of the heat T-pass.
// The product Z = D' V^{-1} Theta V W (frequency domain) goes through the H buffer:
//   A: W --V--> u --(window, monitor)--> Theta u --V^{-1}--> D' z = Z            (out = H buffer)
//   B: Z --V--> s; X = Gamma F_static h^2/N - (h^2/(2 N tau^a)) Theta^{-1} s --V^{-1}--> + D W = H
// HBM: A reads W, writes Z; B reads Z and W, writes H: 80 B/unknown instead of 32.
// ---------------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(TPB, PINT_TPASS_MINB) tpass_cq_a_kernel(const TPassArgs a, long ntiles) {
  using TM = TimeMap<N>;
  using FM = FreqMap<N>;
  constexpr int WB = TILE / N;
  extern __shared__ double2 sm[];
  const int k = a.k;
  double upd = 0.0;
  bool nonfinite = false;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int tid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    const long base = tile * (long)TILE;
    if (a.prefetch) {
      const long nt = tile + gridDim.x;
      if (tid < 4 && nt < ntiles) prefetch_l2_t(a.in + nt * (long)TILE + tid * (TILE / 4), TILE / 4 * 16);
    }
    double2 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = a.in[base + FM::e(t, tid)];
    run_passes<N, +1, false>(v, sm, a.tw, tid);          // u = V W
    if (a.ufull) {   // full-array monitor: every level of U_m
#pragma unroll
      for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
        for (int s2 = 0; s2 < TM::RL; ++s2)
          full_monitor<true>(a.ufull, base + TM::e(j, s2, tid), cscale(v[j * TM::RL + s2], __ldg(&a.igs[TM::n(j, s2, tid)])),
                             upd, nonfinite);
    }
    // window levels of U_m = Gamma^{-1} u: monitor and new wrap state
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s2 = 0; s2 < TM::RL; ++s2) {
        const int n = TM::n(j, s2, tid);
        if ((s2 == TM::RL - 1 || TM::PL < 8) && n >= N - k) {
          const double2 U = cscale(v[j * TM::RL + s2], __ldg(&a.igs[n]));
          const long wi = (tile * k + (n - (N - k))) * WB + TM::c(j, tid);
          const double d = sqrt(cabs2(csub(U, a.wrap_old[wi])));
          if (!(d <= 1.7976931348623157e308)) nonfinite = true;
          upd = fmax(upd, d);
          a.wrap_new[wi] = U;
        }
      }
    // Z = D' V^{-1} Theta u
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s2 = 0; s2 < TM::RL; ++s2) v[j * TM::RL + s2] = cmul(v[j * TM::RL + s2], __ldg(&a.thp[TM::n(j, s2, tid)]));
    run_passes<N, -1, true>(v, sm, a.tw, tid);
#pragma unroll
    for (int t = 0; t < 16; ++t) a.out[base + FM::e(t, tid)] = cmul(v[t], __ldg(&a.dpr[FM::p(t, tid)]));
    __syncthreads();   // smem reused by the next tile
  }
  if (nonfinite) upd = __longlong_as_double(0x7ff0000000000000LL);
  block_max_atomic(upd, a.upd);
}

// a.in = Z (may alias a.out), a.vsrc = W, a.chat = [S][N] spectra of the static sources:
// H = V^{-1}(-(h^2/(2 N tau^a)) Theta^{-1} V Z) + sum_s chat_s[p] src_s + D W
template <int N>
__global__ void __launch_bounds__(TPB, PINT_TPASS_MINB) tpass_cq_b_kernel(const TPassArgs a, long ntiles) {
  using TM = TimeMap<N>;
  using FM = FreqMap<N>;
  constexpr int WB = TILE / N;
  static_assert(TPB % WB == 0, "fixed column per thread");
  extern __shared__ double2 sm[];
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int tid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    const long base = tile * (long)TILE;
    // L2 bulk prefetch: the next tile's Z, and this tile's W (read only after both transforms)
    if (tid < 4) {
      const long nt = tile + gridDim.x;
      if (nt < ntiles) prefetch_l2_t(a.in + nt * (long)TILE + tid * (TILE / 4), TILE / 4 * 16);
    } else if (tid < 8) {
      prefetch_l2_t(a.vsrc + base + (tid - 4) * (TILE / 4), TILE / 4 * 16);
    }
    double2 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = a.in[base + FM::e(t, tid)];
    run_passes<N, +1, false>(v, sm, a.tw, tid);          // s = V Z
#pragma unroll
    for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
      for (int s2 = 0; s2 < TM::RL; ++s2) v[j * TM::RL + s2] = cmul(v[j * TM::RL + s2], __ldg(&a.thm[TM::n(j, s2, tid)]));
    run_passes<N, -1, true>(v, sm, a.tw, tid);
    const int cc = tid % WB;
    double2 sv[CQ_SV];
#pragma unroll
    for (int q = 0; q < CQ_SV; ++q) sv[q] = q < a.S ? __ldg(&a.src[(long)q * ntiles * WB + tile * WB + cc]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int p = FM::p(t, tid);
      double2 h = cfma(a.vsrc[base + FM::e(t, tid)], __ldg(&a.dh[p]), v[t]);
#pragma unroll
      for (int q = 0; q < CQ_SV; ++q)
        if (q < a.S) h = cfma(__ldg(&a.chat[(long)q * N + p]), sv[q], h);
      for (int q = CQ_SV; q < a.S; ++q)
        h = cfma(__ldg(&a.chat[(long)q * N + p]), __ldg(&a.src[(long)q * ntiles * WB + tile * WB + cc]), h);
      a.out[base + FM::e(t, tid)] = h;
    }
    __syncthreads();
  }
}

}  // namespace pint

namespace pint {

// ---------------------------------------------------------------------------------------------
// Pruned-FFT T-pass for heat (alpha = 1), mode FREQ -> H, N >= 512 (schedule 16.16.RL, PL = 256).
// The next iterate needs only the k window levels n in [N-k, N) of U_m, and
// X = Gamma F vanishes for n >= nk = max(k, nmax) <= 16.  Standard FFT pruning on the same
// Stockham passes (index maps derived in DESIGN.md "Pruned T-pass"):
//   inverse: pass 0 (radix 16, P = 1) in full, keeping the k outputs s0 in [16-k, 16) the window
//            needs; pass 1 only for the 16k butterflies (per tile) feeding the window, output
//            s1 = 15 only; pass 2 only the k window outputs (s2 = RL-1).
//   forward: with X supported on n < 16, passes 0 and 1 are broadcasts and pass 2 sees inputs
//            X_0..X_15: H_{i + (N/16) s} = DFT16_s( X_t w_N^{t i} ).
// ---------------------------------------------------------------------------------------------
template <int N, bool DENSE>
__global__ void __launch_bounds__(TPB, PINT_PRUNED_MINB) tpass_heat_pruned_kernel(const TPassArgs a, long ntiles) {
  static_assert(N >= 256 && N <= 4096, "16.16.RL schedule (RL = 1 for N = 256)");
  constexpr int WB = TILE / N;
  constexpr int NB16 = N / 16;          // radix-16 butterflies per column
  constexpr int RL = N / 256;
  constexpr int NBLK = N / 256;         // pass-1 blocks per column
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int k = a.k;
  const int nk = a.nk;                  // X_n = 0 for n >= nk (host guarantees nk <= 16)
  // pass-0 outputs s0 >= 16-k, slot (c, i0, j = s0-16+k): c*(9 NB16 + 1) + 9 i0 + j (k <= 8;
  // stride 9 and the +1 column skew keep the 16-byte stores/loads bank-conflict free)
  double2* Y0 = sm;
  double2* Y1 = Y0 + WB * (9 * NB16 + 1);             // [WB][NBLK][16]  pass-1 window outputs
  double2* sW = Y1 + WB * NBLK * 16;                  // [k][WB]        window of U_m
  double2* Xs = sW + 16 * WB;                         // [WB][16]       X_0..X_15
  const double2* tw = a.tw;
  double upd = 0.0;
  bool nonfinite = false;
  const int i0 = tid / WB, c0 = tid % WB;             // FreqMap butterfly of this thread

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long base = tile * (long)TILE;
    // (no L2 prefetch here: measured to evict and re-read ~45% of the tiles at this speed)
    // ---- inverse pass 0: DFT16 of W[i0 + (N/16) t], keep outputs s0 >= 16-k ----
    double2 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = a.in[base + tid + t * TPB];
    dft16<+1>(v);
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if (s >= 16 - k) Y0[c0 * (9 * NB16 + 1) + 9 * i0 + s - (16 - k)] = v[s];
    __syncthreads();
    // ---- inverse pass 1 (window butterflies only): i1 = 16 b + k1, k1 in [16-k, 16), output s1 = 15
    if (tid < 16 * k) {
      const int kk = tid % k, b = (tid / k) % NBLK, c = tid / (k * NBLK);
      const int k1 = 16 - k + kk;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int t1 = 0; t1 < 16; ++t1) {
        // input y0[i1 + (N/16) t1]: pass-0 butterfly b + NBLK t1, output k1
        const double2 x = Y0[c * (9 * NB16 + 1) + 9 * (b + NBLK * t1) + kk];
        double2 w = __ldg(&tw[((t1 * (k1 + 240)) & 255) * (N / 256)]);
        w.y = -w.y;                                    // inverse: e^{+2 pi i m / 256}
        acc = cfma(x, w, acc);
      }
      Y1[(c * NBLK + b) * 16 + kk] = acc;
    }
    __syncthreads();
    // ---- inverse pass 2 (window outputs, level n = N-k+j) fused with X_t, t < 16 ----
    // thread (c, t): X_t needs U^{N+t-jw} for jw = t+1..k, i.e. window entries j = k+t-jw; it
    // recomputes those from Y1 (RL terms each).  Threads t < k also own window entry j = t for
    // the monitor and the wrap state.
    if (tid < 16 * WB) {
      const int t = tid % 16, c = tid / 16;
      auto window = [&](int j) {   // U^{N-k+j} of column c
        const int i2 = 256 - k + j;
        double2 u = make_double2(0.0, 0.0);
#pragma unroll
        for (int t2 = 0; t2 < RL; ++t2) {
          double2 w = __ldg(&tw[(t2 * (i2 + 256 * (RL - 1))) & (N - 1)]);
          w.y = -w.y;
          u = cfma(Y1[(c * NBLK + t2) * 16 + j], w, u);
        }
        return cscale(u, __ldg(&a.igs[N - k + j]));
      };
      if (t < k) {
        const double2 U = window(t);
        const long wi = (tile * k + t) * WB + c;
        const double2 o = a.wrap_old[wi];
        const double d = sqrt(cabs2(csub(U, o)));
        if (!(d <= 1.7976931348623157e308)) nonfinite = true;
        upd = fmax(upd, d);
        a.wrap_new[wi] = U;
      }
      double2 F = make_double2(0.0, 0.0);
      if (t < nk) {
        const double2* srcp = a.src + tile * WB + c;
        for (int i = 0; i < a.nsparse; ++i) {
          const int s = __ldg(&a.spar[i]);
          F = cfmar(__ldg(&srcp[(long)s * ntiles * WB]), __ldg(&a.coef[(long)s * N + t]), F);
        }
        for (int jw = t + 1; jw <= k; ++jw) F = cfmar(window(k + t - jw), __ldg(&a.wk[jw]), F);
        F = cscale(F, __ldg(&a.gsf[t]));
      }
      Xs[c * 16 + t] = F;
    }
    __syncthreads();
    // ---- forward pass 2 with inputs X_t: H[i0 + (N/16) s] ----
    v[0] = Xs[c0 * 16];
#pragma unroll
    for (int t = 1; t < 16; ++t) {
      if (t < nk) v[t] = cmul(Xs[c0 * 16 + t], __ldg(&tw[t * i0]));   // w_N^{t i0}, forward
      else v[t] = make_double2(0.0, 0.0);
    }
    dft16<-1>(v);
    // dense static sources, synthesised in the frequency domain (precomputed DFT of their coefficients)
    if constexpr (DENSE) {
      for (int dd = 0; dd < a.ndense; ++dd) {
        const double2 g = __ldg(&a.src[((long)__ldg(&a.dsrc[dd]) * ntiles + tile) * WB + c0]);
        const double2* ch = a.chat + (long)dd * N + i0;
#pragma unroll
        for (int s = 0; s < 16; ++s) v[s] = cfma(__ldg(&ch[s * (N / 16)]), g, v[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < 16; ++s) a.out[base + tid + s * TPB] = v[s];
    __syncthreads();   // Xs / Y0 reused by the next tile
  }
  if (nonfinite) upd = __longlong_as_double(0x7ff0000000000000LL);
  block_max_atomic(upd, a.upd);
}

}  // namespace pint
