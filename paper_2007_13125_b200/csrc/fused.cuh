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

constexpr int FG = 8;      // lines per group
constexpr int FT = 256;    // threads per CTA: warp s solves line s of the group

// Per line (q, p): the iteration-invariant constants of the Toeplitz factorisation (spass.cuh),
// computed once at plan time (line_const_kernel).
struct LineConst {
  double2 u;        // 1 - a,  a = 1/r, r + 1/r = 2 + sigma, |r| > 1
  double2 uc[7];    // u-forms of a^{C 2^i}
  double2 uE;       // u-form of a^{(2L+2) mod C}
  double2 ru2L;     // 1 / (1 - a^{2L+2})
  double2 rr;       // r
  double la, thr;   // log|a|;  log(1e-18 |1 - a^{2L+2}|)
};

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
};

// smem row swizzle: lane l of the solve owns rows [lC, lC + C); XOR-ing the low bits with the
// chunk index keeps its 16-byte accesses bank-conflict free, and consecutive rows (row phases)
// stay within their aligned 8-row block.
template <int C> __device__ __forceinline__ int swz(int y) {
  constexpr int CM = C < 8 ? C : 8;
  constexpr int SH = C >= 8 ? 0 : (C == 4 ? 1 : (C == 2 ? 2 : 3));
  return y ^ (((y / C) >> SH) & (CM - 1));
}

__device__ __forceinline__ double2 one_minus(double2 u) { return make_double2(1.0 - u.x, -u.y); }

template <int C>
__device__ __forceinline__ void fused_synth(const FusedArgs& a, double2* Hs, const double2* Xq, long q, int i) {
  constexpr int LF = 32 * C;
  const int NG = (int)(a.N / FG);
  for (int y = threadIdx.x; y < LF; y += FT) {
    double2 z[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      z[t] = make_double2(0.0, 0.0);
      if (t < a.nk) {
        const double2 x = Xq[t * LF + y];
        z[t] = t == 0 ? x : cmul(x, __ldg(&a.tw[t * i]));   // X_t w_N^{t i}
      }
    }
    dft8<-1>(z);                                           // H_{i + (N/8) s} = sum_t z_t e^{-2 pi i ts/8}
    for (int d = 0; d < a.ndense; ++d) {
      const double2 g = y < a.L ? __ldg(&a.src[((long)__ldg(&a.dsrc[d]) * a.Qb + q) * a.Lpad + y])
                                : make_double2(0.0, 0.0);
      const double2* ch = a.chat + (long)d * a.N + i;
#pragma unroll
      for (int s = 0; s < 8; ++s) z[s] = cfma(__ldg(&ch[s * NG]), g, z[s]);
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) Hs[s * LF + swz<C>(y)] = z[s];
  }
}

template <int C>
__device__ __forceinline__ void fused_window(const FusedArgs& a, const double2* Hs, double2* acc, int i) {
  constexpr int LF = 32 * C;
  const int N = (int)a.N, k = a.k;
  for (int y = threadIdx.x; y < LF; y += FT) {
    double2 x[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) x[s] = Hs[s * LF + swz<C>(y)];
    dft8<+1>(x);                                           // Y_r = sum_s e^{+2 pi i rs/8} W_{i + (N/8) s}
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int j = r - 8 + k;                             // level n = N - 8 + r = N - k + j
      if (j >= 0) {
        double2 w = __ldg(&a.tw[((N - 8 + r) * i) & (N - 1)]);
        w.y = -w.y;                                        // e^{+2 pi i n i/N}
        acc[j * LF + y] = cfma(x[r], w, acc[j * LF + y]);
      }
    }
  }
}

// Step 2 for line (q, p) by one warp; rows lane*C .. lane*C + C - 1 (chunked warp scan, spass.cuh)
template <int C, bool STORE_W>
__device__ __forceinline__ void fused_solve(const FusedArgs& a, double2* Hl, long q, long p) {
  const int lane = threadIdx.x & 31;
  const int L = a.L;
  const LineConst* lc = a.lc + q * a.N + p;
  const double2 u = lc->u;
  double2 uc[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) uc[i] = lc->uc[i];
  const int y0 = lane * C;
  const int nv = min(max(L - y0, 0), C);
  double2 d[C];
#pragma unroll
  for (int r = 0; r < C; ++r) d[r] = (r < nv) ? Hl[swz<C>(y0 + r)] : make_double2(0.0, 0.0);

  // forward recurrence f_y = d_y + a f_{y-1}
  double2 f = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 0; r < C; ++r) f = cadd(d[r], amul(u, f));
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_up_sync(0xffffffffu, f.x, o);
    x.y = __shfl_up_sync(0xffffffffu, f.y, o);
    if (lane >= o) f = cadd(f, amul(uc[i], x));
  }
  double2 carry;
  carry.x = __shfl_up_sync(0xffffffffu, f.x, 1);
  carry.y = __shfl_up_sync(0xffffffffu, f.y, 1);
  if (lane == 0) carry = make_double2(0.0, 0.0);
  f = carry;
#pragma unroll
  for (int r = 0; r < C; ++r) {
    f = cadd(d[r], amul(u, f));
    d[r] = (r < nv) ? f : make_double2(0.0, 0.0);
  }
  // backward recurrence w_y = f_y + a w_{y+1}
  double2 w = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = C - 1; r >= 0; --r) w = cadd(d[r], amul(u, w));
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_down_sync(0xffffffffu, w.x, o);
    x.y = __shfl_down_sync(0xffffffffu, w.y, o);
    if (lane + o < 32) w = cadd(w, amul(uc[i], x));
  }
  carry.x = __shfl_down_sync(0xffffffffu, w.x, 1);
  carry.y = __shfl_down_sync(0xffffffffu, w.y, 1);
  if (lane == 31) carry = make_double2(0.0, 0.0);
  w = carry;
#pragma unroll
  for (int r = C - 1; r >= 0; --r) {
    w = cadd(d[r], amul(u, w));
    d[r] = w;
  }
  // rank-1 Dirichlet correction x = a (w - w_0 phi), phi_y = (a^{y+2} - a^{2L+2-y}) / (1 - a^{2L+2})
  double2 w0;
  w0.x = __shfl_sync(0xffffffffu, d[0].x, 0);
  w0.y = __shfl_sync(0xffffffffu, d[0].y, 0);
  const double2 K = cmul(w0, lc->ru2L);
  if (nv > 0) {
    const double la = lc->la, thr = lc->thr;
    if ((y0 + 2) * la > thr) {                              // |a^{y+2}| is largest at y0
      double2 ul = uprod(u, u);                             // a^2
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if ((lane >> i) & 1) ul = uprod(ul, uc[i]);         // a^{C lane + 2}
      double2 KP = cmul(K, one_minus(ul));
      const double2 a1 = one_minus(u);
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = csub(d[r], KP); KP = cmul(KP, a1); }
    }
    if ((2.0 * L + 2 - (y0 + nv - 1)) * la > thr) {         // |a^{2L+2-y}| is largest at the chunk end
      // 2L+2-y0 = e + C (m0 - lane),  e = (2L+2) mod C
      const int m = (2 * L + 2) / C - lane;
      double2 uq = lc->uE;
#pragma unroll
      for (int i = 0; i < 7; ++i)
        if ((m >> i) & 1) uq = uprod(uq, lc->uc[i]);
      double2 KQ = cmul(K, one_minus(uq));
      const double2 rr = lc->rr;
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = cadd(d[r], KQ); KQ = cmul(KQ, rr); }
    }
  }
  if constexpr (STORE_W) {
    double2* Wq = a.W + (q * a.NB * a.N + p) * a.WB;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int y = y0 + r;
      if (y < a.Lpad) Wq[((long)(y / a.WB) * a.N) * a.WB + (y % a.WB)] = (r < nv) ? amul(u, d[r]) : make_double2(0.0, 0.0);
    }
  } else {
#pragma unroll
    for (int r = 0; r < C; ++r) Hl[swz<C>(y0 + r)] = (r < nv) ? amul(u, d[r]) : make_double2(0.0, 0.0);
  }
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
};

#ifdef PINT_DEFINE_FUSED_KERNELS
// grid = Qb * nch CTAs; CTA (q, ch) runs groups [ch*gpc, (ch+1)*gpc) of x-mode q.
template <int C, bool STORE_W>
__global__ void __launch_bounds__(FT, 1) wr_fused_kernel(const FusedArgs a) {
  extern __shared__ double2 fsm[];
  constexpr int LF = 32 * C;
  double2* Hs = fsm;              // [8][LF]   H (in) / W (out) of the group's lines
  double2* acc = fsm + 8 * LF;    // [k][LF]   window partial sums
  const long q = blockIdx.x / a.nch;
  const int ch = blockIdx.x % a.nch;
  const int NG = (int)(a.N / FG);
  const int g0 = ch * a.gpc, g1 = min(g0 + a.gpc, NG);
  const int warp = threadIdx.x >> 5;
  const double2* Xq = a.X + q * 8 * LF;
  if (!STORE_W)
    for (int y = threadIdx.x; y < LF; y += FT)
      for (int j = 0; j < a.k; ++j) acc[j * LF + y] = make_double2(0.0, 0.0);
  fused_synth<C>(a, Hs, Xq, q, g0);
  __syncthreads();
  for (int i = g0; i < g1; ++i) {
    fused_solve<C, STORE_W>(a, Hs + warp * LF, q, i + (long)NG * warp);
    __syncthreads();
    if (!STORE_W) fused_window<C>(a, Hs, acc, i);     // rows owned by this thread: no barrier
    if (i + 1 < g1) fused_synth<C>(a, Hs, Xq, q, i + 1);
    __syncthreads();
  }
  if (!STORE_W) {
    double2* P = a.P + ((q * a.nch + ch) * a.k) * LF;
    for (int y = threadIdx.x; y < LF; y += FT)
      for (int j = 0; j < a.k; ++j) P[j * LF + y] = acc[j * LF + y];
  }
}

__global__ void __launch_bounds__(TPB) wr_finish_kernel(const FinishArgs a, int mode) {
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
          for (int c = 0; c < a.nch; ++c) s = cadd(s, a.P[((q * a.nch + c) * k + j) * a.Lf + y]);
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

// ---- plan time: per-line constants ----
__global__ void line_const_kernel(LineConst* lc, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int L) {
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
    for (int i = 1; i < 7; ++i) c.uc[i] = uprod(c.uc[i - 1], c.uc[i - 1]);
    const double2 u2L = upow(c.u, 2L * L + 2);
    c.ru2L = cdiv(make_double2(1.0, 0.0), u2L);
    c.uE = upow(c.u, (2L * L + 2) % C);
    c.la = 0.5 * log(cabs2(one_minus(c.u)));
    c.thr = -41.44653167389282 + 0.5 * log(cabs2(u2L));
    lc[e] = c;
  }
}
#endif  // PINT_DEFINE_FUSED_KERNELS

}  // namespace pint
