// spass.cuh — the shifted spatial solves ("S-pass"), Step 2 of Algorithm 1/2 (PAPER.md:472,
// 1057):  (d_p/tau^a + lambda_q + A_y) Q_{p,q} = H_{p,q}  for every frequency p and (2D)
// every DST-x mode q, along lines of length L in y.  Multiplying by h^2 (folded into H by
// the T-pass), each line is the constant-coefficient Dirichlet system
//     T_L x = d,   T_L = tridiag(-1, b, -1),   b = 2 + sigma,  sigma = h^2 (d_p/tau^a + lambda_q).
// Factorisation: with r + 1/r = b, |r| > 1, a = 1/r,
//     T_L = r (I - a L)(I - a U) + a e_1 e_1^T        (L, U = sub/super-diagonal shifts)
// so  x = x0 - x0_1 phi,   x0 = a (I - aU)^{-1} (I - aL)^{-1} d,
//     phi_y = (a^{y+2} - a^{2L+2-y}) / (1 - a^{2L+2})   (Sherman-Morrison, rows y = 0..L-1).
// The two first-order recurrences are evaluated as a warp-parallel chunked scan (one warp per
// line, lane t owns rows [tC, tC+C) in registers).  Shift accuracy (SURVEY §8(c) item 15,
// E-4): sigma is never added to 2; a is carried as 1 - u with u = t/(1+t) computed from
// sigma without cancellation, and every multiplication by a^m is z - u_m z.
#pragma once
#include "fft.cuh"

namespace pint {

// Per-line constants of the pair S-pass (plan time, spass_const_kernel): the factorisation
// a = 1 - u of tridiag(-1, 2 + sigma, -1), the u-form of a^C (C rows per lane), 1/(1 - a^{2L+2}),
// r = 1/a, and tl = log(1e-18 |1 - a^{2L+2}|) / log|a| (a^e / (1 - a^{2L+2}) matters iff e < tl)
struct SPassConst {
  double2 u, uc0, ru2L, rr;
  double tl, pad;
};
static_assert(sizeof(SPassConst) == 80, "SPassConst layout");

struct SPassArgs {
  const double2* in;      // H, tile-blocked layout [q][yb][N][WB]
  double2* out;           // W (may not alias in)
  const double2* sig_p;   // [N]  h^2 d_p / tau^a
  const double* sig_q;    // [Qb] h^2 lambda_q (0 in 1D)
  long N, NB;
  int WB, L;
  int lwb, lgw;           // log2(WB), log2(G*WB)
  long nwork;             // Qb * (N / G) strips
  const SPassConst* lc;   // [Qb][N] pair-kernel line constants (C/2 rows per lane)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double s = 1.0 / fma(b.x, b.x, b.y * b.y);
  return make_double2(fma(a.x, b.x, a.y * b.y) * s, fma(a.y, b.x, -a.x * b.y) * s);
}
__device__ __forceinline__ double2 csqrt_(double2 z) {
  const double r = hypot(z.x, z.y);
  if (r == 0.0) return make_double2(0.0, 0.0);
  if (z.x >= 0.0) {
    const double t = sqrt(0.5 * (r + z.x));
    return make_double2(t, z.y / (2.0 * t));
  }
  const double t = sqrt(0.5 * (r - z.x));
  return make_double2(fabs(z.y) / (2.0 * t), copysign(t, z.y));
}
// a * z with a = 1 - u  :  z - u z
__device__ __forceinline__ double2 amul(double2 u, double2 z) {
  return make_double2(fma(-u.x, z.x, fma(u.y, z.y, z.x)), fma(-u.x, z.y, fma(-u.y, z.x, z.y)));
}
// u-form product: (1 - u1)(1 - u2) = 1 - (u1 + u2 - u1 u2)
__device__ __forceinline__ double2 uprod(double2 u1, double2 u2) { return csub(cadd(u1, u2), cmul(u1, u2)); }
__device__ __forceinline__ double2 upow(double2 u, long n) {   // u-form of (1-u)^n
  double2 res = make_double2(0.0, 0.0), b = u;
  while (n) {
    if (n & 1) res = uprod(res, b);
    b = uprod(b, b);
    n >>= 1;
  }
  return res;
}

template <int C, int G>
__global__ void __launch_bounds__(32 * G, (C >= 32 ? 3 : 4)) spass_kernel(const SPassArgs a) {
  extern __shared__ double2 sm[];
  constexpr int SLINE0 = 32 * (C + 1);
  const int WB = a.WB, lwb = a.lwb, lgw = a.lgw;
  const int off = (WB >= 8) ? 0 : (WB > 8 / G ? WB : 8 / G);
  const int SLINE = SLINE0 + off;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long N = a.N, NB = a.NB;
  const long nblk = N / G;
  const int L = a.L;
  const int total = (int)NB * G * WB;
  const int gwm = G * WB - 1, wbm = WB - 1;

  for (long work = blockIdx.x; work < a.nwork; work += gridDim.x) {
    const long q = work / nblk;
    const long p0 = (work - q * nblk) * G;
    const double2* in_base = a.in + (q * NB * N + p0) * WB;
    // ---- stage the strip [NB][G][WB] into line-major padded smem (all copies in flight) ----
    // element e = tid + i*32G: (yb, g, j) = (e >> lgw, .., ..); y = yb*WB + j advances by 32 per
    // i and y/C by 32/C, so both addresses are linear in i.
    {
      const int e0 = threadIdx.x;
      const int yb0 = e0 >> lgw, rem = e0 & gwm, g = rem >> lwb, j = rem & wbm;
      const int y0s = (yb0 << lwb) + j;
      const double2* gp = in_base + ((long)yb0 * N + g) * WB + j;
      double2* sp_ = sm + g * SLINE + y0s + y0s / C;
      const long gstep = (long)(32 / WB) * N * WB;
      const int nit = (total + 32 * G - 1) / (32 * G);
      if (WB <= 32) {
        for (int i = 0; i < nit; ++i)
          if (e0 + i * 32 * G < total && y0s + 32 * i < 32 * C) cp_async16(sp_ + i * (32 + 32 / C), gp + i * gstep);
      } else {
        for (int e = threadIdx.x; e < total; e += 32 * G) {
          const int yb = e >> lgw, rm = e & gwm, gg = rm >> lwb, jj = rm & wbm;
          const int y = (yb << lwb) + jj;
          if (y < 32 * C) cp_async16(&sm[gg * SLINE + y + y / C], in_base + ((long)yb * N + gg) * WB + jj);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- per line setup: sigma -> t -> u = 1 - a ----
    const long p = p0 + warp;
    const double2 sp = a.sig_p[p];
    const double2 sig = make_double2(sp.x + a.sig_q[q], sp.y);
    const double2 s = csqrt_(cmul(sig, make_double2(4.0 + sig.x, sig.y)));
    const double2 t1 = cscale(cadd(sig, s), 0.5), t2 = cscale(csub(sig, s), 0.5);
    const double2 tb = cabs2(t1) >= cabs2(t2) ? t1 : t2;
    const double2 ts = cdiv(make_double2(-sig.x, -sig.y), tb);          // tb * ts = -sigma
    const double2 rb = make_double2(1.0 + tb.x, tb.y), rs = make_double2(1.0 + ts.x, ts.y);
    const double2 tt = cabs2(rb) > cabs2(rs) ? tb : ts;
    const double2 rr = make_double2(1.0 + tt.x, tt.y);                  // r = 1/a, |r| > 1
    const double2 u = cdiv(tt, rr);                                     // u = 1 - a
    double2 uc[5];                                                      // u-forms of a^{C 2^j}
    uc[0] = upow(u, C);
#pragma unroll
    for (int i = 1; i < 5; ++i) uc[i] = uprod(uc[i - 1], uc[i - 1]);

    // ---- registers: rows y = lane*C + r ----
    double2 d[C];
    double2* line = sm + warp * SLINE + lane * (C + 1);
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int y = lane * C + r;
      d[r] = (y < L) ? line[r] : make_double2(0.0, 0.0);
    }

    // ---- forward recurrence f_y = d_y + a f_{y-1} ----
    double2 f = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < C; ++r) f = cadd(d[r], amul(u, f));
#pragma unroll
    for (int i = 0; i < 5; ++i) {                                       // S_t = sum_{s<=t} a^{C(t-s)} loc_s
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
      d[r] = (lane * C + r < L) ? f : make_double2(0.0, 0.0);
    }

    // ---- backward recurrence w_y = f_y + a w_{y+1} ----
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

    // ---- rank-1 Dirichlet correction: x = a (w - w_0 phi) ----
    double2 w0;
    w0.x = __shfl_sync(0xffffffffu, d[0].x, 0);
    w0.y = __shfl_sync(0xffffffffu, d[0].y, 0);
    const double2 u2L = upow(u, 2L * L + 2);             // 1 - a^{2L+2}
    const double2 K = cdiv(w0, u2L);                      // w_0 / (1 - a^{2L+2})
    const int y0 = lane * C;
    if (y0 < L) {
      // skip chunks where |phi| < 1e-18 throughout (|a^{y+2}| falls and |a^{2L+2-y}| rises along y)
      const double2 a1 = make_double2(1.0 - u.x, -u.y);   // a as a value
      const double la = 0.5 * log(cabs2(a1));             // log|a| < 0
      const double thr = -41.44653167389282 + 0.5 * log(cabs2(u2L));   // log(1e-18 |1-a^{2L+2}|)
      const int ylast = min(y0 + C, L) - 1;
      if ((y0 + 2) * la > thr || (2.0 * L + 2 - ylast) * la > thr) {
        const double2 uP = upow(u, y0 + 2);               // a^{y0+2} = 1 - uP
        const double2 uQ = upow(u, 2L * L + 2 - y0);      // a^{2L+2-y0}
        double2 P = make_double2(1.0 - uP.x, -uP.y);
        double2 Q = make_double2(1.0 - uQ.x, -uQ.y);
#pragma unroll
        for (int r = 0; r < C; ++r) {
          d[r] = csub(d[r], cmul(K, csub(P, Q)));
          P = cmul(P, a1);
          Q = cmul(Q, rr);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int y = lane * C + r;
      line[r] = (y < L) ? amul(u, d[r]) : make_double2(0.0, 0.0);
    }
    __syncthreads();

    {
      double2* out_base = a.out + (q * NB * N + p0) * WB;
      const int e0 = threadIdx.x;
      const int yb0 = e0 >> lgw, rem = e0 & gwm, g = rem >> lwb, j = rem & wbm;
      const int y0s = (yb0 << lwb) + j;
      double2* gp = out_base + ((long)yb0 * N + g) * WB + j;
      const double2* sp_ = sm + g * SLINE + y0s + y0s / C;
      const long gstep = (long)(32 / WB) * N * WB;
      const int nit = (total + 32 * G - 1) / (32 * G);
      if (WB <= 32) {
        for (int i = 0; i < nit; ++i)
          if (e0 + i * 32 * G < total)
            gp[i * gstep] = (y0s + 32 * i < 32 * C) ? sp_[i * (32 + 32 / C)] : make_double2(0.0, 0.0);
      } else {
        for (int e = threadIdx.x; e < total; e += 32 * G) {
          const int yb = e >> lgw, rm = e & gwm, gg = rm >> lwb, jj = rm & wbm;
          const int y = (yb << lwb) + jj;
          out_base[((long)yb * N + gg) * WB + jj] = (y < 32 * C) ? sm[gg * SLINE + y + y / C] : make_double2(0.0, 0.0);
        }
      }
    }
    __syncthreads();   // smem reused by the next strip
  }
}


// ---- direct variant (WB >= 2, C even): each lane moves its row pairs (y, y+1) as one full
// 32-byte sector with 256-bit loads/stores straight between HBM and registers.  No shared
// memory and no barriers: warps desynchronise freely, and a lane issues all C/2 loads at once.
__device__ __forceinline__ void ld256(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void st256(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}

template <int C>
__device__ __forceinline__ void solve_line_regs(double2 (&d)[C], double2 sig, int L, int lane) {
  const double2 s = csqrt_(cmul(sig, make_double2(4.0 + sig.x, sig.y)));
  const double2 t1 = cscale(cadd(sig, s), 0.5), t2 = cscale(csub(sig, s), 0.5);
  const double2 tb = cabs2(t1) >= cabs2(t2) ? t1 : t2;
  const double2 ts = cdiv(make_double2(-sig.x, -sig.y), tb);          // tb * ts = -sigma
  const double2 rb = make_double2(1.0 + tb.x, tb.y), rs = make_double2(1.0 + ts.x, ts.y);
  const double2 tt = cabs2(rb) > cabs2(rs) ? tb : ts;
  const double2 rr = make_double2(1.0 + tt.x, tt.y);                  // r = 1/a, |r| > 1
  const double2 u = cdiv(tt, rr);                                     // u = 1 - a
  double2 uc[5];
  uc[0] = u;
#pragma unroll
  for (int c = 1; c < C; c <<= 1) uc[0] = uprod(uc[0], uc[0]);        // a^C (C power of two)
#pragma unroll
  for (int i = 1; i < 5; ++i) uc[i] = uprod(uc[i - 1], uc[i - 1]);
  const int nv = min(max(L - lane * C, 0), C);                         // valid rows of this lane

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
  const double2 u2L = upow(u, 2L * L + 2);
  const double2 K = cdiv(w0, u2L);
  const int y0 = lane * C;
  if (nv > 0) {
    const double2 a1 = make_double2(1.0 - u.x, -u.y);
    const double la = 0.5 * log(cabs2(a1));                           // log|a| < 0
    const double thr = -41.44653167389282 + 0.5 * log(cabs2(u2L));    // log(1e-18 |1 - a^{2L+2}|)
    const bool needP = (y0 + 2) * la > thr;                             // |a^{y+2}| largest at y0
    const bool needQ = (2.0 * L + 2 - (y0 + nv - 1)) * la > thr;        // |a^{2L+2-y}| largest at the chunk end
    if (needP) {
      const double2 uP = upow(u, y0 + 2);
      double2 KP = cmul(K, make_double2(1.0 - uP.x, -uP.y));          // K a^{y+2}
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = csub(d[r], KP); KP = cmul(KP, a1); }
    }
    if (needQ) {
      const double2 uQ = upow(u, 2L * L + 2 - y0);
      double2 KQ = cmul(K, make_double2(1.0 - uQ.x, -uQ.y));          // K a^{2L+2-y}
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = cadd(d[r], KQ); KQ = cmul(KQ, rr); }
    }
  }
#pragma unroll
  for (int r = 0; r < C; ++r) d[r] = (r < nv) ? amul(u, d[r]) : make_double2(0.0, 0.0);
}

template <int C>
__global__ void __launch_bounds__(128, 3) spass_direct_kernel(const SPassArgs a) {
  static_assert(C % 2 == 0, "row pairs");
  const int lane = threadIdx.x % 32;
  const long line = (long)blockIdx.x * 4 + threadIdx.x / 32;         // line = q * N + p
  const long N = a.N, NB = a.NB;
  if (line >= (long)a.nwork) return;
  const long q = line / N, p = line - q * N;
  const int WB = a.WB, lwb = a.lwb, L = a.L;
  const int Lpad = (int)NB * WB;
  const double2* in = a.in + (q * NB * N + p) * WB;
  double2* out = a.out + (q * NB * N + p) * WB;
  double2 d[C];
#pragma unroll
  for (int r = 0; r < C; r += 2) {
    const int y = lane * C + r;
    if (y < Lpad) ld256(in + ((long)(y >> lwb) * N) * WB + (y & (WB - 1)), d[r], d[r + 1]);
    else { d[r] = make_double2(0.0, 0.0); d[r + 1] = d[r]; }
  }
  const double2 sp = __ldg(&a.sig_p[p]);
  const double2 sig = make_double2(sp.x + __ldg(&a.sig_q[q]), sp.y);
  const int nv = min(max(L - lane * C, 0), C);
#pragma unroll
  for (int r = 0; r < C; ++r) if (r >= nv) d[r] = make_double2(0.0, 0.0);
  solve_line_regs<C>(d, sig, L, lane);
#pragma unroll
  for (int r = 0; r < C; r += 2) {
    const int y = lane * C + r;
    if (y < Lpad) st256(out + ((long)(y >> lwb) * N) * WB + (y & (WB - 1)), d[r], d[r + 1]);
  }
}

// ---- two-warp variant (WB >= 2): a line of up to 64*C rows is split over 2 warps (lane gl =
// 32*half + lane owns rows [gl*C, gl*C + C)); the warps exchange their scan totals through
// shared memory under a pair-scoped named barrier.  Halves the recurrence chains and the
// per-thread registers (more resident warps) relative to one warp per line.
__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

#ifndef PINT_PAIR_MINB
#define PINT_PAIR_MINB 4
#endif
// recurrence step d + m z with the multiplier in u-form (c = 1 - m; shift-accurate: z - c z) or, AF, in
// value form (c = m; one complex FMA) — the value form for lines with |u| >= 1e-3, where rounding
// a = 1 - u perturbs u (hence the shift) by at most 2e-13 relatively (as the fused solve, fused.cuh)
template <bool AF> __device__ __forceinline__ double2 pstep(double2 c, double2 z, double2 d) {
  if constexpr (AF) return cfma(c, z, d);
  else return cadd(d, amul(c, z));
}
template <bool AF> __device__ __forceinline__ double2 pconv(double2 uform) {
  return AF ? make_double2(1.0 - uform.x, -uform.y) : uform;
}
#ifndef PINT_PAIR_AF
#define PINT_PAIR_AF 1
#endif
constexpr double PAIR_AF_U2 = 1e-6;

#ifndef PINT_PAIR_LPC
#define PINT_PAIR_LPC 2   // lines (consecutive frequencies of one x-mode) per CTA, two warps each
#endif

// The pair solve: lane gl = 32 half + lane of the pair owns rows [gl C, gl C + C) in d (rows >= L
// zero on entry); on exit d holds the solution rows (zero beyond L).  xch: the pair's exchange slots.
template <int C, bool AF = false>
__device__ __forceinline__ void pair_solve(double2 (&d)[C], const SPassConst& lc, int L, int lane, int half, int gl,
                                           int nv, double2* xch, int pair) {
  // ---- line constants (plan-time table) ----
  const double2 u = lc.u, rr = lc.rr;
  const double2 um = pconv<AF>(u);                   // the step multiplier (u- or value form)
  // the lane holding row L-1 zeroes its rows >= L (2^n - 1 lines: one pad row, a single register)
  const bool pad1 = L >= 64 * C - 1;
  auto zero_tail = [&](double2 (&v)[C]) {
    if (pad1) {
      if (nv < C) v[C - 1] = make_double2(0.0, 0.0);
    } else if (nv < C) {
#pragma unroll
      for (int r = 0; r < C; ++r)
        if (r >= nv) v[r] = make_double2(0.0, 0.0);
    }
  };
  double2 uc[6];                                     // u-forms of a^{C 2^j}, j = 0..5
  uc[0] = lc.uc0;
#pragma unroll
  for (int i = 1; i < 6; ++i) uc[i] = uprod(uc[i - 1], uc[i - 1]);
  // per-lane u-form of a^{C (lane+1)} and a^{C (32-lane)} (for the cross-warp carries)
  double2 ufw = make_double2(0.0, 0.0), ubw = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    if ((lane + 1) & (1 << i)) ufw = uprod(ufw, uc[i]);
    if ((32 - lane) & (1 << i)) ubw = uprod(ubw, uc[i]);
  }
  double2 ucm[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) ucm[i] = pconv<AF>(uc[i]);
  // in-warp scan levels i < nlev: |a^{C 2^i}| >= 2^-64 (the others add nothing to the lane totals);
  // C = 16 keeps all five (A/B: the count's registers cost more than the skipped levels, 16.9 -> 17.9 ms
  // for the C4 streaming S-pass), C <= 8 skips (C5 S-pass 2.22 -> 2.17 ms)
  int nlev = 5;
  if constexpr (C <= 8) {
    nlev = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) nlev += cabs2(make_double2(1.0 - uc[i].x, -uc[i].y)) >= 0x1p-128 ? 1 : 0;
  }
  const double2 ufm = pconv<AF>(ufw), ubm = pconv<AF>(ubw);

  // ---- forward recurrence ----
  double2 f = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 0; r < C; ++r) f = pstep<AF>(um, f, d[r]);
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i >= nlev) break;
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_up_sync(0xffffffffu, f.x, o);
    x.y = __shfl_up_sync(0xffffffffu, f.y, o);
    if (lane >= o) f = pstep<AF>(ucm[i], x, f);
  }
  if (half == 0 && lane == 31) xch[0] = f;     // warp-0 total (inclusive at its last row)
  pair_bar(1 + pair);
  if (half == 1) f = pstep<AF>(ufm, xch[0], f);
  double2 carry;
  carry.x = __shfl_up_sync(0xffffffffu, f.x, 1);
  carry.y = __shfl_up_sync(0xffffffffu, f.y, 1);
  if (lane == 0) carry = half ? xch[0] : make_double2(0.0, 0.0);
  f = carry;
#pragma unroll
  for (int r = 0; r < C; ++r) {
    f = pstep<AF>(um, f, d[r]);
    d[r] = f;
  }
  zero_tail(d);
  // ---- backward recurrence ----
  double2 w = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = C - 1; r >= 0; --r) w = pstep<AF>(um, w, d[r]);
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i >= nlev) break;
    const int o = 1 << i;
    double2 x;
    x.x = __shfl_down_sync(0xffffffffu, w.x, o);
    x.y = __shfl_down_sync(0xffffffffu, w.y, o);
    if (lane + o < 32) w = pstep<AF>(ucm[i], x, w);
  }
  if (half == 1 && lane == 0) xch[1] = w;      // warp-1 total (suffix from its first row)
  pair_bar(1 + pair);
  if (half == 0) w = pstep<AF>(ubm, xch[1], w);
  carry.x = __shfl_down_sync(0xffffffffu, w.x, 1);
  carry.y = __shfl_down_sync(0xffffffffu, w.y, 1);
  if (lane == 31) carry = half ? make_double2(0.0, 0.0) : xch[1];
  w = carry;
#pragma unroll
  for (int r = C - 1; r >= 0; --r) {
    w = pstep<AF>(um, w, d[r]);
    d[r] = w;
  }
  // ---- rank-1 Dirichlet correction ----
  if (half == 0 && lane == 0) xch[2] = d[0];
  pair_bar(1 + pair);
  const double2 w0 = xch[2];
  const double2 K = cmul(w0, lc.ru2L);
  const int y0 = gl * C;
  if (nv > 0) {
    const double2 a1 = make_double2(1.0 - u.x, -u.y);
    const bool needP = y0 + 2 < lc.tl;
    const bool needQ = 2.0 * L + 2 - (y0 + nv - 1) < lc.tl;
    if (needP) {
      const double2 uP = upow(u, y0 + 2);
      double2 KP = cmul(K, make_double2(1.0 - uP.x, -uP.y));
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = csub(d[r], KP); KP = cmul(KP, a1); }
    }
    if (needQ) {
      const double2 uQ = upow(u, 2L * L + 2 - y0);
      double2 KQ = cmul(K, make_double2(1.0 - uQ.x, -uQ.y));
#pragma unroll
      for (int r = 0; r < C; ++r) { d[r] = cadd(d[r], KQ); KQ = cmul(KQ, rr); }
    }
  }
#pragma unroll
  for (int r = 0; r < C; ++r) d[r] = AF ? cmul(um, d[r]) : amul(u, d[r]);
  zero_tail(d);
}

// plan time: per-line constants of the pair S-pass (C = rows per lane of the pair kernel)
static __global__ void spass_const_kernel(SPassConst* out, const double2* sig_p, const double* sig_q, long N, long Qb, int C,
                                   int L) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < N * Qb; e += (long)gridDim.x * blockDim.x) {
    const long q = e / N, p = e % N;
    const double2 sp = sig_p[p];
    const double2 sig = make_double2(sp.x + sig_q[q], sp.y);
    const double2 s2 = csqrt_(cmul(sig, make_double2(4.0 + sig.x, sig.y)));
    const double2 t1 = cscale(cadd(sig, s2), 0.5), t2 = cscale(csub(sig, s2), 0.5);
    const double2 tb = cabs2(t1) >= cabs2(t2) ? t1 : t2;
    const double2 ts = cdiv(make_double2(-sig.x, -sig.y), tb);          // tb * ts = -sigma
    const double2 rb = make_double2(1.0 + tb.x, tb.y), rs = make_double2(1.0 + ts.x, ts.y);
    const double2 tt = cabs2(rb) > cabs2(rs) ? tb : ts;
    SPassConst c;
    c.rr = make_double2(1.0 + tt.x, tt.y);                              // r = 1/a, |r| > 1
    c.u = cdiv(tt, c.rr);                                               // u = 1 - a
    c.uc0 = upow(c.u, C);
    const double2 u2L = upow(c.u, 2L * L + 2);                          // 1 - a^{2L+2}
    c.ru2L = cdiv(make_double2(1.0, 0.0), u2L);
    const double la = 0.5 * log(cabs2(make_double2(1.0 - c.u.x, -c.u.y)));   // log|a| < 0
    const double thr = -41.44653167389282 + 0.5 * log(cabs2(u2L));
    c.tl = la < 0.0 ? thr / la : INFINITY;
    c.pad = 0.0;
    out[e] = c;
  }
}



template <int C>
__global__ void __launch_bounds__(64 * PINT_PAIR_LPC, PINT_PAIR_MINB * 2 / PINT_PAIR_LPC) spass_pair_kernel(const SPassArgs a) {
  __shared__ double2 xch[PINT_PAIR_LPC][4];          // per pair: fwd total, bwd total, w0, spare
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int pair = warp >> 1, half = warp & 1;
  const long line = (long)blockIdx.x * PINT_PAIR_LPC + pair;
  const long N = a.N, NB = a.NB;
  const bool live = line < a.nwork;
  const long q = live ? line / N : 0, p = live ? line - q * N : 0;
  const int WB = a.WB, lwb = a.lwb, L = a.L;
  const int Lpad = (int)NB * WB;
  const int gl = half * 32 + lane;
  const double2* in = a.in + (q * NB * N + p) * WB;
  double2 d[C];
#pragma unroll
  for (int r = 0; r < C; r += 2) {
    const int y = gl * C + r;
    if (live && y < Lpad) ld256(in + ((long)(y >> lwb) * N) * WB + (y & (WB - 1)), d[r], d[r + 1]);
    else { d[r] = make_double2(0.0, 0.0); d[r + 1] = d[r]; }
  }
  const int nv = min(max(L - gl * C, 0), C);
  // input rows y >= L are exact zeros (pad rows of H), so no masking after the loads
  SPassConst lc = live ? a.lc[q * N + p] : a.lc[0];
  // (C = 16, N = 2048: the second instance of the solve no longer fits the 128-register budget)
  if (PINT_PAIR_AF && C <= 8 && cabs2(lc.u) >= PAIR_AF_U2) pair_solve<C, (C <= 8)>(d, lc, L, lane, half, gl, nv, xch[pair], pair);
  else pair_solve<C, false>(d, lc, L, lane, half, gl, nv, xch[pair], pair);
  double2* out = a.out + (q * NB * N + p) * WB;
#pragma unroll
  for (int r = 0; r < C; r += 2) {
    const int y = gl * C + r;
    if (live && y < Lpad) st256(out + ((long)(y >> lwb) * N) * WB + (y & (WB - 1)), d[r], d[r + 1]);
  }
}

}  // namespace pint
