// fft.cuh — register/shared-memory Stockham FFT building blocks for complex128 tiles.
//
// A tile holds TILE = 4096 complex values laid out [n][WB] (time level n, WB = TILE/N
// contiguous spatial columns).  TPB = 256 threads; every thread owns 16 values per pass.
// Radix sequence for the inverse transform: 16, 16, ..., N/16^(np-1); the forward transform
// runs the reversed sequence, so that the inverse's output mapping IS the forward's input
// mapping (no shared-memory exchange between them) and the forward's output mapping is the
// inverse's input mapping (frequency-domain values stay in the same registers).
//
// Stockham auto-sort pass (radix R, span P): butterfly i in [0, N/R), k = i mod P,
//   inputs x[i + t N/R] * w_{PR}^{t k},  t < R;  outputs y[(i-k) R + k + s P] = DFT_R,  s < R.
// After all passes the output is in natural order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pint {

// Checked builds (-DPINT_CHECK, `build.py -D PINT_CHECK --lib libpint_check.so`): device-side bounds and
// protocol assertions on the shared-memory, tensor-memory, bulk-copy and grid-barrier indexing (a
// failed check traps: the launch fails loudly).  compute-sanitizer is closed on this GPU pool.
#ifdef PINT_CHECK
#define PINT_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define PINT_ASSERT(c) do { } while (0)
#endif

constexpr int TPB = 256;
constexpr int TILE = 4096;

__device__ __forceinline__ int phys(int e) { return e + (e >> 4); }   // 1 pad slot / 16: conflict-free
constexpr int phys_size(int n) { return n + (n >> 4) + 1; }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {   // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cfmar(double2 a, double s, double2 c) {   // a*s + c (s real)
  return make_double2(fma(a.x, s, c.x), fma(a.y, s, c.y));
}
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

template <int DIR> __device__ __forceinline__ double2 mul_i(double2 a) {   // a * (DIR i)
  return DIR > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
template <int DIR> __device__ __forceinline__ double2 cmul_w(double2 a, double c, double s) {
  // a * (c + DIR i s)
  return DIR > 0 ? make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c))
                 : make_double2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));
}

// ---- radix-R DFTs in registers: b_s = sum_t a_t exp(DIR 2 pi i s t / R) ------------------
template <int DIR> __device__ __forceinline__ void dft2(double2& a0, double2& a1) {
  const double2 t = a0; a0 = cadd(t, a1); a1 = csub(t, a1);
}
template <int DIR> __device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = mul_i<DIR>(csub(a1, a3));
  a0 = cadd(t0, t2); a2 = csub(t0, t2); a1 = cadd(t1, t3); a3 = csub(t1, t3);
}
constexpr double R2H = 0.70710678118654752440;   // cos(pi/4)
constexpr double C8 = 0.92387953251128675613;    // cos(pi/8)
constexpr double S8 = 0.38268343236508977173;    // sin(pi/8)

template <int DIR> __device__ __forceinline__ void dft8(double2* a) {
  double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
  double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
  dft4<DIR>(e0, e1, e2, e3);
  dft4<DIR>(o0, o1, o2, o3);
  o1 = cmul_w<DIR>(o1, R2H, R2H);
  o2 = mul_i<DIR>(o2);
  o3 = cmul_w<DIR>(o3, -R2H, R2H);
  a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
  a[1] = cadd(e1, o1); a[5] = csub(e1, o1);
  a[2] = cadd(e2, o2); a[6] = csub(e2, o2);
  a[3] = cadd(e3, o3); a[7] = csub(e3, o3);
}
// dft8 with a[t] = 0 for t >= NIN (compile time): the additions of known zeros are skipped (the
// compiler may not drop x + 0.0 itself: it is not an identity for x = -0.0)
template <int DIR, int NIN> __device__ __forceinline__ void dft4z(double2& a0, double2& a1, double2& a2, double2& a3) {
  // inputs (a0, a1, a2, a3) are time indices (i, i+2, i+4, i+6) of the dft8 below: NIN counts those < NIN
  if constexpr (NIN >= 4) {
    dft4<DIR>(a0, a1, a2, a3);
  } else if constexpr (NIN == 3) {                      // a3 = 0
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t3 = mul_i<DIR>(a1);
    a0 = cadd(t0, a1); a2 = csub(t0, a1); a1 = cadd(t1, t3); a3 = csub(t1, t3);
  } else if constexpr (NIN == 2) {                      // a2 = a3 = 0
    const double2 t3 = mul_i<DIR>(a1);
    a2 = csub(a0, a1); const double2 b0 = cadd(a0, a1); a1 = cadd(a0, t3); a3 = csub(a0, t3); a0 = b0;
  } else {                                              // a1 = a2 = a3 = 0
    a1 = a0; a2 = a0; a3 = a0;
  }
}
template <int DIR, int NIN> __device__ __forceinline__ void dft8z(double2* a) {
  if constexpr (NIN >= 8) {
    dft8<DIR>(a);
  } else {
    double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
    double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
    dft4z<DIR, (NIN + 1) / 2>(e0, e1, e2, e3);         // even times 0, 2, 4, 6
    dft4z<DIR, NIN / 2>(o0, o1, o2, o3);               // odd times 1, 3, 5, 7
    o1 = cmul_w<DIR>(o1, R2H, R2H);
    o2 = mul_i<DIR>(o2);
    o3 = cmul_w<DIR>(o3, -R2H, R2H);
    a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
    a[1] = cadd(e1, o1); a[5] = csub(e1, o1);
    a[2] = cadd(e2, o2); a[6] = csub(e2, o2);
    a[3] = cadd(e3, o3); a[7] = csub(e3, o3);
  }
}
template <int DIR> __device__ __forceinline__ void dft16(double2* a) {
  // index t = t1 + 4 t2; inner DFT4 over t2, twiddle w16^{t1 s1}, outer DFT4 over t1.
#pragma unroll
  for (int t1 = 0; t1 < 4; ++t1) dft4<DIR>(a[t1], a[t1 + 4], a[t1 + 8], a[t1 + 12]);
  // a[t1 + 4 s1] now holds inner output s1 of column t1
  a[5] = cmul_w<DIR>(a[5], C8, S8);          // t1=1 s1=1 : w^1
  a[9] = cmul_w<DIR>(a[9], R2H, R2H);        // t1=1 s1=2 : w^2
  a[13] = cmul_w<DIR>(a[13], S8, C8);        // t1=1 s1=3 : w^3
  a[6] = cmul_w<DIR>(a[6], R2H, R2H);        // t1=2 s1=1 : w^2
  a[10] = mul_i<DIR>(a[10]);                 // t1=2 s1=2 : w^4
  a[14] = cmul_w<DIR>(a[14], -R2H, R2H);     // t1=2 s1=3 : w^6
  a[7] = cmul_w<DIR>(a[7], S8, C8);          // t1=3 s1=1 : w^3
  a[11] = cmul_w<DIR>(a[11], -R2H, R2H);     // t1=3 s1=2 : w^6
  a[15] = cmul_w<DIR>(a[15], -C8, -S8);      // t1=3 s1=3 : w^9
#pragma unroll
  for (int s1 = 0; s1 < 4; ++s1) dft4<DIR>(a[4 * s1], a[4 * s1 + 1], a[4 * s1 + 2], a[4 * s1 + 3]);
  // a[s2 + 4 s1] holds b[s1 + 4 s2]: transpose 4x4
  double2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = a[i];
#pragma unroll
  for (int s1 = 0; s1 < 4; ++s1)
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) a[s1 + 4 * s2] = t[s2 + 4 * s1];
}
template <int R, int DIR> __device__ __forceinline__ void dft(double2* a) {
  if constexpr (R == 2) dft2<DIR>(a[0], a[1]);
  else if constexpr (R == 4) dft4<DIR>(a[0], a[1], a[2], a[3]);
  else if constexpr (R == 8) dft8<DIR>(a);
  else dft16<DIR>(a);
}

// ---- pass schedule -------------------------------------------------------------------
constexpr int np_of(int N) { return N <= 16 ? 1 : (N <= 256 ? 2 : 3); }
constexpr int last_radix(int N) { return np_of(N) == 1 ? N : (np_of(N) == 2 ? N / 16 : N / 256); }
constexpr int radix_inv(int N, int pi) { return pi < np_of(N) - 1 ? 16 : last_radix(N); }
constexpr int radix(int N, bool rev, int pi) { return rev ? radix_inv(N, np_of(N) - 1 - pi) : radix_inv(N, pi); }
constexpr int span(int N, bool rev, int pi) {
  int p = 1;
  for (int q = 0; q < pi; ++q) p *= radix(N, rev, q);
  return p;
}

template <int N, int R> __device__ __forceinline__ int in_index(int j, int t, int tid) {
  constexpr int WB = TILE / N;
  const int b = tid + j * TPB, i = b / WB, c = b % WB;
  return (i + t * (N / R)) * WB + c;
}
template <int N, int R, int P> __device__ __forceinline__ int out_index(int j, int s, int tid) {
  constexpr int WB = TILE / N;
  const int b = tid + j * TPB, i = b / WB, c = b % WB, k = i % P;
  return ((i - k) * R + k + s * P) * WB + c;
}

// twiddle table tw[m] = exp(-2 pi i m / N), m < N
template <int N, int R, int P, int DIR>
__device__ __forceinline__ void butterfly_pass(double2 (&v)[16], const double2* __restrict__ tw, int tid) {
  constexpr int WB = TILE / N;
#pragma unroll
  for (int j = 0; j < 16 / R; ++j) {
    if constexpr (P > 1) {
      const int b = tid + j * TPB, i = b / WB, k = i % P;
#pragma unroll
      for (int t = 1; t < R; ++t) {
        // volatile load: keeps the compiler from hoisting every pass's twiddles above the
        // barriers (which blew the CQ kernel up to 255 registers + spills)
        double2 w;
        asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "l"(&tw[t * k * (N / (P * R))]));
        if (DIR > 0) w.y = -w.y;
        v[j * R + t] = cmul(v[j * R + t], w);
      }
    }
    dft<R, DIR>(&v[j * R]);
  }
}

// Runs passes PI.. of the (REV ? forward-order : inverse-order) schedule.  On entry v holds
// the inputs of pass PI in its input mapping; on exit the outputs of the last pass in its
// output mapping.  Exchanges go through the shared tile `sm` (phys-padded).
template <int N, int DIR, bool REV, int PI = 0>
__device__ __forceinline__ void run_passes(double2 (&v)[16], double2* sm, const double2* __restrict__ tw, int tid) {
  constexpr int R = radix(N, REV, PI), P = span(N, REV, PI);
  butterfly_pass<N, R, P, DIR>(v, tw, tid);
  if constexpr (PI + 1 < np_of(N)) {
    constexpr int R2 = radix(N, REV, PI + 1);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16 / R; ++j)
#pragma unroll
      for (int s = 0; s < R; ++s) sm[phys(out_index<N, R, P>(j, s, tid))] = v[j * R + s];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16 / R2; ++j)
#pragma unroll
      for (int t = 0; t < R2; ++t) v[j * R2 + t] = sm[phys(in_index<N, R2>(j, t, tid))];
    run_passes<N, DIR, REV, PI + 1>(v, sm, tw, tid);
  }
}

// Element of register v[j*R + s] in the time-domain mapping (output of the inverse schedule,
// input of the forward schedule): level n = i + s*(N/RL), column c.
template <int N> struct TimeMap {
  static constexpr int WB = TILE / N;
  static constexpr int RL = last_radix(N);
  static constexpr int PL = N / RL;
  static constexpr int NJ = 16 / RL;
  __device__ __forceinline__ static int n(int j, int s, int tid) { return ((tid + j * TPB) / WB) + s * PL; }
  __device__ __forceinline__ static int c(int j, int tid) { return (tid + j * TPB) % WB; }
  __device__ __forceinline__ static int e(int j, int s, int tid) { return n(j, s, tid) * WB + c(j, tid); }
};
// Frequency-domain mapping (input of the inverse schedule, output of the forward): v[t],
// one radix-16 butterfly per thread: p = i + t*(N/16), column c, element = tid + t*256.
template <int N> struct FreqMap {
  static constexpr int WB = TILE / N;
  __device__ __forceinline__ static int p(int t, int tid) { return (tid / WB) + t * (N / 16); }
  __device__ __forceinline__ static int e(int t, int tid) { return tid + t * TPB; }
};

}  // namespace pint
