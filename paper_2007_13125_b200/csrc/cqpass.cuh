// cqpass.cuh — the CQ (subdiffusion) T-pass of one WR iteration as ONE kernel per iteration.
//
// Per tile (all N levels of WB = 4096/N adjacent spatial columns, 64 KB, contiguous in HBM):
//   W_m --V--> u                      U_m = Gamma^{-1} u: full-array update monitor,
//                                     U_m -> ufull, window levels -> wrap state        (Step 3)
//   u --Theta/N, V^{-1}--> z --D'--> --V--> s --C Theta^{-1}, V^{-1}--> H'
//   H_{m+1} = H' + D W_m + sum_s chat_s src_s                       (kappa-wrap + Step 1)
// i.e. the circulant +- skew-circulant form of the kappa-wrap of eq:BDF-subdiff-F (DESIGN.md §5.2,
// "CQ wrap"): four length-N transforms per column, all on chip.
//
// B200 design (replaces the two-kernel split of tpass.cuh, which moved 80 B/unknown and ran each
// transform as three radix-16 passes with two shared-memory exchanges):
//  * N = N1 * N1 (N1 = 32: N = 1024, the C5 configuration; N1 = 16: N = 256) as a 4-step transform:
//    thread (i, c) owns the N1 values i + N1 t of column c; pass A = DFT_N1 over t in registers, twiddle
//    w^{i k2}, ONE shared-memory exchange (rows XOR-swizzled: conflict-free 16-byte accesses), pass B = DFT_N1.
//    Input and output mappings are the same (thread i holds index i + N1 t), so the four transforms
//    chain without further exchanges: 4 exchanges per tile instead of 8 (+2 for the split halves).
//  * The diagonal Theta factors of the forward transforms: theta^n = theta^i e^{i pi t / N1}, the
//    per-thread theta^i in a register, the per-register part a compile-time rotation (no table); the
//    1/N and c_x are moved onto D'.  d_p and chat_0 (the stash factors) live in shared memory.
//  * The tile arrives by a 1D TMA bulk copy (cp.async.bulk, completion on an mbarrier) into the same
//    shared buffer the exchanges use; the next tile's copy is issued as soon as the last exchange of
//    the current tile has been read, and lands while the current tile finishes its last DFT, the
//    monitor-free epilogue and the stores.  The next tile (and this tile's U_{m-1}) are prefetched
//    into L2 at the start of each tile.
//  * U_{m-1} of the tile (the full-array monitor's copy) is bulk-copied into the same buffer right
//    after the first transform's exchange and lands during its second DFT pass.
//  * D W + H_static (the iteration-invariant static spectrum) is formed when W arrives and parked in
//    tensor memory (TMEM, otherwise idle) until the end of the tile, instead of re-reading W from
//    HBM/L2; the thread's (c_x/N) d'_p values sit in TMEM for the whole kernel (256 columns per CTA).
//  * The four transforms share ONE code body (a forward transform is conj . inverse . conj): a fully
//    unrolled four-transform tile was 13k instructions and stalled on instruction fetch.
// HBM per unknown: W in 16 B, H out 16 B, U_{m-1} in + U_m out 32 B (full monitor) = 64 B.
#pragma once
#include "tpass.cuh"

namespace pint {

// cos(pi n / 32), n = 0..16 (quarter wave; the rest by symmetry; literals: no table in device code)
__host__ __device__ constexpr double cosq32(int n) {
  switch (n) {
    case 0: return 1.0;
    case 1: return 0.9951847266721968862448;
    case 2: return 0.9807852804032304491262;
    case 3: return 0.9569403357322088649358;
    case 4: return 0.9238795325112867561282;
    case 5: return 0.8819212643483550297128;
    case 6: return 0.8314696123025452370788;
    case 7: return 0.7730104533627369608109;
    case 8: return 0.7071067811865475244008;
    case 9: return 0.6343932841636454982152;
    case 10: return 0.5555702330196022247428;
    case 11: return 0.4713967368259976485564;
    case 12: return 0.3826834323650897717285;
    case 13: return 0.2902846772544623676362;
    case 14: return 0.1950903220161282678483;
    case 15: return 0.0980171403295606019942;
    case 16: return 0.0;
  }
  return 0.0;
}
__host__ __device__ constexpr double cos32(int n) {   // cos(pi n / 32), any integer n
  n = ((n % 64) + 64) % 64;
  return n <= 16 ? cosq32(n) : (n <= 32 ? -cosq32(32 - n) : (n <= 48 ? -cosq32(n - 32) : cosq32(64 - n)));
}
__host__ __device__ constexpr double sin32(int n) { return cos32(n - 16); }

// a * e^{i pi m / 32} (m a compile-time constant after unrolling)
__device__ __forceinline__ double2 crot32(double2 a, int m) {
  m = ((m % 64) + 64) % 64;
  if (m == 0) return a;
  if (m == 16) return make_double2(-a.y, a.x);
  if (m == 32) return make_double2(-a.x, -a.y);
  if (m == 48) return make_double2(a.y, -a.x);
  const double c = cos32(m), s = sin32(m);
  return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
}

// b_s = sum_t a_t exp(DIR 2 pi i s t / 32): radix-2 step over two DFT16s (decimation in time)
template <int DIR> __device__ __forceinline__ void dft32(double2* a) {
  double2 e[16], o[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    e[t] = a[2 * t];
    o[t] = a[2 * t + 1];
  }
  dft16<DIR>(e);
  dft16<DIR>(o);
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const double2 w = crot32(o[s], 2 * DIR * s);
    a[s] = cadd(e[s], w);
    a[s + 16] = csub(e[s], w);
  }
}
template <int N1, int DIR> __device__ __forceinline__ void dft_n1(double2* a) {
  if constexpr (N1 == 32) dft32<DIR>(a);
  else dft16<DIR>(a);
}

#ifndef PINT_CQ_STAGGER
#define PINT_CQ_STAGGER 1   // A/B: C5 T-pass 4.19 -> 4.16-4.18 ms (r2_gpu_ab_stag*.sh; after transform 0: 4.34, worse)
#endif
template <int N1> struct CQCfg {
  static constexpr int N = N1 * N1;
  static constexpr int WB = TILE / N;                       // columns per tile
  static constexpr int GT = N1 * WB;                        // threads per tile group: (i, c) = (t / WB, t % WB)
  static constexpr int GROUPS = 2;                          // tile groups per CTA (one CTA per SM)
  static constexpr int THREADS = GROUPS * GT;
  static constexpr int ROW = N1 * WB;                       // exchange row stride (complex; see xidx)
  static constexpr int BUF = TILE;                          // per group: tile landing zone = exchange buffer
  static constexpr int TWROW = N1 + 1;                      // twiddle row stride (padded: conflict-free)
  static constexpr int SCH = 2;                             // chat_s staged in shared memory, s < SCH
  // two tile buffers + the tables both groups share (three pass-A twiddle tables: w^{i k2} and
  // w^{i k2} theta^{-+i} for the two Theta transforms; d_p, chat_0, chat_1): 225.5 KB at N1 = 32
  static constexpr int SMEM = (GROUPS * BUF + 3 * N1 * TWROW + (1 + SCH) * N) * 16;
  static constexpr int TCOLS = 512;                         // all TMEM columns of the SM: per thread N1 complex
                                                            // of stash (D W + H_static) and N1 of (c_x/N) D'
  // exchange slot of (row r, column j): WB = 4 rows XOR-swizzled by the row parity (the 8 threads of a
  // 16-byte wavefront read rows i, i+1 at the same column: the swizzle puts them on disjoint banks)
  static __device__ __forceinline__ int xidx(int r, int j) { return r * ROW + (WB == 4 ? (j ^ ((r & 1) << 2)) : j); }
};

struct CQArgs {
  const double2* in;          // W_m, tile layout [ntiles][N][WB]
  double2* out;               // H_{m+1} (may alias in: a tile is read into shared memory first)
  double2* ufull;             // U_{m-1} -> U_m, every level (tile layout)
  double2* wrap_new;          // [ntiles][k][WB] window levels of U_m
  unsigned long long* upd;    // max |U_m - U_{m-1}| as ordered bits
  const double2* tw;          // [N] pass-A twiddles w^{+i k2} at [i N1 + k2] (every transform runs as an
                              //     inverse 4-step transform; a forward one as conj . inverse . conj)
  const double2* th;          // [N] theta^n = e^{i pi n / N} (the skew-circulant rotation Theta; the kernel
                              //     reads theta^i, i < N1, and rotates by theta^{N1 t} = e^{i pi t / N1})
  const double2* dpr;         // [N] (c_x / N) d'_p: d'_p the eigenvalues of C(-kappa), c_x = -h^2/(2 tau^a N)
                              //     (the 1/N of V^{-1} and c_x of the Theta^{-1} factor, moved onto D')
  const double2* dh;          // [N] (h^2/(2 tau^a)) d_p
  const double2* chat;        // [S][N] DFT of kappa^{n/N} h^2/N c_s(n)  (static right-hand side)
  const double2* src;         // [S][ntiles][WB] spatial sources (DST-x basis)
  const double* igs;          // [N] kappa^{-n/N}: Gamma^{-1} = igs[i] * gt[t] (separable, n = i + N1 t)
  double gt[32];              // kappa^{-N1 t/N}, t < N1 (parameter space; compile-time index)
  int S, k;
  long ntiles;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tile_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  } while (!done);
}

// 4 complex doubles <-> 16 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st4c(uint32_t addr, const double2* x) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    w[4 * j + 0] = (uint32_t)__double2loint(x[j].x); w[4 * j + 1] = (uint32_t)__double2hiint(x[j].x);
    w[4 * j + 2] = (uint32_t)__double2loint(x[j].y); w[4 * j + 3] = (uint32_t)__double2hiint(x[j].y);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
               ::"r"(addr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]) : "memory");
}
__device__ __forceinline__ void tmem_ld4c(uint32_t addr, double2* x) {
  uint32_t w[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                 "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 4; ++j)
    x[j] = make_double2(__hiloint2double((int)w[4 * j + 1], (int)w[4 * j + 0]),
                        __hiloint2double((int)w[4 * j + 3], (int)w[4 * j + 2]));
}

// a <- conj(a) for all N1 values: the sign bit of the imaginary parts (integer pipe)
template <int N1> __device__ __forceinline__ void conj_all(double2 (&v)[N1]) {
#pragma unroll
  for (int t = 0; t < N1; ++t) v[t].y = __longlong_as_double(__double_as_longlong(v[t].y) ^ (long long)0x8000000000000000ULL);
}

// the tile group's barrier (named barrier 1 + g over its GT threads; 0 is __syncthreads)
template <int GT> __device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "n"(GT) : "memory");
}

template <int N1>
__global__ void __launch_bounds__(CQCfg<N1>::THREADS, 1) tpass_cq_fused_kernel(const CQArgs a) {
  using G = CQCfg<N1>;
  constexpr int N = G::N, WB = G::WB, NW = G::THREADS / 32;
  extern __shared__ __align__(128) double2 smem_cq[];
  __shared__ __align__(8) unsigned long long bars[2 * G::GROUPS];   // per group: W tile landed, U_{m-1} landed
  __shared__ uint32_t tbase;
  __shared__ double red[NW];
  const int tid = threadIdx.x, warp = tid / 32, g = tid / G::GT, gtid = tid % G::GT;
  const int i = gtid / WB, c = gtid % WB;
  double2* buf = smem_cq + g * G::BUF;                        // this group's tile / exchange buffer
  const uint32_t sbuf = smem_u32(buf), sbar = smem_u32(&bars[2 * g]), subar = smem_u32(&bars[2 * g + 1]);
  if (tid < 2 * G::GROUPS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bars[tid])) : "memory");
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 ::"r"(smem_u32(&tbase)), "n"(G::TCOLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // the pass-A twiddles, d_p, chat_0 and chat_1, staged once per CTA (persistent kernel) and shared by
  // both groups: conflict-free shared loads (per-tile L2 loads of them stalled the stash, ncu v9/v10)
  double2* stw = smem_cq + G::GROUPS * G::BUF; // [N1][TWROW] w^{i k2}
  double2* stm = stw + N1 * G::TWROW;          // [N1][TWROW] w^{i k2} theta^{-i}  (x = 1)
  double2* stp = stm + N1 * G::TWROW;          // [N1][TWROW] w^{i k2} theta^{+i}  (x = 3)
  double2* sdh = stp + N1 * G::TWROW;          // [N]
  double2* sch = sdh + N;                      // [SCH][N] chat_s, s < min(S, SCH)
  for (int e = tid; e < N; e += G::THREADS) {
    const int r = e / N1, k2 = e % N1;
    const double2 w = __ldg(&a.tw[e]), th = __ldg(&a.th[r]);
    stw[r * G::TWROW + k2] = w;
    stm[r * G::TWROW + k2] = cmul(w, make_double2(th.x, -th.y));
    stp[r * G::TWROW + k2] = cmul(w, th);
    sdh[e] = __ldg(&a.dh[e]);
#pragma unroll
    for (int s = 0; s < G::SCH; ++s)
      if (s < a.S) sch[s * N + e] = __ldg(&a.chat[(long)s * N + e]);
  }
  __syncthreads();
  // this thread's columns: lane 32 (warp % 4) + lane; the warps sharing a lane quarter take 2 N1 * 4
  // columns each: N1 complex of stash, then N1 complex of (c_x/N) d'_p, p = i + N1 t (whole kernel)
  const uint32_t tst = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 2 * N1 * 4);
  const uint32_t tdp = tst + N1 * 4;
#pragma unroll
  for (int q = 0; q < N1 / 4; ++q) {
    double2 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __ldg(&a.dpr[i + N1 * (4 * q + j)]);
    tmem_st4c(tdp + 16 * q, x);
  }
  const double gi0 = __ldg(&a.igs[i]);
  const long ntiles = a.ntiles;
  const long tstride = (long)gridDim.x * G::GROUPS;
  long tile = (long)blockIdx.x * G::GROUPS + g;
  uint32_t phase = 0;
  if (gtid == 0 && tile < ntiles) tile_bulk_load(sbuf, a.in + tile * (long)TILE, TILE * 16, sbar);
  double upd2 = 0.0;                   // max |U_m - U_{m-1}|^2 (one square root at the end)
  bool nonfinite = false;
  PINT_ASSERT(blockDim.x == G::THREADS && i < N1 && c < WB && g < G::GROUPS);
  static_assert(G::TCOLS >= (G::THREADS / 128) * 2 * N1 * 4, "TMEM columns");
  static_assert(N1 * CQCfg<N1>::ROW <= CQCfg<N1>::BUF && TILE <= CQCfg<N1>::BUF, "exchange buffer");
#if PINT_CQ_STAGGER
  // the two tile groups run half a tile apart: group 1 starts when group 0 has finished the second
  // transform of its first tile (one named-barrier hand-off), so that one group's shared-memory phases
  // (tile loads, exchanges) meet the other's FP64 phases instead of their own copies
  bool stag = g == 0;                  // group 0: arrive once
  if (g == 1) asm volatile("bar.sync 3, %0;\n" ::"n"(G::THREADS) : "memory");
#endif
  for (; tile < ntiles; tile += tstride) {
    const long base = tile * (long)TILE, nt = tile + tstride;
    if (gtid < 4) {
      if (nt < ntiles) prefetch_l2_t(a.in + nt * (long)TILE + gtid * (TILE / 4), TILE / 4 * 16);
    } else if (gtid < 8) {                   // this tile's U_{m-1}: its bulk copy (after u = V W) hits L2
      prefetch_l2_t(a.ufull + base + (gtid - 4) * (TILE / 4), TILE / 4 * 16);
    }
    // the tile's spatial sources (issued before the wait: their latency hides behind it)
    const double2* srcp = a.src + tile * WB + c;
    const long sstr = ntiles * WB;
    const double2 g0 = a.S > 0 ? __ldg(&srcp[0]) : make_double2(0.0, 0.0);
    const double2 g1 = a.S > 1 ? __ldg(&srcp[sstr]) : make_double2(0.0, 0.0);
    mbar_wait(sbar, phase);
    phase ^= 1;
    double2 v[N1];
#pragma unroll
    for (int t = 0; t < N1; ++t) v[t] = buf[(i + N1 * t) * WB + c];
    // stash = D W + H_static (frequency p = i + N1 t) -> TMEM, 4 values per tcgen05.st
    {
#pragma unroll
      for (int q = 0; q < N1 / 4; ++q) {
        double2 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int p = i + N1 * (4 * q + j);
          double2 h = cmul(v[4 * q + j], sdh[p]);
          if (a.S > 0) h = cfma(sch[p], g0, h);
          if (a.S > 1) h = cfma(sch[N + p], g1, h);
          x[j] = h;
        }
        tmem_st4c(tst + 16 * q, x);
      }
      if (a.S > G::SCH) {                    // further sources (not staged): read-modify-write of the stash
#pragma unroll 1
        for (int q = 0; q < N1 / 4; ++q) {
          double2 x[4];
          tmem_ld4c(tst + 16 * q, x);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            for (int s = G::SCH; s < a.S; ++s)
              x[j] = cfma(__ldg(&a.chat[(long)s * N + i + N1 * (4 * q + j)]), __ldg(&srcp[s * sstr]), x[j]);
          tmem_st4c(tst + 16 * q, x);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    // ---- the four length-N transforms, ONE code body (instruction-cache footprint), all run as
    // inverse 4-step transforms (a forward one is conj . inverse . conj):
    //   x = 0: u = V W                      -> U_m = Gamma^{-1} u: monitor, U_m -> ufull, window
    //   x = 1: z = V^{-1} Theta u           -> Z = (c_x / N) D' z
    //   x = 2: s = V Z
    //   x = 3: H' = V^{-1} Theta^{-1} s     -> + stash; the buffer is free after its exchange
#pragma unroll 1
    for (int x = 0; x < 4; ++x) {
      const bool fwd = (x & 1) != 0;
      // x = 1: conj(y) theta^{-n} = conj(y theta^{N1 t}) theta^{-i}; x = 3: conj(y) theta^{N1 t} theta^{+i}
      // (theta^n = theta^i theta^{N1 t}): the rotation theta^{N1 t} = e^{i pi t / N1} is a compile-time
      // constant per register, and theta^{-+i}, constant over the pass-A DFT (over t), rides on its twiddles
      if (fwd) {
        if (x == 3) conj_all<N1>(v);
#pragma unroll
        for (int t = 1; t < N1; ++t) v[t] = crot32(v[t], t * (32 / N1));
        if (x == 1) conj_all<N1>(v);
      }
      dft_n1<N1, +1>(v);
      {
        const double2* tr = (x == 1 ? stm : (x == 3 ? stp : stw)) + i * G::TWROW;
        if (fwd) v[0] = cmul(v[0], tr[0]);
#pragma unroll
        for (int k2 = 1; k2 < N1; ++k2) v[k2] = cmul(v[k2], tr[k2]);
      }
      group_sync<G::GT>(g);                  // the buffer is free (previous exchange / tile input read)
#pragma unroll
      for (int k2 = 0; k2 < N1; ++k2) buf[G::xidx(k2, i * WB + c)] = v[k2];
      group_sync<G::GT>(g);
#pragma unroll
      for (int t = 0; t < N1; ++t) v[t] = buf[G::xidx(i, t * WB + c)];
      PINT_ASSERT(G::xidx(N1 - 1, i * WB + c) < G::BUF && G::xidx(i, (N1 - 1) * WB + c) < G::BUF);
      if (x == 0) {                          // U_{m-1} of this tile lands during the pass-B DFT
        group_sync<G::GT>(g);
        if (gtid == 0) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          tile_bulk_load(sbuf, a.ufull + base, TILE * 16, subar);
        }
      } else if (x == 3) {
        group_sync<G::GT>(g);
        if (gtid == 0 && nt < ntiles) {      // the next tile lands while this one finishes
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          tile_bulk_load(sbuf, a.in + nt * (long)TILE, TILE * 16, sbar);
        }
      }
      dft_n1<N1, +1>(v);
      if (fwd) conj_all<N1>(v);
#if PINT_CQ_STAGGER
      if (stag && x == 1) {                 // after the second transform of the first tile
        asm volatile("bar.arrive 3, %0;\n" ::"n"(G::THREADS) : "memory");
        stag = false;
      }
#endif
      if (x == 0) {
        double gi;   // kappa^{-i/N}, through an opaque move per tile: its 32 products with gt[t] would
        asm volatile("mov.b64 %0, %1;" : "=d"(gi) : "d"(gi0));   // otherwise be hoisted and kept live
        mbar_wait(subar, phase ^ 1);         // (phase was flipped after the W wait of this tile)
#pragma unroll
        for (int t = 0; t < N1; ++t) {
          const int n = i + N1 * t;
          const double2 U = cscale(v[t], gi * a.gt[t]);
          const double d2 = cabs2(csub(U, buf[n * WB + c]));
          if (!(d2 <= 1.7976931348623157e308)) nonfinite = true;
          upd2 = fmax(upd2, d2);
          a.ufull[base + (long)n * WB + c] = U;
          PINT_ASSERT(n * WB + c < TILE);
          if (t == N1 - 1 && i >= N1 - a.k) {
            PINT_ASSERT(n - (N - a.k) >= 0 && n - (N - a.k) < a.k);
            a.wrap_new[(tile * a.k + (n - (N - a.k))) * WB + c] = U;
          }
        }
      } else if (x == 1) {
#pragma unroll
        for (int q = 0; q < N1 / 4; ++q) {   // (c_x/N) D' from tensor memory
          double2 dq[4];
          tmem_ld4c(tdp + 16 * q, dq);
#pragma unroll
          for (int j = 0; j < 4; ++j) v[4 * q + j] = cmul(v[4 * q + j], dq[j]);
        }
      }
    }
    // ---- H = H' + D W + H_static ----
    const unsigned long long ef = l2_evict_first();
#pragma unroll
    for (int q = 0; q < N1 / 4; ++q) {
      double2 xs[4];
      tmem_ld4c(tst + 16 * q, xs);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int p = i + N1 * (4 * q + j);
        st_hint(&a.out[base + (long)p * WB + c], cadd(v[4 * q + j], xs[j]), ef);
      }
    }
  }
#if PINT_CQ_STAGGER
  if (stag) asm volatile("bar.arrive 3, %0;\n" ::"n"(G::THREADS) : "memory");   // group 0 had no tile
#endif
  // ---- update monitor: block max, one atomic per CTA; TMEM release ----
  double upd = sqrt(upd2);
  if (nonfinite) upd = __longlong_as_double(0x7ff0000000000000LL);
  for (int o = 16; o > 0; o >>= 1) upd = fmax(upd, __shfl_xor_sync(0xffffffffu, upd, o));
  if ((tid & 31) == 0) red[warp] = upd;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    double m = red[0];
    for (int w = 1; w < NW; ++w) m = fmax(m, red[w]);
    atomicMax(a.upd, (unsigned long long)__double_as_longlong(m));
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(G::TCOLS) : "memory");
}

// CQ bootstrap (pint.cu bootstrap): U_0^n = v (or 0) at every level, H_1 = sum_s chat_s[p] src_s +
// cwhat[p] v elementwise over the tile layout [tile][N][WB] (p = level slot of the H layout)
struct CqBootArgs {
  double2* H;                 // H_1 (tile layout)
  double2* ufull;             // U_0 for the full monitor (may be NULL)
  double2* wrap;              // [ntiles][k][WB] window of U_0
  const double2* src;         // [S][ntiles][WB]
  const double2* cqhat;       // [S][N]
  const double2* cwhat;       // [N]
  int S, zero, k;
  long N, ntiles;
  int WB;
};
#ifdef PINT_DEFINE_PLAIN_KERNELS
__global__ void cq_boot_kernel(const CqBootArgs b) {
  const long total = b.ntiles * (long)TILE;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long tile = e / TILE;
    const int r = (int)(e % TILE), n = r / b.WB, c = r % b.WB;
    const long sstr = b.ntiles * b.WB, so = tile * b.WB + c;
    const double2 v = b.zero ? make_double2(0.0, 0.0) : __ldg(&b.src[so]);
    double2 h = cmul(__ldg(&b.cwhat[n]), v);
    for (int s = 0; s < b.S; ++s) h = cfma(__ldg(&b.cqhat[(long)s * b.N + n]), __ldg(&b.src[s * sstr + so]), h);
    b.H[e] = h;
    if (b.ufull) b.ufull[e] = v;
    if (n >= b.N - b.k) b.wrap[(tile * b.k + (n - (b.N - b.k))) * b.WB + c] = v;
  }
}
#else
__global__ void cq_boot_kernel(const CqBootArgs b);
#endif

}  // namespace pint
