// inst_n.cu — per-FFT-length instantiation unit; compiled once per PINT_N (build.py).
#include "kernels.h"

#ifndef PINT_N
#error "define PINT_N"
#endif
#define PINT_CAT2(a, b) a##b
#define PINT_CAT(a, b) PINT_CAT2(a, b)

namespace pint {

// opt in to `smem` bytes of dynamic shared memory and return SMs x resident CTAs (0 on error)
static long persistent_grid(const void* kern, int smem, int threads = TPB) {
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem);
  return (long)nsm * (per > 0 ? per : 1);
}

template <int MI, int MO, bool CQ, bool FD = false>
static cudaError_t go(const TPassArgs& a, long ntiles, cudaStream_t st) {
  auto kern = tpass_kernel<PINT_N, MI, MO, CQ, FD>;
  const int smem = phys_size(TILE) * (int)sizeof(double2);
  // persistent grid: SMs x resident CTAs per SM (thread-safe one-time init; one device per process)
  static const long resident = persistent_grid((const void*)kern, smem);
  if (resident <= 0) return cudaErrorInvalidValue;
  if (ntiles <= 0) return cudaSuccess;
  const long grid = ntiles < resident ? ntiles : resident;
  kern<<<(unsigned)grid, TPB, smem, st>>>(a, ntiles);
  return cudaGetLastError();
}

#if PINT_N >= 256
template <bool DENSE>
static cudaError_t go_pruned(const TPassArgs& a, long ntiles, cudaStream_t st) {
  auto kern = tpass_heat_pruned_kernel<PINT_N, DENSE>;
  constexpr int WBp = TILE / PINT_N;
  const int smem = (WBp * (9 * (PINT_N / 16) + 1) + WBp * (PINT_N / 256) * 16 + 16 * WBp + WBp * 16) * (int)sizeof(double2);
  static const long resident = persistent_grid((const void*)kern, smem);
  if (resident <= 0) return cudaErrorInvalidValue;
  if (ntiles <= 0) return cudaSuccess;
  const long grid = ntiles < resident ? ntiles : resident;
  kern<<<(unsigned)grid, TPB, smem, st>>>(a, ntiles);
  return cudaGetLastError();
}
#endif

template <bool B>
static cudaError_t go_cq_split(const TPassArgs& a, long ntiles, cudaStream_t st) {
  auto kern = B ? tpass_cq_b_kernel<PINT_N> : tpass_cq_a_kernel<PINT_N>;
  const int smem = phys_size(TILE) * (int)sizeof(double2);
  static const long resident = persistent_grid((const void*)kern, smem);
  if (resident <= 0) return cudaErrorInvalidValue;
  if (ntiles <= 0) return cudaSuccess;
  const long grid = ntiles < resident ? ntiles : resident;
  kern<<<(unsigned)grid, TPB, smem, st>>>(a, ntiles);
  return cudaGetLastError();
}

cudaError_t PINT_CAT(launch_tpass_cq_fused_, PINT_N)(const CQArgs& a, cudaStream_t st) {
#if PINT_N == 1024 || PINT_N == 256
  constexpr int N1 = PINT_N == 1024 ? 32 : 16;
  using G = CQCfg<N1>;
  auto kern = tpass_cq_fused_kernel<N1>;
  // persistent grid of one CTA per SM (two tile groups; 191.5 KB of shared memory and all 512 TMEM
  // columns) with a shared-memory carve-out of just what it needs: the rest stays L1
  static const long resident = [&]() -> long {
    const int need = G::SMEM + 1024 + 256;
    const int pct = (int)((100LL * need + 233471) / 233472);
    if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct) != cudaSuccess)
      return 0;
    if (persistent_grid((const void*)kern, G::SMEM, G::THREADS) <= 0) return 0;   // sets the smem attribute
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (long)nsm;
  }();
  if (resident <= 0) return cudaErrorInvalidValue;
  if (a.ntiles <= 0) return cudaSuccess;
  const long want = (a.ntiles + G::GROUPS - 1) / G::GROUPS;
  const long grid = want < resident ? want : resident;
  kern<<<(unsigned)grid, G::THREADS, G::SMEM, st>>>(a);
  return cudaGetLastError();
#else
  (void)a; (void)st;
  return cudaErrorInvalidValue;
#endif
}

cudaError_t PINT_CAT(launch_tpass_cq_split_, PINT_N)(int half, const TPassArgs& a, long ntiles, cudaStream_t st) {
  return half ? go_cq_split<true>(a, ntiles, st) : go_cq_split<false>(a, ntiles, st);
}

cudaError_t PINT_CAT(launch_tpass_pruned_, PINT_N)(const TPassArgs& a, long ntiles, cudaStream_t st) {
#if PINT_N >= 256
  return a.ndense > 0 ? go_pruned<true>(a, ntiles, st) : go_pruned<false>(a, ntiles, st);
#else
  (void)a; (void)ntiles; (void)st;
  return cudaErrorInvalidValue;
#endif
}

// dense right-hand side (a.fdense: pint_set_problem with the streaming path, Newton inner solves)
template <bool CQ>
static cudaError_t go_fd(int mi, const TPassArgs& a, long ntiles, cudaStream_t st) {
  switch (mi) {
    case IN_FREQ: return go<IN_FREQ, OUT_H, CQ, true>(a, ntiles, st);
    case IN_TIME_V: return go<IN_TIME_V, OUT_H, CQ, true>(a, ntiles, st);
    case IN_TIME_ZERO: return go<IN_TIME_ZERO, OUT_H, CQ, true>(a, ntiles, st);
    default: return go<IN_TIME_BUF, OUT_H, CQ, true>(a, ntiles, st);
  }
}

cudaError_t PINT_CAT(launch_tpass_, PINT_N)(int mi, int mo, bool cq, const TPassArgs& a, long ntiles, cudaStream_t st) {
  if (mo == OUT_U) return go<IN_FREQ, OUT_U, false>(a, ntiles, st);
  if (a.fdense) return cq ? go_fd<true>(mi, a, ntiles, st) : go_fd<false>(mi, a, ntiles, st);
  if (!cq) {
    switch (mi) {
      case IN_FREQ: return go<IN_FREQ, OUT_H, false>(a, ntiles, st);
      case IN_TIME_V: return go<IN_TIME_V, OUT_H, false>(a, ntiles, st);
      case IN_TIME_ZERO: return go<IN_TIME_ZERO, OUT_H, false>(a, ntiles, st);
      default: return go<IN_TIME_BUF, OUT_H, false>(a, ntiles, st);
    }
  }
  switch (mi) {
    case IN_FREQ: return go<IN_FREQ, OUT_H, true>(a, ntiles, st);
    case IN_TIME_V: return go<IN_TIME_V, OUT_H, true>(a, ntiles, st);
    case IN_TIME_ZERO: return go<IN_TIME_ZERO, OUT_H, true>(a, ntiles, st);
    default: return go<IN_TIME_BUF, OUT_H, true>(a, ntiles, st);
  }
}

cudaError_t PINT_CAT(launch_dst_, PINT_N)(const DstArgs& a, int mode, cudaStream_t st) {
  auto kern = dst_kernel<PINT_N>;
  const int smem = phys_size(TILE) * (int)sizeof(double2);
  static const long ok = persistent_grid((const void*)kern, smem);   // sets the smem attribute once
  if (ok <= 0) return cudaErrorInvalidValue;
  const long rb = TILE / PINT_N;
  const long blocks = (a.rows + rb - 1) / rb;
  if (blocks <= 0) return cudaSuccess;
  kern<<<(unsigned)blocks, TPB, smem, st>>>(a, mode);
  return cudaGetLastError();
}

}  // namespace pint
