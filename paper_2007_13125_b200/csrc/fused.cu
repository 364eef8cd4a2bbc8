// fused.cu — launchers of the fused heat iteration (fused.cuh).
#define PINT_DEFINE_FUSED_KERNELS
#include "kernels.h"

namespace pint {

size_t fused_smem_bytes(int lanes, int C, int k, bool tm) {
  return (size_t)(FG + (tm ? 0 : k)) * lanes * C * sizeof(double2) + 8 * sizeof(LineConst) +
         (lanes == 64 ? 8 * 4 * sizeof(double2) : 0);
}

using FusedKern = void (*)(const FusedArgs);

// hot instantiation: real-data variant and the compile-time nk bound (one warp per line only)
template <int C, int LANES, bool HALF>
static FusedKern fused_pick(int nk) {
  if constexpr (LANES == 32) {
    if (nk <= 4) return wr_fused_kernel<C, LANES, false, true, HALF, 4>;
    if (nk <= 6) return wr_fused_kernel<C, LANES, false, true, HALF, 6>;
  }
  return wr_fused_kernel<C, LANES, false, true, HALF, 8>;
}

template <int C, int LANES, bool SW, bool TM>
static cudaError_t fused_go(const FusedArgs& a, long grid, cudaStream_t st) {
  FusedKern kern = wr_fused_kernel<C, LANES, SW, TM>;
  if constexpr (TM && !SW) kern = a.half ? fused_pick<C, LANES, true>(a.nk) : fused_pick<C, LANES, false>(a.nk);
  // X staged in shared memory only by the shared-memory-window variant (the TMEM kernels keep X in TMEM)
  const size_t smem = fused_smem_bytes(LANES, C, a.k, TM && !SW) + ((a.xs && !(TM && !SW)) ? (size_t)a.nk * LANES * C * sizeof(double2) : 0);
  // set on every launch: the occupancy query at plan creation (fused_occ) also sets this attribute
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, FCfg<LANES>::THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

template <int LANES, bool SW, bool TM>
static cudaError_t fused_c(int C, const FusedArgs& a, long grid, cudaStream_t st) {
  switch (C) {
    case 1: return fused_go<1, LANES, SW, TM>(a, grid, st);
    case 2: return fused_go<2, LANES, SW, TM>(a, grid, st);
    case 4: return fused_go<4, LANES, SW, TM>(a, grid, st);
    case 8: return fused_go<8, LANES, SW, TM>(a, grid, st);
    case 16: return fused_go<16, LANES, SW, TM>(a, grid, st);
    case 32: if constexpr (LANES == 32) return fused_go<32, LANES, SW, TM>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fused(int lanes, int C, bool store_w, bool tm, const FusedArgs& a, cudaStream_t st) {
  // one warp per line; iteration launches keep the window sums in TMEM, the materialising launch
  // (store_w) has no window
  if (lanes != 32 || !(tm || store_w)) return cudaErrorInvalidValue;
  const long grid = a.Qb * a.nch;
  if (store_w) return fused_c<32, true, false>(C, a, grid, st);
  return fused_c<32, false, true>(C, a, grid, st);
}

template <int C, int LANES>
static int fused_occ(int k, bool tm) {
  int per = 0;
  const size_t smem = fused_smem_bytes(LANES, C, k, tm);
  if (!tm) return 0;
  auto kern = wr_fused_kernel<C, LANES, false, true>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, FCfg<LANES>::THREADS, smem) != cudaSuccess) return 0;
  return per;
}

template <int LANES>
static int fused_occ_c(int C, int k, bool tm) {
  switch (C) {
    case 1: return fused_occ<1, LANES>(k, tm);
    case 2: return fused_occ<2, LANES>(k, tm);
    case 4: return fused_occ<4, LANES>(k, tm);
    case 8: return fused_occ<8, LANES>(k, tm);
    case 16: return fused_occ<16, LANES>(k, tm);
    case 32: if constexpr (LANES == 32) return fused_occ<32, LANES>(k, tm);
  }
  return 0;
}

// resident CTAs per SM; with the window sums (and X) in TMEM each CTA allocates its columns, so at
// most 512 / columns of them (C <= 16: 256 columns, two CTAs)
int fused_ctas_per_sm(int lanes, int C, int k, bool tm) {
  if (lanes != 32) return 0;
  const int per = fused_occ_c<32>(C, k, tm);
  if (!tm) return per;
  const int cols = lanes == 32 && C <= 16 ? 256 : 512;
  return std::min(per, 512 / cols);
}

int fused_rows_per_subchain(int lanes, int C) {
  const int nsmax = lanes == 32 ? PINT_FUSED_NS : 2;
  return C / (C < nsmax ? C : nsmax);
}

cudaError_t launch_modal(bool store_w, const FusedArgs& a, cudaStream_t st) {
  const long warps = a.Qb * (long)a.L;
  const long blocks = (warps * 32 + 255) / 256;
  if (blocks <= 0) return cudaSuccess;
  if (store_w) wr_modal_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(a);
  else wr_modal_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_finish(const FinishArgs& a0, int mode, cudaStream_t st) {
  FinishArgs a = a0;
  // many chunks, or several chunks of a small problem: warp per row (lanes over the chunks)
  if (mode == FIN_PARTIALS && (a.nch > 16 || (a.nch >= 2 && a.Qb * (long)a.Lf <= 4096))) {
    const long blocks = (a.Qb * (long)a.Lf * 32 + TPB - 1) / TPB;
    wr_reduce_finish_kernel<<<(unsigned)blocks, TPB, 0, st>>>(a);
    return cudaGetLastError();
  }
  const long total = a.Qb * a.Lf;
  const long blocks = std::min<long>((total + TPB - 1) / TPB, 148L * 8);
  if (blocks <= 0) return cudaSuccess;
  wr_finish_kernel<<<(unsigned)blocks, TPB, 0, st>>>(a, mode);
  return cudaGetLastError();
}

// one thread: the stopping rule after the monitor (fully modal plans; otherwise the finish kernel's
// last block does it, finish_loop_tail)
__global__ void wr_loop_ctl_kernel(LoopCtl* s, const unsigned long long* upd, cudaGraphConditionalHandle h) {
  loop_ctl_step(s, __longlong_as_double((long long)*upd), h);
}

// the cooperative whole-loop kernel (fused.cuh wr_loop_kernel): NKC 4 or 8
template <int C, int NKC>
static cudaError_t loop_go(const LoopKArgs& L, long grid, int k, cudaStream_t st, int* capacity) {
  auto kern = wr_loop_kernel<C, NKC>;
  const size_t smem = fused_smem_bytes(32, C, k, true);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (capacity) {   // co-resident CTAs on this device (the cooperative launch requires grid <= it)
    int per = 0, dev = 0, nsm = 148;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, FG * 32, smem);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    *capacity = per * nsm;
    return cudaSuccess;
  }
  void* args[] = {(void*)&L};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(FG * 32), args, smem, st);
}

template <int NKC>
static cudaError_t loop_c(int C, const LoopKArgs& L, long grid, int k, cudaStream_t st, int* capacity) {
  switch (C) {
    case 1: return loop_go<1, NKC>(L, grid, k, st, capacity);
    case 2: return loop_go<2, NKC>(L, grid, k, st, capacity);
    case 4: return loop_go<4, NKC>(L, grid, k, st, capacity);
    case 8: return loop_go<8, NKC>(L, grid, k, st, capacity);
    case 16: return loop_go<16, NKC>(L, grid, k, st, capacity);
    case 32: return loop_go<32, NKC>(L, grid, k, st, capacity);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_loop_kernel(int C, int nk, const LoopKArgs& L, long grid, int k, cudaStream_t st, int* capacity) {
  return nk <= 4 ? loop_c<4>(C, L, grid, k, st, capacity) : loop_c<8>(C, L, grid, k, st, capacity);
}

cudaError_t launch_loop_ctl(LoopCtl* s, const unsigned long long* upd, cudaGraphConditionalHandle h, cudaStream_t st) {
  wr_loop_ctl_kernel<<<1, 1, 0, st>>>(s, upd, h);
  return cudaGetLastError();
}

cudaError_t launch_line_const(LineConst* lc, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int CS,
                              int L, cudaStream_t st) {
  const long total = N * Qb;
  const long blocks = std::min<long>((total + 127) / 128, 148L * 16);
  line_const_kernel<<<(unsigned)blocks, 128, 0, st>>>(lc, sig_p, sig_q, N, Qb, C, CS, L);
  return cudaGetLastError();
}

}  // namespace pint
