// fused.cu — launchers of the fused heat iteration (fused.cuh).
#define PINT_DEFINE_FUSED_KERNELS
#include "kernels.h"

namespace pint {

size_t fused_smem_bytes(int C, int k) { return (size_t)(FG + k) * 32 * C * sizeof(double2); }

template <int C, bool SW>
static cudaError_t fused_go(const FusedArgs& a, long grid, cudaStream_t st) {
  auto kern = wr_fused_kernel<C, SW>;
  const size_t smem = fused_smem_bytes(C, a.k);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, FT, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool SW>
static cudaError_t fused_sw(int C, const FusedArgs& a, long grid, cudaStream_t st) {
  switch (C) {
    case 1: return fused_go<1, SW>(a, grid, st);
    case 2: return fused_go<2, SW>(a, grid, st);
    case 4: return fused_go<4, SW>(a, grid, st);
    case 8: return fused_go<8, SW>(a, grid, st);
    case 16: return fused_go<16, SW>(a, grid, st);
    case 32: return fused_go<32, SW>(a, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fused(int C, bool store_w, const FusedArgs& a, cudaStream_t st) {
  const long grid = a.Qb * a.nch;
  return store_w ? fused_sw<true>(C, a, grid, st) : fused_sw<false>(C, a, grid, st);
}

template <int C>
static int fused_occ(int k) {
  int per = 0;
  const size_t smem = fused_smem_bytes(C, k);
  cudaFuncSetAttribute(wr_fused_kernel<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wr_fused_kernel<C, false>, FT, smem) != cudaSuccess) return 0;
  return per;
}

int fused_ctas_per_sm(int C, int k) {
  switch (C) {
    case 1: return fused_occ<1>(k);
    case 2: return fused_occ<2>(k);
    case 4: return fused_occ<4>(k);
    case 8: return fused_occ<8>(k);
    case 16: return fused_occ<16>(k);
    case 32: return fused_occ<32>(k);
  }
  return 0;
}

cudaError_t launch_finish(const FinishArgs& a, int mode, cudaStream_t st) {
  const long total = a.Qb * a.Lf;
  const long blocks = std::min<long>((total + TPB - 1) / TPB, 148L * 8);
  if (blocks <= 0) return cudaSuccess;
  wr_finish_kernel<<<(unsigned)blocks, TPB, 0, st>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t launch_line_const(LineConst* lc, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int L,
                              cudaStream_t st) {
  const long total = N * Qb;
  const long blocks = std::min<long>((total + 127) / 128, 148L * 16);
  line_const_kernel<<<(unsigned)blocks, 128, 0, st>>>(lc, sig_p, sig_q, N, Qb, C, L);
  return cudaGetLastError();
}

}  // namespace pint
