// dispatch.cu — runtime dispatch over the compiled FFT lengths and S-pass chunk sizes.
#define PINT_DEFINE_PLAIN_KERNELS
#include "kernels.h"
#include <algorithm>
#include <cstdlib>

namespace pint {

cudaError_t launch_tpass(int N, int mi, int mo, bool cq, const TPassArgs& a, long ntiles, cudaStream_t st) {
  switch (N) {
    case 16: return launch_tpass_16(mi, mo, cq, a, ntiles, st);
    case 32: return launch_tpass_32(mi, mo, cq, a, ntiles, st);
    case 64: return launch_tpass_64(mi, mo, cq, a, ntiles, st);
    case 128: return launch_tpass_128(mi, mo, cq, a, ntiles, st);
    case 256: return launch_tpass_256(mi, mo, cq, a, ntiles, st);
    case 512: return launch_tpass_512(mi, mo, cq, a, ntiles, st);
    case 1024: return launch_tpass_1024(mi, mo, cq, a, ntiles, st);
    case 2048: return launch_tpass_2048(mi, mo, cq, a, ntiles, st);
    case 4096: return launch_tpass_4096(mi, mo, cq, a, ntiles, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tpass_pruned(int N, const TPassArgs& a, long ntiles, cudaStream_t st) {
  switch (N) {
    case 256: return launch_tpass_pruned_256(a, ntiles, st);
    case 512: return launch_tpass_pruned_512(a, ntiles, st);
    case 1024: return launch_tpass_pruned_1024(a, ntiles, st);
    case 2048: return launch_tpass_pruned_2048(a, ntiles, st);
    case 4096: return launch_tpass_pruned_4096(a, ntiles, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tpass_cq_split(int N, int half, const TPassArgs& a, long ntiles, cudaStream_t st) {
  switch (N) {
    case 16: return launch_tpass_cq_split_16(half, a, ntiles, st);
    case 32: return launch_tpass_cq_split_32(half, a, ntiles, st);
    case 64: return launch_tpass_cq_split_64(half, a, ntiles, st);
    case 128: return launch_tpass_cq_split_128(half, a, ntiles, st);
    case 256: return launch_tpass_cq_split_256(half, a, ntiles, st);
    case 512: return launch_tpass_cq_split_512(half, a, ntiles, st);
    case 1024: return launch_tpass_cq_split_1024(half, a, ntiles, st);
    case 2048: return launch_tpass_cq_split_2048(half, a, ntiles, st);
    case 4096: return launch_tpass_cq_split_4096(half, a, ntiles, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tpass_cq_fused(int N, const CQArgs& a, cudaStream_t st) {
  switch (N) {
    case 256: return launch_tpass_cq_fused_256(a, st);
    case 1024: return launch_tpass_cq_fused_1024(a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dst(int NE, const DstArgs& a, int mode, cudaStream_t st) {
  switch (NE) {
    case 16: return launch_dst_16(a, mode, st);
    case 32: return launch_dst_32(a, mode, st);
    case 64: return launch_dst_64(a, mode, st);
    case 128: return launch_dst_128(a, mode, st);
    case 256: return launch_dst_256(a, mode, st);
    case 512: return launch_dst_512(a, mode, st);
    case 1024: return launch_dst_1024(a, mode, st);
    case 2048: return launch_dst_2048(a, mode, st);
    case 4096: return launch_dst_4096(a, mode, st);
  }
  return cudaErrorInvalidValue;
}

constexpr int SG = 4;   // lines (warps) per S-pass CTA

template <int C>
static cudaError_t spass_go(const SPassArgs& a, long Qb, cudaStream_t st) {
  auto kern = spass_kernel<C, SG>;
  const int off = (a.WB >= 8) ? 0 : (a.WB > 8 / SG ? a.WB : 8 / SG);
  const int smem = SG * (32 * (C + 1) + off) * (int)sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  SPassArgs b = a;
  int lwb = 0;
  while ((1 << lwb) < a.WB) ++lwb;
  int lg = 0;
  while ((1 << lg) < SG) ++lg;
  b.lwb = lwb;
  b.lgw = lwb + lg;
  b.nwork = Qb * (a.N / SG);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * SG, smem);
  const long grid = std::min<long>(b.nwork, (long)nsm * std::max(per, 1));
  kern<<<(unsigned)grid, 32 * SG, smem, st>>>(b);
  return cudaGetLastError();
}

template <int C>
static cudaError_t spass_direct_go(const SPassArgs& a, long Qb, cudaStream_t st) {
  SPassArgs b = a;
  int lwb = 0;
  while ((1 << lwb) < a.WB) ++lwb;
  b.lwb = lwb;
  b.nwork = Qb * a.N;                        // lines
  const long grid = (b.nwork + 3) / 4;
  spass_direct_kernel<C><<<(unsigned)grid, 128, 0, st>>>(b);
  return cudaGetLastError();
}

template <int C>
static cudaError_t spass_pair_go(const SPassArgs& a, long Qb, cudaStream_t st) {
  SPassArgs b = a;
  int lwb = 0;
  while ((1 << lwb) < a.WB) ++lwb;
  b.lwb = lwb;
  b.nwork = Qb * a.N;                        // lines, PINT_PAIR_LPC per CTA
  const long grid = (b.nwork + PINT_PAIR_LPC - 1) / PINT_PAIR_LPC;
  spass_pair_kernel<C><<<(unsigned)grid, 64 * PINT_PAIR_LPC, 0, st>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_spass_const(SPassConst* out, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int L,
                               cudaStream_t st) {
  const long total = N * Qb;
  const long blocks = std::min<long>((total + 127) / 128, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  spass_const_kernel<<<(unsigned)blocks, 128, 0, st>>>(out, sig_p, sig_q, N, Qb, C, L);
  return cudaGetLastError();
}

cudaError_t launch_spass(int C, const SPassArgs& a, long Qb, cudaStream_t st) {
  constexpr bool staged = false, direct = false;   // (the staged strip kernel serves C = 1 and WB = 1)
  // two warps per line (C/2 rows per lane) when the line needs C >= 4 rows per lane
  if (!staged && !direct && a.WB >= 2 && C >= 4 && a.lc) {
    switch (C) {
      case 4: return spass_pair_go<2>(a, Qb, st);
      case 8: return spass_pair_go<4>(a, Qb, st);
      case 16: return spass_pair_go<8>(a, Qb, st);
      case 32: return spass_pair_go<16>(a, Qb, st);
    }
  }
  if (!staged && a.WB >= 2 && C >= 2) {
    switch (C) {
      case 2: return spass_direct_go<2>(a, Qb, st);
      case 4: return spass_direct_go<4>(a, Qb, st);
      case 8: return spass_direct_go<8>(a, Qb, st);
      case 16: return spass_direct_go<16>(a, Qb, st);
      case 32: return spass_direct_go<32>(a, Qb, st);
    }
  }
  switch (C) {
    case 1: return spass_go<1>(a, Qb, st);
    case 2: return spass_go<2>(a, Qb, st);
    case 4: return spass_go<4>(a, Qb, st);
    case 8: return spass_go<8>(a, Qb, st);
    case 16: return spass_go<16>(a, Qb, st);
    case 32: return spass_go<32>(a, Qb, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fem2d(const Fem2dArgs& a, bool init, cudaStream_t st) {
  const long blocks = std::min<long>((a.total + 255) / 256, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  if (init) fem2d_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(a);
  else fem2d_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fem2d_mixed(const double2* Y, double2* Z, long levels, int mx, int my, int NB, int WB, long total,
                               cudaStream_t st) {
  const long blocks = std::min<long>((total + 255) / 256, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  fem2d_mixed_kernel<<<(unsigned)blocks, 256, 0, st>>>(Y, Z, levels, mx, my, NB, WB, total);
  return cudaGetLastError();
}

cudaError_t launch_cq_boot(const CqBootArgs& b, cudaStream_t st) {
  const long total = b.ntiles * (long)TILE;
  const long blocks = std::min<long>((total + 255) / 256, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  cq_boot_kernel<<<(unsigned)blocks, 256, 0, st>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_remap(const RemapArgs& a, int mode, cudaStream_t st) {
  if (a.count <= 0) return cudaSuccess;
  const long blocks = (a.count + 255) / 256;
  remap_kernel<<<(unsigned)(blocks < 148L * 64 ? blocks : 148L * 64), 256, 0, st>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t launch_stencil(const double2* v, double2* Av, int mx, int my, double ihx2, double ihy2, cudaStream_t st) {
  const long M = (long)mx * my;
  const long blocks = (M + 255) / 256;
  stencil_kernel<<<(unsigned)(blocks < 148L * 64 ? blocks : 148L * 64), 256, 0, st>>>(v, Av, mx, my, ihx2, ihy2);
  return cudaGetLastError();
}

}  // namespace pint
