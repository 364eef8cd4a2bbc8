// newton.cu — launchers of the semilinear (Newton-WR) kernels (newton.cuh).
#define PINT_DEFINE_NEWTON_KERNELS
#include "kernels.h"

namespace pint {

static unsigned grid_for(long n, int tpb) {
  const long b = (n + tpb - 1) / tpb;
  return (unsigned)(b < 148L * 16 ? (b > 0 ? b : 1) : 148L * 16);
}

cudaError_t launch_nl_coeff(const NewtonArgs& a, cudaStream_t st) {
  nl_coeff_kernel<<<grid_for(a.L, 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_nl_residual(const NewtonArgs& a, cudaStream_t st) {
  nl_residual_kernel<<<grid_for(a.N * a.L, 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_spass_vc(const VcArgs& a, cudaStream_t st) {
  spass_vc_kernel<<<(unsigned)((a.N + 63) / 64), 64, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_nl_update(double2* U, const double2* W, long N, int L, int WB, unsigned long long* upd,
                             cudaStream_t st) {
  nl_update_kernel<<<grid_for(N * L, 256), 256, 0, st>>>(U, W, N, L, WB, upd);
  return cudaGetLastError();
}
cudaError_t launch_nl_diffmax(const double2* A, const double2* B, long count, unsigned long long* upd,
                              cudaStream_t st) {
  nl_diffmax_kernel<<<grid_for(count, 256), 256, 0, st>>>(A, B, count, upd);
  return cudaGetLastError();
}

cudaError_t launch_imag_max(const double2* A, long count, unsigned long long* upd, cudaStream_t st) {
  imag_max_kernel<<<grid_for(count, 256), 256, 0, st>>>(A, count, upd);
  return cudaGetLastError();
}

cudaError_t launch_modal_div(const SPassArgs& a, const double* mu, long Qb, cudaStream_t st) {
  const long total = Qb * a.NB * a.N * a.WB;
  const long blocks = std::min<long>((total + 255) / 256, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  modal_div_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, mu, total);
  return cudaGetLastError();
}

cudaError_t launch_resid(const ResidArgs& a, cudaStream_t st) {
  const long total = a.Qb * a.NB * a.N * a.WB;
  const long blocks = std::min<long>((total + 255) / 256, 148L * 16);
  if (blocks <= 0) return cudaSuccess;
  resid_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, total);
  return cudaGetLastError();
}

cudaError_t launch_resid_cq_time(const double2* U, double2* T, const double* w, long N, long ntiles,
                                 cudaStream_t st) {
  const int smem = TILE * (int)sizeof(double2);   // one whole tile (fft.cuh TILE) in shared memory
  cudaError_t e = cudaFuncSetAttribute(resid_cq_time_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const long grid = std::min<long>(ntiles, 148L * 3);
  if (grid <= 0) return cudaSuccess;
  resid_cq_time_kernel<<<(unsigned)grid, 256, smem, st>>>(U, T, w, N, ntiles);
  return cudaGetLastError();
}

cudaError_t launch_mode_scale(double2* out, const double2* in, const double* mu, double s, int L, cudaStream_t st) {
  mode_scale_kernel<<<grid_for(L, 256), 256, 0, st>>>(out, in, mu, s, L);
  return cudaGetLastError();
}

}  // namespace pint
