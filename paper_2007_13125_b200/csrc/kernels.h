// kernels.h — host-side launch interface of the device kernels (one .cu per FFT length).
#pragma once
#include <cuda_runtime.h>
#include "tpass.cuh"
#include "spass.cuh"
#include "dst.cuh"
#include "fused.cuh"
#include "newton.cuh"
#include "cqpass.cuh"
#include "fem2d.cuh"
#include <algorithm>

namespace pint {

// T-pass for FFT length N (power of two, 16..4096); returns the launch error.
cudaError_t launch_tpass(int N, int mode_in, int mode_out, bool cq, const TPassArgs& a, long ntiles, cudaStream_t st);
// S-pass: chunk C = ceil(L/32) rounded up to a power of two (1..32), G lines per CTA.
cudaError_t launch_spass(int C, const SPassArgs& a, long Qb, cudaStream_t st);
// plan time: pair S-pass line constants for C rows per lane (spass.cuh)
cudaError_t launch_spass_const(SPassConst* out, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int L,
                               cudaStream_t st);
// pruned heat T-pass (FREQ -> H), N in {512, 1024, 2048, 4096}
cudaError_t launch_tpass_pruned(int N, const TPassArgs& a, long ntiles, cudaStream_t st);
// CQ FREQ -> H as two kernels (half 0: W -> Z, half 1: Z, W -> H; tpass.cuh)
cudaError_t launch_tpass_cq_split(int N, int half, const TPassArgs& a, long ntiles, cudaStream_t st);
// CQ FREQ -> H as one kernel (cqpass.cuh), N in {256, 1024}; UNSUPPORTED lengths return cudaErrorInvalidValue
cudaError_t launch_tpass_cq_fused(int N, const CQArgs& a, cudaStream_t st);
// 2D P1-FEM Step 2 (fem2d.cuh, dispatch.cu): fixed-point init / step, the mixed stencil Dx Dy / 24
cudaError_t launch_fem2d(const Fem2dArgs& a, bool init, cudaStream_t st);
cudaError_t launch_fem2d_mixed(const double2* Y, double2* Z, long levels, int mx, int my, int NB, int WB, long total,
                               cudaStream_t st);
// CQ bootstrap: U_0 and H_1 elementwise from the separable sources (cqpass.cuh, dispatch.cu)
cudaError_t launch_cq_boot(const CqBootArgs& b, cudaStream_t st);
// layout remaps and the FD stencil (dispatch.cu)
cudaError_t launch_remap(const RemapArgs& a, int mode, cudaStream_t st);
cudaError_t launch_stencil(const double2* v, double2* Av, int mx, int my, double ihx2, double ihy2, cudaStream_t st);
// DST-I rows, extended FFT length NE = 2(mx+1).
cudaError_t launch_dst(int NE, const DstArgs& a, int mode, cudaStream_t st);
// fused heat iteration (fused.cu): one CTA per (x-mode, group chunk); lanes (32 | 64) per line,
// C rows per lane
size_t fused_smem_bytes(int lanes, int C, int k, bool tm);
int fused_ctas_per_sm(int lanes, int C, int k, bool tm);
int fused_rows_per_subchain(int lanes, int C);
cudaError_t launch_fused(int lanes, int C, bool store_w, bool tm, const FusedArgs& a, cudaStream_t st);
cudaError_t launch_finish(const FinishArgs& a, int mode, cudaStream_t st);
// the whole WR loop as one cooperative kernel (small fused problems; fused.cu): capacity != NULL only
// queries the number of co-resident CTAs
cudaError_t launch_loop_kernel(int C, int nk, const LoopKArgs& L, long grid, int k, cudaStream_t st, int* capacity);
// device-side WR loop: the stopping rule after each iteration, sets the while-node condition (fused.cu)
cudaError_t launch_loop_ctl(LoopCtl* s, const unsigned long long* upd, cudaGraphConditionalHandle h, cudaStream_t st);
// fully modal variant (PINT_FLAG_MODAL): one warp per (x-mode, y-mode)
cudaError_t launch_modal(bool store_w, const FusedArgs& a, cudaStream_t st);
// semilinear extension (newton.cu): Newton coefficient, residual, variable-coefficient line solves
cudaError_t launch_nl_coeff(const NewtonArgs& a, cudaStream_t st);
cudaError_t launch_nl_residual(const NewtonArgs& a, cudaStream_t st);
cudaError_t launch_spass_vc(const VcArgs& a, cudaStream_t st);
cudaError_t launch_nl_update(double2* U, const double2* W, long N, int L, int WB, unsigned long long* upd,
                             cudaStream_t st);
cudaError_t launch_imag_max(const double2* A, long count, unsigned long long* upd, cudaStream_t st);
// streaming modal path: W = H / (sig_p + sig_q + mu_j) over the tile layout (Step 2 as a division)
cudaError_t launch_modal_div(const SPassArgs& a, const double* mu, long Qb, cudaStream_t st);
// fixed-point residual of the heat scheme for the materialised iterate (newton.cuh)
cudaError_t launch_resid(const ResidArgs& a, cudaStream_t st);
cudaError_t launch_resid_cq_time(const double2* U, double2* T, const double* w, long N, long ntiles, cudaStream_t st);
// out[j] = in[j] mu[j] s, j < L (modal-basis operator application: P1-FEM A v)
cudaError_t launch_mode_scale(double2* out, const double2* in, const double* mu, double s, int L, cudaStream_t st);
cudaError_t launch_nl_diffmax(const double2* A, const double2* B, long count, unsigned long long* upd,
                              cudaStream_t st);
cudaError_t launch_line_const(LineConst* lc, const double2* sig_p, const double* sig_q, long N, long Qb, int C, int CS,
                              int L, cudaStream_t st);

#define PINT_DECLARE_N(NN)                                                                         \
  cudaError_t launch_tpass_##NN(int mode_in, int mode_out, bool cq, const TPassArgs& a, long ntiles, \
                                cudaStream_t st);                                                  \
  cudaError_t launch_dst_##NN(const DstArgs& a, int mode, cudaStream_t st);                    \
  cudaError_t launch_tpass_pruned_##NN(const TPassArgs& a, long ntiles, cudaStream_t st);        \
  cudaError_t launch_tpass_cq_split_##NN(int half, const TPassArgs& a, long ntiles, cudaStream_t st);  \
  cudaError_t launch_tpass_cq_fused_##NN(const CQArgs& a, cudaStream_t st);
PINT_DECLARE_N(16)
PINT_DECLARE_N(32)
PINT_DECLARE_N(64)
PINT_DECLARE_N(128)
PINT_DECLARE_N(256)
PINT_DECLARE_N(512)
PINT_DECLARE_N(1024)
PINT_DECLARE_N(2048)
PINT_DECLARE_N(4096)
#undef PINT_DECLARE_N

}  // namespace pint
