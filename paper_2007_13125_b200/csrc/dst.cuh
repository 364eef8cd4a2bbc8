// dst.cuh — orthonormal DST-I along x (the diagonaliser of the x part of the 2D FD
// Laplacian, A_x = S diag(lambda_q) S, S = S^T = S^{-1}, S_{qi} = sqrt(2/(mx+1)) sin(pi q i/(mx+1)))
// and the layout remaps between the caller's [n][y][x] arrays and the tile-blocked layout.
//
// The DST-x commutes with every time-axis step (wrap, scale, time DFT, unscale are per spatial
// point and linear), so it is hoisted out of the WR loop: applied once to v, A v, g_r (and a
// user initial guess) and once to the requested output levels.
// DST-I of length mx via the complex FFT of the odd extension z (length NE = 2(mx+1)):
//   z_0 = z_{mx+1} = 0, z_i = x_{i-1}, z_{NE-i} = -x_{i-1};  X_{q-1} = sqrt(2/(mx+1)) (i/2) Z_q.
#pragma once
#include "fft.cuh"

namespace pint {

enum { DST_PHYS_TO_SRC = 0, DST_PHYS_LEVELS_TO_INT = 1, DST_INT_TO_PHYS_LEVELS = 2, DST_ROWS = 3, DST_INT_TO_INT = 4,
       // along y inside the tile layout [q][yb][N][WB] (fully modal path): row = q * N + level,
       // element y (transform length a.mx := my)
       DST_TILE_Y = 5 };

struct DstArgs {
  const double2* in;
  double2* out;
  long rows;        // number of length-mx rows to transform
  int mx, my, WB;
  long NB, N, q0, Qb, n0, M;
  double scale;     // sqrt(2/(mx+1))
  const double2* tw;  // [NE] exp(-2 pi i m/NE)
};

__device__ __forceinline__ long dst_in_index(const DstArgs& a, int mode, long row, int x) {
  if (mode == DST_PHYS_TO_SRC) return row * a.mx + x;
  if (mode == DST_PHYS_LEVELS_TO_INT) return (row / a.my) * a.M + (row % a.my) * a.mx + x;
  if (mode == DST_TILE_Y) {
    const long qq = row / a.N, nl = row % a.N;
    return ((qq * a.NB + x / a.WB) * a.N + nl) * a.WB + x % a.WB;
  }
  if (mode == DST_INT_TO_PHYS_LEVELS || mode == DST_INT_TO_INT) {
    const long nl = row / a.my, y = row % a.my;
    return (((long)x * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB;
  }
  return row * a.mx + x;
}
// returns -1 when the mode index is outside this rank's slab
__device__ __forceinline__ long dst_out_index(const DstArgs& a, int mode, long row, int q) {
  if (mode == DST_PHYS_TO_SRC) {
    const long ql = q - a.q0;
    if (ql < 0 || ql >= a.Qb) return -1;
    return (ql * a.NB + row / a.WB) * a.WB + row % a.WB;
  }
  if (mode == DST_PHYS_LEVELS_TO_INT) {
    const long ql = q - a.q0;
    if (ql < 0 || ql >= a.Qb) return -1;
    const long nl = row / a.my, y = row % a.my;
    return ((ql * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB;
  }
  if (mode == DST_INT_TO_PHYS_LEVELS) return (row / a.my) * a.M + (row % a.my) * a.mx + q;
  if (mode == DST_TILE_Y) {
    const long qq = row / a.N, nl = row % a.N;
    return ((qq * a.NB + q / a.WB) * a.N + nl) * a.WB + q % a.WB;
  }
  if (mode == DST_INT_TO_INT) {   // tile layout, x index -> mode index (per-iteration DST ablation)
    const long nl = row / a.my, y = row % a.my;
    return (((long)q * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB;
  }
  return row * a.mx + q;
}

template <int NE>
__global__ void __launch_bounds__(TPB) dst_kernel(const DstArgs a, int mode) {
  using TM = TimeMap<NE>;
  using FM = FreqMap<NE>;
  constexpr int RB = TILE / NE;
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int c = tid % RB;
  const long row = (long)blockIdx.x * RB + c;
  const bool valid = row < a.rows;
  double2 v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int i = FM::p(t, tid);
    double2 z = make_double2(0.0, 0.0);
    if (valid) {
      if (i >= 1 && i <= a.mx) z = a.in[dst_in_index(a, mode, row, i - 1)];
      else if (i >= a.mx + 2) {
        const double2 x = a.in[dst_in_index(a, mode, row, NE - i - 1)];
        z = make_double2(-x.x, -x.y);
      }
    }
    v[t] = z;
  }
  run_passes<NE, -1, false>(v, sm, a.tw, tid);
  if (!valid) return;
#pragma unroll
  for (int j = 0; j < TM::NJ; ++j)
#pragma unroll
    for (int s = 0; s < TM::RL; ++s) {
      const int q = TM::n(j, s, tid);
      if (q >= 1 && q <= a.mx && TM::c(j, tid) == c) {
        const long o = dst_out_index(a, mode, row, q - 1);
        const double2 Z = v[j * TM::RL + s];
        if (o >= 0) a.out[o] = make_double2(-0.5 * a.scale * Z.y, 0.5 * a.scale * Z.x);
      }
    }
}

// ---- plain gathers (1D layouts, modal slab export) ----
enum { RM_1D_LEVELS_TO_INT = 0, RM_INT_TO_1D_LEVELS = 1, RM_INT_TO_MODAL = 2, RM_1D_TO_SRC = 3,
       // 2D physical-x layouts (no DST: per-iteration DST ablation, PINT_FLAG_DST_PER_ITER)
       RM_2D_PHYS_TO_SRC = 4, RM_2D_LEVELS_TO_INT = 5, RM_INT_TO_2D_LEVELS = 6 };
struct RemapArgs {
  const double2* in;
  double2* out;
  long count;   // elements to produce
  int WB, my;
  long NB, N, n0, M, Qb;
};
#ifdef PINT_DEFINE_PLAIN_KERNELS
__global__ void remap_kernel(const RemapArgs a, int mode) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < a.count; e += (long)gridDim.x * blockDim.x) {
    if (mode == RM_1D_LEVELS_TO_INT) {
      const long nl = e / a.M, y = e % a.M;
      a.out[((y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB] = a.in[e];
    } else if (mode == RM_INT_TO_1D_LEVELS) {
      const long nl = e / a.M, y = e % a.M;
      a.out[e] = a.in[((y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB];
    } else if (mode == RM_INT_TO_MODAL) {
      const long ql = e % a.Qb, r = e / a.Qb, y = r % a.my, nl = r / a.my;
      a.out[e] = a.in[((ql * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB];
    } else if (mode == RM_2D_PHYS_TO_SRC || mode == RM_2D_LEVELS_TO_INT || mode == RM_INT_TO_2D_LEVELS) {
      const long mx = a.M / a.my;
      const long nl = e / a.M, r = e % a.M, y = r / mx, x = r % mx;
      if (mode == RM_2D_PHYS_TO_SRC) a.out[(x * a.NB + y / a.WB) * a.WB + y % a.WB] = a.in[e];
      else if (mode == RM_2D_LEVELS_TO_INT) a.out[((x * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB] = a.in[e];
      else a.out[e] = a.in[((x * a.NB + y / a.WB) * a.N + a.n0 + nl) * a.WB + y % a.WB];
    } else {  // RM_1D_TO_SRC: src tile layout [NB][WB] of one vector == identity with padding
      a.out[e] = a.in[e];
    }
  }
}

// A v with the 3-point (my == 1) or 5-point stencil, zero Dirichlet data; physical layout.
__global__ void stencil_kernel(const double2* __restrict__ v, double2* __restrict__ Av, int mx, int my,
                               double ihx2, double ihy2) {
  const long M = (long)mx * my;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < M; e += (long)gridDim.x * blockDim.x) {
    const int x = e % mx, y = e / mx;
    const double2 c = v[e];
    const double2 l = x > 0 ? v[e - 1] : make_double2(0, 0);
    const double2 r = x < mx - 1 ? v[e + 1] : make_double2(0, 0);
    double2 o = make_double2((2 * c.x - l.x - r.x) * ihx2, (2 * c.y - l.y - r.y) * ihx2);
    if (my > 1) {
      const double2 d = y > 0 ? v[e - mx] : make_double2(0, 0);
      const double2 u = y < my - 1 ? v[e + mx] : make_double2(0, 0);
      o.x += (2 * c.x - d.x - u.x) * ihy2;
      o.y += (2 * c.y - d.y - u.y) * ihy2;
    }
    Av[e] = o;
  }
}
#endif  // PINT_DEFINE_PLAIN_KERNELS

}  // namespace pint
