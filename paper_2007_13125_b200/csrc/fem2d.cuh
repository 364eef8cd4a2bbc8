// fem2d.cuh — Step 2 for the paper's own 2D discretisation: P1 finite elements
// on the uniform triangulation of the unit square (Example 3 PAPER.md:1567-1575), each
// cell split by its '/' diagonal (reading R-FEM2D).  With h = 1/(m+1) and the interior nodes,
//   K = -Delta_h h^2 (5-point; right triangles have no diagonal couplings),
//   M = h^2 [ M_sym + E ],  M_sym = (6 + Tx + Ty + Tx Ty / 2) / 12,  E = Dx Dy / 24,
// T = S + S^T, D = S - S^T (S the zero-padded shift).  K and M_sym are diagonal in the DST-x (x) DST-y
// basis of the fully modal path: K -> lambda_q + lambda_j, M_sym -> m_qj = (2 + (1 + cx)(1 + cy)) / 6,
// c = cos(mode pi h).  E is not (D maps sines to cosines), so the shifted systems of Step 2,
//   (s_p M + K) W_p = M H_p  (s_p = d_p / tau^a; P1 FEM form of (s_p + A) W = H, A = M^{-1} K),
// are solved by the preconditioned fixed-point iteration
//   W <- P^{-1} (M H - s_p E W),   P = s_p M_sym + K  (diagonal in the modes),
// with E applied in physical space (DST-y, DST-x, the 4-point mixed stencil, DST-x, DST-y).  Its
// contraction is |s_p| |E| / |P| <= 1/2 (|E| <= 1/6, m_qj >= 1/3), far smaller whenever K dominates.
// In the h^2-scaled quantities of the modal path (sig_p = h^2 s_p, sig_q + mu_j = h^2 (lambda_q +
// lambda_j)) the iteration is W <- (b - sig_p E W) / (sig_p m_qj + sig_q + mu_j), b = m_qj H + E H.
// A v (the Table-1 corrections) is M^{-1} K v: y <- (K' v - E y) / m_qj (K' = (sig_q + mu_j) / h^2).
#pragma once
#include "fft.cuh"

namespace pint {

struct Fem2dArgs {
  double2* b;               // right-hand side of the fixed point (written by the init modes)
  const double2* H;         // input (modal tile layout [q][jb][levels][WB])
  const double2* EH;        // E H (init) or E X (step)
  double2* X;               // iterate (modal tile layout)
  const double2* sig_p;     // [levels] h^2 d_p / tau^a (S-pass: level index = frequency p); AV: unused
  const double* sig_q;      // [Qb] h^2 lambda_q
  const double* mu;         // [L] h^2 lambda_j
  const double* cx;         // [Qb] cos(q pi h)
  const double* cy;         // [L] cos(j pi h)
  long levels, total;       // levels per tile, total = Qb * NB * levels * WB
  int L, NB, WB, av;        // av: A v mode (shift-free mass solve)
  double kscale;            // 1 / h^2 (A v mode)
  unsigned long long* upd;  // [2]: max |X_new - X| (step), max |X| (init)
};

__device__ __forceinline__ void fem2d_decode(const Fem2dArgs& a, long e, long& q, int& j, long& n) {
  const int w = (int)(e % a.WB);
  long r = e / a.WB;
  n = r % a.levels;
  r /= a.levels;
  const int jb = (int)(r % a.NB);
  q = r / a.NB;
  j = jb * a.WB + w;
}

// init: b and the first iterate X = P^{-1} b (mode 0: b = m H + E H; AV: b = K' v, P = m)
// step: X <- P^{-1} (b - s E X), max |dX| -> upd[0]
template <bool INIT>
__global__ void fem2d_kernel(const Fem2dArgs a) {
  double dm = 0.0;
  bool nonfinite = false;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < a.total; e += (long)gridDim.x * blockDim.x) {
    long q, n;
    int j;
    fem2d_decode(a, e, q, j, n);
    PINT_ASSERT(n < a.levels && j < a.NB * a.WB);
    if (j >= a.L) continue;                               // pad modes stay zero
    const double cq = __ldg(&a.cx[q]), cj = __ldg(&a.cy[j]);
    const double m = (2.0 + (1.0 + cq) * (1.0 + cj)) / 6.0;
    const double kk = __ldg(&a.sig_q[q]) + __ldg(&a.mu[j]);
    double2 s = make_double2(1.0, 0.0), P;
    if (a.av) {
      P = make_double2(m, 0.0);
    } else {
      s = __ldg(&a.sig_p[n]);
      P = make_double2(fma(s.x, m, kk), s.y * m);
    }
    const double ip = 1.0 / cabs2(P);
    const double2 Pi = make_double2(P.x * ip, -P.y * ip);  // 1 / P
    if constexpr (INIT) {
      const double2 h = a.H[e];
      const double2 bb = a.av ? cscale(h, kk * a.kscale) : cadd(cscale(h, m), a.EH[e]);
      a.b[e] = bb;
      const double2 x = cmul(bb, Pi);
      a.X[e] = x;
      const double ax = cabs2(x);
      if (!(ax <= 1.7976931348623157e308)) nonfinite = true;
      dm = fmax(dm, ax);
    } else {
      const double2 x = cmul(csub(a.b[e], cmul(s, a.EH[e])), Pi);
      const double d = cabs2(csub(x, a.X[e]));
      if (!(d <= 1.7976931348623157e308)) nonfinite = true;
      dm = fmax(dm, d);
      a.X[e] = x;
    }
  }
  double r = sqrt(dm);
  if (nonfinite) r = __longlong_as_double(0x7ff0000000000000LL);
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&a.upd[INIT ? 1 : 0], (unsigned long long)__double_as_longlong(r));
}

#ifdef PINT_DEFINE_PLAIN_KERNELS
// Z = (1/24) Dx Dy Y in physical space, tile layout [x][yb][levels][WB] (zero Dirichlet padding):
// Z(x, y) = (Y(x+1, y+1) - Y(x+1, y-1) - Y(x-1, y+1) + Y(x-1, y-1)) / 24
__global__ void fem2d_mixed_kernel(const double2* Y, double2* Z, long levels, int mx, int my, int NB, int WB, long total) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int w = (int)(e % WB);
    long r = e / WB;
    const long n = r % levels;
    r /= levels;
    const int yb = (int)(r % NB);
    const int x = (int)(r / NB);
    const int y = yb * WB + w;
    double2 z = make_double2(0.0, 0.0);
    if (y < my) {
      auto at = [&](int xx, int yy) -> double2 {
        if (xx < 0 || xx >= mx || yy < 0 || yy >= my) return make_double2(0.0, 0.0);
        return Y[(((long)xx * NB + yy / WB) * levels + n) * WB + yy % WB];
      };
      const double2 s = csub(cadd(at(x + 1, y + 1), at(x - 1, y - 1)), cadd(at(x + 1, y - 1), at(x - 1, y + 1)));
      z = cscale(s, 1.0 / 24.0);
    }
    Z[e] = z;
  }
}
#else
__global__ void fem2d_mixed_kernel(const double2* Y, double2* Z, long levels, int mx, int my, int NB, int WB, long total);
#endif

}  // namespace pint
