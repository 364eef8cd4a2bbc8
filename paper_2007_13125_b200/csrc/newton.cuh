// newton.cuh — the semilinear extension (Algorithm 3): Newton's method whose
// linearised problems are solved by the WR iteration of the streaming path.  1D operator only:
// the Newton coefficient g'(Ubar(x)) varies in x, so the DST no longer diagonalises the operator
// and the line solves become general (non-Toeplitz) tridiagonal systems.
//
//   outer l:  c = g'(Ubar_{l-1}),  Ubar = (1/N) sum_n U_{l-1}^n
//             R^n = fbar_n - dbar^a U^n - A U^n - g(U^n)                   (eqn:BDF-CQ-m-r-N rhs)
//             inner WR: (dbar^a + A + diag(c)) W = R, W^{<=0} = 0, kappa-wrap
//             U_l = U_{l-1} + W
// Allen-Cahn: g(u) = (u^3 - u)/eps^2 (Example 4).
#pragma once
#include "spass.cuh"

namespace pint {

struct NewtonArgs {
  const double2* U;      // U_{l-1}, physical [N][L] (1D)
  double2* R;            // residual, tile layout [yb][N][WB]
  double2* c;            // [L] h^2 g'(Ubar)  (line-solve diagonal shift)
  const double2* src;    // [S][Lpad] separable sources (0 = v, 1 = A v, 2.. = g_r)
  const double* coef;    // [S][N]   F_static_n = sum_s coef[s][n] src_s  (= fbar_n + tau^-a psum_n v)
  const double* wt;      // [N]      tau^-a omega_j (heat: zero for j > k)
  const double* anl;     // [N]      a_n of Table 1 (the -a_n g(v) part of fbar)
  const double2* fd;     // dense forcing f(t_n) (tile layout) or NULL (pint_set_problem)
  int S, L, Lpad, WB;
  long N;
  double ih2, h2, ieps2;
};

struct VcArgs {
  const double2* in;      // H, tile layout [yb][N][WB]
  double2* out;           // W
  double2* piv;           // [N][L] scratch: 1/m_i
  const double2* sig_p;   // [N] h^2 d_p / tau^a
  const double2* c;       // [L]
  long N;
  int L, Lpad, WB;
};

struct ResidArgs {
  const double2* U;          // [q][yb][N][WB]
  const double2* src;        // [S][Qb * NB][WB]; source 0 is v
  const double* coef;        // [S][N]
  const double* wk;          // [k+1] (kappa/tau) omega_j
  const double* sig_q;       // [Qb] h^2 lambda_q
  unsigned long long* out;   // [2]
  long N, NB, Qb;
  int WB, L, S, k;
  double ikappa, ih2;
  const double* mu;          // modal plans (U in (q, j) modes): A_y = mu_j / h^2 instead of the stencil
  const double2* tconv;      // CQ: the time term tau^-a sum_{j<=n} omega_j U^{n-j}, precomputed (same layout)
};

#ifdef PINT_DEFINE_NEWTON_KERNELS

__device__ __forceinline__ double2 nl_g(double2 u, double ieps2) {        // (u^3 - u) / eps^2
  const double2 u3 = cmul(cmul(u, u), u);
  return cscale(csub(u3, u), ieps2);
}

// c[y] = h^2 g'(Ubar[y]) = h^2 (3 Ubar^2 - 1) / eps^2
__global__ void nl_coeff_kernel(const NewtonArgs a) {
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < a.L; y += gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (long n = 0; n < a.N; ++n) s = cadd(s, a.U[n * a.L + y]);
    const double2 ub = cscale(s, 1.0 / (double)a.N);
    const double2 d = cscale(make_double2(3.0 * (ub.x * ub.x - ub.y * ub.y) - 1.0, 6.0 * ub.x * ub.y), a.ieps2);
    a.c[y] = cscale(d, a.h2);
  }
}

// R^n = F_static_n - sum_{j=0}^{n-1} tau^-a omega_j U^{n-j} - A U^n - g(U^n) - a_n g(v)
// (the v-terms of fbar and dbar^a cancel against the psum_n v part of F_static)
__global__ void nl_residual_kernel(const NewtonArgs a) {
  const long total = a.N * a.L;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long n = e / a.L;                 // 0-based level (level n+1)
    const int y = (int)(e % a.L);
    double2 r = make_double2(0.0, 0.0);
    for (int s = 0; s < a.S; ++s) r = cfmar(a.src[(long)s * a.Lpad + y], a.coef[(long)s * a.N + n], r);
    for (long j = 0; j <= n; ++j) {
      const double w = a.wt[j];
      if (w != 0.0) r = cfmar(a.U[(n - j) * a.L + y], -w, r);
    }
    const double2 u = a.U[n * a.L + y];
    const double2 ul = y > 0 ? a.U[n * a.L + y - 1] : make_double2(0.0, 0.0);
    const double2 ur = y < a.L - 1 ? a.U[n * a.L + y + 1] : make_double2(0.0, 0.0);
    const double2 Au = cscale(csub(cscale(u, 2.0), cadd(ul, ur)), a.ih2);
    r = csub(r, Au);
    r = csub(r, nl_g(u, a.ieps2));
    if (a.anl[n] != 0.0) r = cfmar(nl_g(a.src[y], a.ieps2), -a.anl[n], r);   // source 0 is v
    if (a.fd) r = cadd(r, a.fd[((long)(y / a.WB) * a.N + n) * a.WB + y % a.WB]);
    a.R[((long)(y / a.WB) * a.N + n) * a.WB + y % a.WB] = r;
  }
}


// Shifted solves with a varying diagonal, one thread per line p (1D): T x = d,
// T = tridiag(-1, 2 + s_i, -1), s_i = h^2 (d_p / tau^a) + c_i.  Shift-accurate pivots
// (SURVEY §8(c) E-6): m_i = 1 + e_i, e_0 = 1 + s_0, e_i = s_i + e_{i-1}/(1 + e_{i-1}) — the 2 of the
// diagonal never meets the small shift.  Thomas: y_i = (d_i + y_{i-1})/m_i, x_i = y_i + x_{i+1}/m_i.
__global__ void spass_vc_kernel(const VcArgs a) {
  const long p = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (p >= a.N) return;
  const double2 sp = a.sig_p[p];
  double2* piv = a.piv + p * a.L;
  auto idx = [&](int y) { return ((long)(y / a.WB) * a.N + p) * a.WB + y % a.WB; };
  double2 e = make_double2(0.0, 0.0), yv = make_double2(0.0, 0.0);
  for (int i = 0; i < a.L; ++i) {
    const double2 s = cadd(sp, a.c[i]);
    e = (i == 0) ? make_double2(1.0 + s.x, s.y) : cadd(s, cdiv(e, make_double2(1.0 + e.x, e.y)));
    const double2 rm = cdiv(make_double2(1.0, 0.0), make_double2(1.0 + e.x, e.y));
    piv[i] = rm;
    yv = cmul(cadd(a.in[idx(i)], yv), rm);
    a.out[idx(i)] = yv;
  }
  double2 x = make_double2(0.0, 0.0);
  for (int i = a.L - 1; i >= 0; --i) {
    x = cadd(a.out[idx(i)], cmul(x, piv[i]));
    a.out[idx(i)] = x;
  }
  for (int y = a.L; y < a.Lpad; ++y) a.out[idx(y)] = make_double2(0.0, 0.0);
}

// U[n][y] += W (tile layout); max |W| -> upd (ordered bits)
__global__ void nl_update_kernel(double2* U, const double2* W, long N, int L, int WB, unsigned long long* upd) {
  double m = 0.0;
  const long total = N * L;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long n = e / L;
    const int y = (int)(e % L);
    const double2 w = W[((long)(y / WB) * N + n) * WB + y % WB];
    U[e] = cadd(U[e], w);
    m = fmax(m, sqrt(cabs2(w)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(upd, (unsigned long long)__double_as_longlong(m));
}

// max |A - B| over count elements -> upd (inner WR monitor on the full space-time array)
__global__ void nl_diffmax_kernel(const double2* A, const double2* B, long count, unsigned long long* upd) {
  double m = 0.0;
  bool nonfinite = false;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count; e += (long)gridDim.x * blockDim.x) {
    const double d = sqrt(cabs2(csub(A[e], B[e])));
    if (!(d <= 1.7976931348623157e308)) nonfinite = true;
    m = fmax(m, d);
  }
  if (nonfinite) m = __longlong_as_double(0x7ff0000000000000LL);   // fmax drops NaN: report +inf
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(upd, (unsigned long long)__double_as_longlong(m));
}

// max |Im a| over count elements -> upd (PINT_FLAG_REAL_DATA input check)
__global__ void imag_max_kernel(const double2* A, long count, unsigned long long* upd) {
  double m = 0.0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count; e += (long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[e].y));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(upd, (unsigned long long)__double_as_longlong(m));
}

// Streaming modal path (PINT_FLAG_MODAL with CQ or PINT_FLAG_STREAM): with the DST applied along
// the line axis too, Step 2 of Algorithm 1/2 is W_{p,q,j} = H_{p,q,j} / (sigma_p + sigma_q + mu_j)
// (h^2-scaled shift + eigenvalues; the shift is never added to a rounded 2: exact in the shift).
// Tile layout [q][jb][N][WB], j = jb WB + w; pad modes j >= L stay zero.  32 B per unknown.
__global__ void modal_div_kernel(const SPassArgs a, const double* mu, long total) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int w = (int)(e % a.WB);
    const long r = e / a.WB;
    const long n = r % a.N, r2 = r / a.N;
    const long jb = r2 % a.NB, q = r2 / a.NB;
    const int j = (int)(jb * a.WB + w);
    double2 x = make_double2(0.0, 0.0);
    if (j < a.L) {
      const double2 sp = __ldg(&a.sig_p[n]);
      x = cdiv(__ldg(&a.in[e]), make_double2(sp.x + __ldg(&a.sig_q[q]) + __ldg(&mu[j]), sp.y));
    }
    a.out[e] = x;
  }
}

// Fixed-point residual of the heat scheme (SURVEY §8(c) "the GPU also self-checks"): for the
// materialised iterate U (tile layout, x in DST modes q, y physical), level n (0-based, = t_{n+1}):
//   r = (1/tau) sum_{j=0}^{min(k,n)} omega_j U^{n-j} + (lambda_q + A_y) U^n - F_static_n
// (the all-at-once form: the history U^{<=0} = v sits in F_static),
// A_y = (2 U_y - U_{y-1} - U_{y+1}) / h^2, lambda_q = sig_q / h^2, F_static_n = sum_s c_s(n) src_s
// (eqn:BDF).  max|r| -> out[0], max|F_static| -> out[1] (ordered bits).

__global__ void resid_kernel(const ResidArgs a, long total) {
  double rm = 0.0, fm = 0.0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int w = (int)(e % a.WB);
    const long r1 = e / a.WB;
    const long n = r1 % a.N, r2 = r1 / a.N;
    const long yb = r2 % a.NB, q = r2 / a.NB;
    const int y = (int)(yb * a.WB + w);
    if (y >= a.L) continue;
    auto at = [&](long nn, int yy) -> double2 {       // U^{nn} at row yy (zero outside the line)
      if (yy < 0 || yy >= a.L) return make_double2(0.0, 0.0);
      const long ti = q * a.NB + yy / a.WB;
      if (nn < 0) return a.src[ti * a.WB + yy % a.WB];  // history U^{<=0} = v
      return a.U[(ti * a.N + nn) * a.WB + yy % a.WB];
    };
    const double2 u = a.U[e];
    double2 r = a.mu ? cscale(u, a.mu[y] * a.ih2)
                     : cscale(csub(cscale(u, 2.0), cadd(at(n, y - 1), at(n, y + 1))), a.ih2);
    r = cfmar(u, a.sig_q[q] * a.ih2, r);
    // levels >= 1 only: the history U^{<=0} = v is part of F_static (tau^-a sum_{j<n} omega_j v)
    if (a.tconv) r = cadd(r, a.tconv[e]);
    else
      for (int j = 0; j <= a.k && j <= n; ++j) r = cfmar(at(n - j, y), a.wk[j] * a.ikappa, r);
    double2 F = make_double2(0.0, 0.0);
    const long ti = q * a.NB + yb;
    for (int s = 0; s < a.S; ++s) F = cfmar(a.src[((long)s * a.Qb * a.NB + ti) * a.WB + w], a.coef[(long)s * a.N + n], F);
    r = csub(r, F);
    rm = fmax(rm, sqrt(cabs2(r)));
    fm = fmax(fm, sqrt(cabs2(F)));
  }
  for (int o = 16; o > 0; o >>= 1) {
    rm = fmax(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    fm = fmax(fm, __shfl_xor_sync(0xffffffffu, fm, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&a.out[0], (unsigned long long)__double_as_longlong(rm));
    atomicMax(&a.out[1], (unsigned long long)__double_as_longlong(fm));
  }
}

// CQ history term of the residual, one CTA per tile (all N levels of WB columns in shared memory):
// T[n][c] = sum_{j=0}^{n} w_j U[n-j][c], w_j = tau^-a omega_j (eqn:CQ-1, in the
// all-at-once form whose v-history sits in F_static).  O(N) per element: a self-check, not a pass.
__global__ void resid_cq_time_kernel(const double2* U, double2* T, const double* w, long N, long ntiles) {
  extern __shared__ double2 tile[];
  const int WB = (int)(TILE / N);   // tile = all N levels of WB columns (fft.cuh layout)
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long base = t * (long)TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) tile[e] = U[base + e];
    __syncthreads();
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const int n = e / WB, c = e % WB;
      double2 s = make_double2(0.0, 0.0);
      for (int j = 0; j <= n; ++j) s = cfmar(tile[(n - j) * WB + c], __ldg(&w[j]), s);
      T[base + e] = s;
    }
    __syncthreads();
  }
}

// out[j] = in[j] mu[j] s: an operator diagonal in the DST modes applied to a modal vector
// (P1-FEM: A v = M^{-1} K v with mu_j = h^2 K_j / M_j, s = 1/h^2)
__global__ void mode_scale_kernel(double2* out, const double2* in, const double* mu, double s, int L) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < L; j += gridDim.x * blockDim.x)
    out[j] = cscale(in[j], mu[j] * s);
}

#endif  // PINT_DEFINE_NEWTON_KERNELS

}  // namespace pint
