// One-bounce fused solve (chains "R" and "T"): one (query, triangle) pair per thread, FP64.
//   coefficient phase  : explicit coefficient formulas of Eq. 6 (a), Eq. 12 (b, R) / Eq. 9 (b, T)
//   elimination phase  : Bezout matrix Eq. 24 hiding v; R: Laplace expansion of the 3x3 polynomial
//                        matrix; T: det at 13 Chebyshev nodes + exact interpolation to
//                        the monomial coefficients of r(v) (same explicit r(v), fewer FLOPs)
//   univariate roots   : derivative recursion on [0,1], Newton-safeguarded bisection
//   path phase         : back-substitution a(u)|v, <=3 Newton steps on (a,b),
//                        Eq. 3 validation, sides, flags, analytic ray-differential contribution.
#pragma once
#include "common.cuh"
#include "poly_dev.cuh"

namespace spoly {

// monomial -> degree-9 Bernstein basis on [0,1]: b_k = sum_{i<=k} C(k,i)/C(9,i) c_i
static __constant__ double c_bern9[10][10] = {
    {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.1111111111111111, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.2222222222222222, 0.027777777777777776, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.3333333333333333, 0.08333333333333333, 0.011904761904761904, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.4444444444444444, 0.16666666666666666, 0.047619047619047616, 0.007936507936507936, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.5555555555555556, 0.2777777777777778, 0.11904761904761904, 0.03968253968253968, 0.007936507936507936, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.6666666666666666, 0.4166666666666667, 0.23809523809523808, 0.11904761904761904, 0.047619047619047616, 0.011904761904761904, 0.0, 0.0, 0.0},
    {1.0, 0.7777777777777778, 0.5833333333333334, 0.4166666666666667, 0.2777777777777778, 0.16666666666666666, 0.08333333333333333, 0.027777777777777776, 0.0, 0.0},
    {1.0, 0.8888888888888888, 0.7777777777777778, 0.6666666666666666, 0.5555555555555556, 0.4444444444444444, 0.3333333333333333, 0.2222222222222222, 0.1111111111111111, 0.0},
    {1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0}};

constexpr int kMaxSolPerPair = 8;

// monomial -> degree-12 Bernstein basis on [0,1]
static __constant__ double c_bern12[13][13] = {
    {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.08333333333333333, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.16666666666666666, 0.015151515151515152, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.25, 0.045454545454545456, 0.004545454545454545, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.3333333333333333, 0.09090909090909091, 0.01818181818181818, 0.00202020202020202, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.4166666666666667, 0.15151515151515152, 0.045454545454545456, 0.010101010101010102, 0.0012626262626262627, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.5, 0.22727272727272727, 0.09090909090909091, 0.030303030303030304, 0.007575757575757576, 0.0010822510822510823, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.5833333333333334, 0.3181818181818182, 0.1590909090909091, 0.0707070707070707, 0.026515151515151516, 0.007575757575757576, 0.0012626262626262627, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.6666666666666666, 0.42424242424242425, 0.2545454545454545, 0.1414141414141414, 0.0707070707070707, 0.030303030303030304, 0.010101010101010102, 0.00202020202020202, 0.0, 0.0, 0.0, 0.0},
    {1.0, 0.75, 0.5454545454545454, 0.38181818181818183, 0.2545454545454545, 0.1590909090909091, 0.09090909090909091, 0.045454545454545456, 0.01818181818181818, 0.004545454545454545, 0.0, 0.0, 0.0},
    {1.0, 0.8333333333333334, 0.6818181818181818, 0.5454545454545454, 0.42424242424242425, 0.3181818181818182, 0.22727272727272727, 0.15151515151515152, 0.09090909090909091, 0.045454545454545456, 0.015151515151515152, 0.0, 0.0},
    {1.0, 0.9166666666666666, 0.8333333333333334, 0.75, 0.6666666666666666, 0.5833333333333334, 0.5, 0.4166666666666667, 0.3333333333333333, 0.25, 0.16666666666666666, 0.08333333333333333, 0.0},
    {1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0}};

// Bernstein exclusion (exact, no effect on the root set): the degree-D Bernstein coefficients b of r on
// [0,1] bound r there (convex hull property), and the k-th derivative of r has the Bernstein coefficients
// D!/(D-k)! * (k-th forward differences of b).  When the k-th differences all have one strict sign,
// r^(k) has no root in [0,1]; the derivative recursion can then start at level k-1 with
// no critical points, because every higher level only serves to locate the roots of r^(k).
// Returns the smallest such k (0: r itself has no root in [0,1]; N: none found).  N = D + 1.
template <int N>
__device__ __forceinline__ int bernstein_root_free_level(const double* r) {
  double b[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i <= k; ++i) acc = fma(N == 10 ? c_bern9[k][i] : c_bern12[k][i], r[i], acc);
    b[k] = acc;
  }
  // strict signs from the high words (integer min/max on the ALU pipe instead of FP64 compares): hi > 0 is
  // a positive value, hi in (INT_MIN, 0) a negative one; +-0 and denormals below 2^-1022 read as "no strict
  // sign" (conservative: a later level or the full recursion).  Non-finite r never takes a shortcut.
  int fin = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) fin = max(fin, __double2hiint(r[i]) & 0x7fffffff);
  int level = N;
  if (fin >= 0x7ff00000) return level;
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
    int mn = __double2hiint(b[0]), mx = mn;
#pragma unroll
    for (int i = 1; i < N - k; ++i) {
      const int h = __double2hiint(b[i]);
      mn = min(mn, h);
      mx = max(mx, h);
    }
    const bool pos = mn > 0x000fffff, neg = mx < 0 && mn > (int)0x800fffff;
    if ((pos || neg) && level == N) level = k;
#pragma unroll
    for (int i = 0; i < N - 1 - k; ++i) b[i] = b[i + 1] - b[i];
  }
  return level;
}

// T: r(v) = Res_u(a, b) up to a constant, by pseudo-division of b by a (a's u^2 coefficient a_2 is a
// constant because a has total degree 2).  Exact identity with the Bezout determinant of Eq. 24:
// det R(v) = +-lc_u(b)^(n - deg_u a) Res_u(a, b); the lc_u(b) roots it drops never carry a common root
// of (a, b), so the admissible chains are the same (reading R5).
__device__ __forceinline__ void resultant_T(const double* A /*3x3*/, const double* B /*7x7*/, int da, int db,
                                            double* r /*13*/) {
#pragma unroll
  for (int t = 0; t < 13; ++t) r[t] = 0.0;
  double a0[3] = {A[0], A[1], A[2]}, a1[2] = {A[3], A[4]};
  const double a2 = A[6];
  if (db == 0) {  // b u-free: its roots in v, then u from a
#pragma unroll
    for (int t = 0; t < 7; ++t) r[t] = B[t];
    return;
  }
  if (da == 0) {  // a u-free: det = +-a0^n b_n^n -> roots of a0 (b_n roots never admissible)
#pragma unroll
    for (int t = 0; t < 3; ++t) r[t] = a0[t];
    return;
  }
  double c[7][7];
#pragma unroll
  for (int j = 0; j < 7; ++j)
#pragma unroll
    for (int t = 0; t < 7; ++t) c[j][t] = (j + t <= 6) ? B[j * 7 + t] : 0.0;
  if (da == 1) {
    // Res(a, b) = sum_j b_j (-a0)^j a1^(db-j), Horner in (-a0) with running powers of a1
    double t_[13], p[13];  // accumulated polynomial, a1 power
#pragma unroll
    for (int t = 0; t < 13; ++t) t_[t] = p[t] = 0.0;
    p[0] = 1.0;
#pragma unroll
    for (int j = 6; j >= 0; --j) {
      if (j > db) continue;
      if (j == db) {
#pragma unroll
        for (int t = 0; t < 7; ++t) t_[t] = c[j][t];
      } else {
        // p <- p * a1
        double np[13];
#pragma unroll
        for (int t = 0; t < 13; ++t) np[t] = 0.0;
#pragma unroll
        for (int t = 0; t < 12; ++t) {
          np[t] = fma(p[t], a1[0], np[t]);
          np[t + 1] = fma(p[t], a1[1], np[t + 1]);
        }
        // t <- t * (-a0) + c_j * p
        double nt[13];
#pragma unroll
        for (int t = 0; t < 13; ++t) nt[t] = 0.0;
#pragma unroll
        for (int t = 0; t < 11; ++t)
#pragma unroll
          for (int s = 0; s < 3; ++s) nt[t + s] = fma(-t_[t], a0[s], nt[t + s]);
#pragma unroll
        for (int t = 0; t < 7; ++t)
#pragma unroll
          for (int s = 0; s < 13; ++s)
            if (t + s < 13) nt[t + s] = fma(c[j][t], np[s], nt[t + s]);
#pragma unroll
        for (int t = 0; t < 13; ++t) {
          t_[t] = nt[t];
          p[t] = np[t];
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 13; ++t) r[t] = t_[t];
    return;
  }
  // da == 2: pseudo-remainder of b by a (degree <= 1 in u)
#pragma unroll
  for (int j = 6; j >= 2; --j) {
    if (j > db) continue;
    double lead[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) lead[t] = c[j][t];
#pragma unroll
    for (int i = 0; i < j; ++i)
#pragma unroll
      for (int t = 0; t < 7; ++t) c[i][t] *= a2;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      c[j - 1][t] = fma(-lead[t], a1[0], c[j - 1][t]);
      c[j - 1][t + 1] = fma(-lead[t], a1[1], c[j - 1][t + 1]);
    }
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int s = 0; s < 3; ++s) c[j - 2][t + s] = fma(-lead[t], a0[s], c[j - 2][t + s]);
  }
  // Res(a, rho1 u + rho0) = a2 rho0^2 - a1 rho0 rho1 + a0 rho1^2
  const double* rho0 = c[0];
  const double* rho1 = c[1];
#pragma unroll
  for (int t = 0; t < 7; ++t)
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      r[t + s] = fma(a2 * rho0[t], rho0[s], r[t + s]);
      r[t + s] = fma(a0[0] * rho1[t], rho1[s], r[t + s]);
      if (t + s + 1 < 13) r[t + s + 1] = fma(a0[1] * rho1[t], rho1[s], r[t + s + 1]);
      if (t + s + 2 < 13) r[t + s + 2] = fma(a0[2] * rho1[t], rho1[s], r[t + s + 2]);
      r[t + s] = fma(-a1[0] * rho0[t], rho1[s], r[t + s]);
      if (t + s + 1 < 13) r[t + s + 1] = fma(-a1[1] * rho0[t], rho1[s], r[t + s + 1]);
    }
}

struct PairOut {
  int nsol;
  uint32_t flags;
  double u[kMaxSolPerPair], v[kMaxSolPerPair], contrib[kMaxSolPerPair];
  float resid[kMaxSolPerPair];
  uint32_t slot[kMaxSolPerPair];
};

// ---------------------------------------------------------------- path-space helpers (Eq. 3)
__device__ __forceinline__ double vertex_residual(d3 xp, d3 x, d3 xn, d3 n, double eta_prev, double eta_next) {
  d3 dp = normalize(x - xp), dn = normalize(xn - x), nh = normalize(n);
  d3 h = eta_next * dn - eta_prev * dp;
  return norm(cross(h, nh)) * fast_rcp(fmax(norm(h), 1e-3 * (eta_prev + eta_next)));
}
__device__ __forceinline__ bool side_ok(bool refract, d3 xp, d3 x, d3 xn, d3 n, d3 g) {
  double spn = dot(xp - x, n), snn = dot(xn - x, n), spg = dot(xp - x, g), sng = dot(xn - x, g);
  if (!(spn * spg > 0)) return false;
  if (!refract) return spn * snn > 0 && spg * sng > 0;
  return spn * snn < 0 && spg * sng < 0;
}

// Analytic ray differential of the light-side trace: J = |d(x0-plane position)/d(omega)|
// for a point light at L = x_2 emitting along omega towards x_1; one reflection/refraction with the
// interpolated normal's derivative; planar triangle transfer.
__device__ double jacobian_k1(bool refract, d3 x0, d3 L, d3 x1, d3 e1, d3 e2, d3 m1, d3 m2, d3 n, double eta_in,
                              double eta_out) {
  d3 w = x1 - L;
  const double lam = norm(w);
  w = fast_rcp(lam) * w;
  d3 g = cross(e1, e2);
  const double nn = norm(n);
  const double inn = fast_rcp(nn);
  const d3 nh = inn * n;
  d3 dref = x0 - x1;
  const double lam0 = norm(dref);
  dref = fast_rcp(lam0) * dref;
  // orthonormal frame perpendicular to w (same construction as any: J is frame-invariant)
  d3 ax = fabs(w.x) < 0.6 ? mk3(1, 0, 0) : (fabs(w.y) < 0.6 ? mk3(0, 1, 0) : mk3(0, 0, 1));
  d3 b1 = normalize(cross(w, ax));
  d3 b2 = cross(w, b1);
  const double e11 = dot(e1, e1), e12 = dot(e1, e2), e22 = dot(e2, e2);
  const double igdet = fast_rcp(e11 * e22 - e12 * e12);
  const double iwg = fast_rcp(dot(w, g));
  const double mu = dot(w, nh);
  const double ep = eta_in / eta_out;
  const double kk = 1.0 - ep * ep * (1.0 - mu * mu);
  const double sk = refract ? sqrt(fmax(kk, 0.0)) : 0.0;
  const double isk = refract ? fast_rcp(sk) : 0.0;
  d3 dP[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    d3 b = c == 0 ? b1 : b2;
    d3 dy = lam * (b - (dot(b, g) * iwg) * w);  // hit point moves in the triangle plane
    double r1 = dot(e1, dy), r2 = dot(e2, dy);
    double du = (e22 * r1 - e12 * r2) * igdet, dv = (e11 * r2 - e12 * r1) * igdet;
    d3 dn = du * m1 + dv * m2;
    d3 dnh = inn * (dn - dot(nh, dn) * nh);
    double dmu = dot(b, nh) + dot(w, dnh);
    d3 dt;
    if (!refract) {
      dt = b - 2.0 * (dmu * nh + mu * dnh);
    } else {
      double sg = mu > 0 ? 1.0 : -1.0;
      dt = ep * (b - dmu * nh - mu * dnh) + sg * ((ep * ep * mu * dmu * isk) * nh + sk * dnh);
    }
    dP[c] = dy + lam0 * dt;
  }
  return fabs(dot(dref, cross(dP[0], dP[1])));
}

// ---------------------------------------------------------------- coefficient phase
// a = ((x1 - x0) x (x2 - x0)) . n  (Eq. 6, Eq. 21/22 first line), x1 = p0 + u e1 + v e2, n = n0 + u m1 + v m2
__device__ __forceinline__ void build_a(d3 q, d3 w, d3 e1, d3 e2, d3 n0, d3 m1, d3 m2, double* A /*3x3*/) {
  d3 A0 = cross(q, w), A1 = cross(e1, w), A2 = cross(e2, w);
  A[0 * 3 + 0] = dot(A0, n0);
  A[1 * 3 + 0] = dot(A0, m1) + dot(A1, n0);
  A[0 * 3 + 1] = dot(A0, m2) + dot(A2, n0);
  A[2 * 3 + 0] = dot(A1, m1);
  A[1 * 3 + 1] = dot(A1, m2) + dot(A2, m1);
  A[0 * 3 + 2] = dot(A2, m2);
  A[1 * 3 + 2] = A[2 * 3 + 1] = A[2 * 3 + 2] = 0.0;
}

// R: b = (d0.n)(d1.t) + (d0.t)(d1.n), t = n x e1 (Eq. 12 / Eq. 21), d1 = w - d0:
//    b = f (w.t) + g (w.n) - 2 f g with f = d0.n (deg 2), g = d0.t (deg 2, linear in u since e1.t = 0)
__device__ __forceinline__ void build_b_R(d3 q, d3 w, d3 e1, d3 e2, d3 n0, d3 m1, d3 m2, double* B /*5x5*/) {
  double f[9], g[9], wn[9], wt[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) f[i] = g[i] = wn[i] = wt[i] = 0.0;
  f[0] = dot(q, n0);
  f[3] = dot(q, m1) + dot(e1, n0);
  f[1] = dot(q, m2) + dot(e2, n0);
  f[6] = dot(e1, m1);
  f[4] = dot(e1, m2) + dot(e2, m1);
  f[2] = dot(e2, m2);
  d3 T0 = cross(n0, e1), T1 = cross(m1, e1), T2 = cross(m2, e1);
  g[0] = dot(q, T0);
  g[3] = dot(q, T1);                  // + e1.T0 = 0
  g[1] = dot(q, T2) + dot(e2, T0);
  g[4] = dot(e2, T1);                 // + e1.T2 = 0 ; u^2 coefficient e1.T1 = 0
  g[2] = dot(e2, T2);
  wn[0] = dot(w, n0);
  wn[3] = dot(w, m1);
  wn[1] = dot(w, m2);
  wt[0] = dot(w, T0);
  wt[3] = dot(w, T1);
  wt[1] = dot(w, T2);
#pragma unroll
  for (int i = 0; i < 25; ++i) B[i] = 0.0;
  bmul_acc<2, 1, 3, 3, 5>(f, wt, 1.0, B);
  bmul_acc<2, 1, 3, 3, 5>(g, wn, 1.0, B);
  bmul_acc<2, 2, 3, 3, 5>(f, g, -2.0, B);
  B[4 * 5 + 0] = 0.0;  // structural: deg_u b = 3
}

// T: b = eta0^2 d1^2 P^2 - eta1^2 d0^2 Q^2, P = (d0 x n).l, Q = (d1 x n).l = W - P (Eq. 9 / Eq. 22)
__device__ __forceinline__ void build_b_T(d3 q, d3 w, d3 e1, d3 e2, d3 n0, d3 m1, d3 m2, d3 l, double eta0,
                                          double eta1, double* B /*7x7*/) {
  d3 c0 = cross(n0, l), c1 = cross(m1, l), c2 = cross(m2, l);  // (a x n).l = a . (n x l)
  double P[9], Q[9], D0[9], D1[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) P[i] = Q[i] = D0[i] = D1[i] = 0.0;
  P[0] = dot(q, c0);
  P[3] = dot(q, c1) + dot(e1, c0);
  P[1] = dot(q, c2) + dot(e2, c0);
  P[6] = dot(e1, c1);
  P[4] = dot(e1, c2) + dot(e2, c1);
  P[2] = dot(e2, c2);
  Q[0] = dot(w, c0) - P[0];
  Q[3] = dot(w, c1) - P[3];
  Q[1] = dot(w, c2) - P[1];
  Q[6] = -P[6];
  Q[4] = -P[4];
  Q[2] = -P[2];
  D0[0] = dot(q, q);
  D0[3] = 2.0 * dot(q, e1);
  D0[1] = 2.0 * dot(q, e2);
  D0[6] = dot(e1, e1);
  D0[4] = 2.0 * dot(e1, e2);
  D0[2] = dot(e2, e2);
  // d1^2 = (w - d0)^2 = w.w - 2 w.d0 + d0^2
  D1[0] = dot(w, w) - 2.0 * dot(w, q) + D0[0];
  D1[3] = -2.0 * dot(w, e1) + D0[3];
  D1[1] = -2.0 * dot(w, e2) + D0[1];
  D1[6] = D0[6];
  D1[4] = D0[4];
  D1[2] = D0[2];
  double P2[25], Q2[25];
#pragma unroll
  for (int i = 0; i < 25; ++i) P2[i] = Q2[i] = 0.0;
  bmul_acc<2, 2, 3, 3, 5>(P, P, 1.0, P2);
  bmul_acc<2, 2, 3, 3, 5>(Q, Q, 1.0, Q2);
#pragma unroll
  for (int i = 0; i < 49; ++i) B[i] = 0.0;
  bmul_acc<2, 4, 3, 5, 7>(D1, P2, eta0 * eta0, B);
  bmul_acc<2, 4, 3, 5, 7>(D0, Q2, -eta1 * eta1, B);
}

// ---------------------------------------------------------------- elimination phase
// Eq. 24 entry (i,j) as a polynomial in v: sum_k a_{i-k} b_{j+1+k} - b_{i-k} a_{j+1+k}
// with slices a_i(v) = A[i][.] (degree DA-i), b_i(v) = B[i][.] (degree DB-i).
template <int DA, int DB, int SA, int SB, int NE>
__device__ __forceinline__ void bezout_entry(const double* A, const double* B, int n, int i, int j, double* E) {
#pragma unroll
  for (int t = 0; t < NE; ++t) E[t] = 0.0;
#pragma unroll
  for (int k = 0; k <= DB; ++k) {
    if (k <= i && k <= n - 1 - j) {
      const int ia = i - k, jb = j + 1 + k;
      // a_{ia} * b_{jb}
#pragma unroll
      for (int s = 0; s <= DA; ++s)
#pragma unroll
        for (int t = 0; t <= DB; ++t) {
          if (s <= DA - ia && t <= DB - jb && ia <= DA && jb <= DB && s + t < NE) {
            E[s + t] = fma(A[ia * SA + s], B[jb * SB + t], E[s + t]);
          }
          if (s <= DA - jb && t <= DB - ia && jb <= DA && ia <= DB && s + t < NE) {
            E[s + t] = fma(-B[ia * SB + t], A[jb * SA + s], E[s + t]);
          }
        }
    }
  }
}

// R: 3x3 Bezout (n <= 3) with entry degrees <= 5-i-j, Laplace expansion along row 0 -> r (<= deg 9)
__device__ __forceinline__ void det_R(const double* A, const double* B, int n, double* r /*10*/) {
#pragma unroll
  for (int t = 0; t < 10; ++t) r[t] = 0.0;
  if (n == 3) {
    double E00[6], E01[5], E02[4], E11[4], E12[3], E22[2];
    bezout_entry<2, 4, 3, 5, 6>(A, B, 3, 0, 0, E00);
    bezout_entry<2, 4, 3, 5, 5>(A, B, 3, 0, 1, E01);
    bezout_entry<2, 4, 3, 5, 4>(A, B, 3, 0, 2, E02);
    bezout_entry<2, 4, 3, 5, 4>(A, B, 3, 1, 1, E11);
    bezout_entry<2, 4, 3, 5, 3>(A, B, 3, 1, 2, E12);
    bezout_entry<2, 4, 3, 5, 2>(A, B, 3, 2, 2, E22);
    // symmetric: E10 = E01, E20 = E02, E21 = E12
    double m0[5] = {0, 0, 0, 0, 0}, m1[6] = {0, 0, 0, 0, 0, 0}, m2[7] = {0, 0, 0, 0, 0, 0, 0};
    pmul_acc<4, 2>(E11, E22, 1.0, m0);   // E11 E22 - E12 E21   (deg 4)
    pmul_acc<3, 3>(E12, E12, -1.0, m0);
    pmul_acc<5, 2>(E01, E22, 1.0, m1);   // E10 E22 - E12 E20   (deg 5)
    pmul_acc<3, 4>(E12, E02, -1.0, m1);
    pmul_acc<5, 3>(E01, E12, 1.0, m2);   // E10 E21 - E11 E20   (deg 6)
    pmul_acc<4, 4>(E11, E02, -1.0, m2);
    pmul_acc<6, 5>(E00, m0, 1.0, r);
    pmul_acc<5, 6>(E01, m1, -1.0, r);
    pmul_acc<4, 7>(E02, m2, 1.0, r);
  } else if (n == 2) {
    double E00[6], E01[5], E11[4];
    bezout_entry<2, 4, 3, 5, 6>(A, B, 2, 0, 0, E00);
    bezout_entry<2, 4, 3, 5, 5>(A, B, 2, 0, 1, E01);
    bezout_entry<2, 4, 3, 5, 4>(A, B, 2, 1, 1, E11);
    pmul_acc<6, 4>(E00, E11, 1.0, r);
    pmul_acc<5, 5>(E01, E01, -1.0, r);
  } else if (n == 1) {
    double E00[6];
    bezout_entry<2, 4, 3, 5, 6>(A, B, 1, 0, 0, E00);
#pragma unroll
    for (int t = 0; t < 6; ++t) r[t] = E00[t];
  }
}

}  // namespace spoly
