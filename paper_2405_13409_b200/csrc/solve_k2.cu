// Two-bounce solve, chains "RR" (Eq. 23), "RT", "TR" and "TT" (Eqs. 13-20; square form at a refracting x_2,
// product form at a reflecting one; Table 3 rows), one
// (query, triangle pair) per thread, FP64, polynomial grids and the Bezout matrix in thread-local memory.
//
//   coefficient phase : rational coordinate mapping u_2 = (u~, v~)/kappa (Eqs. 13-16) of the scaled
//                       direction d~_1 (Eq. 17 reflection; Eqs. 18-20 refraction with the piecewise rational
//                       sqrt surrogate, reading R8), then a = Eq. 6 at x_2 and b = Eq. 12 (RR) / Eq. 9 (TT),
//                       denominators cleared; normalise + numerical u-degree truncation (R6)
//   elimination       : Bezout matrix of Eq. 24 evaluated numerically at v by the Chionh recurrence
//                       B_ij = B_{i-1,j+1} + a_i b_{j+1} - b_i a_{j+1} (exact consequence of Eq. 24)
//   roots             : sign of det R(v_j) at v_j = j/100 by Gaussian elimination with partial pivoting,
//                       10 bisections per sign-changing piece
//   path phase        : u-roots of a(., v*) on [-0.1, 1.1], mapping to u_2, raw admission (theta_admit),
//                       <= 3 Newton steps on the exact shooting residual, final Eq. 3
//                       validation, sides, flags, contribution I / J (J by central differences of the
//                       light-side trace, Richardson), emission.
// This is the correctness-first round-1 kernel; the warp-cooperative version is future work.
#include "kernels.cuh"
#include "poly_dev.cuh"

namespace spoly {

// ------------------------------------------------------------------ dense bivariate polynomials
template <int D>
struct BP {
  static constexpr int S = D + 1;
  double c[S * S];  // c[i*S + j]: coefficient of u^i v^j, only i + j <= deg used
  int deg;
};

template <int D>
__device__ __forceinline__ void bp_zero(BP<D>& p, int deg) {
  p.deg = deg;
  for (int i = 0; i < BP<D>::S * BP<D>::S; ++i) p.c[i] = 0.0;
}
template <int D>
__device__ __forceinline__ void bp_linear(BP<D>& p, double a, double b, double c) {
  bp_zero(p, 1);
  p.c[0] = a;
  p.c[BP<D>::S] = b;
  p.c[1] = c;
}
template <int D>
__device__ __forceinline__ void bp_const(BP<D>& p, double a) {
  bp_zero(p, 0);
  p.c[0] = a;
}
// c += s * a * b
template <int DA, int DB, int DC>
__device__ void bp_mul_acc(const BP<DA>& a, const BP<DB>& b, double s, BP<DC>& c) {
  const int SA = BP<DA>::S, SB = BP<DB>::S, SC = BP<DC>::S;
  if (a.deg + b.deg > c.deg) c.deg = a.deg + b.deg;
  for (int i = 0; i <= a.deg; ++i)
    for (int j = 0; i + j <= a.deg; ++j) {
      const double x = s * a.c[i * SA + j];
      if (x == 0.0) continue;
      for (int k = 0; k <= b.deg; ++k)
        for (int l = 0; k + l <= b.deg; ++l) c.c[(i + k) * SC + (j + l)] = fma(x, b.c[k * SB + l], c.c[(i + k) * SC + (j + l)]);
    }
}
// c += s * a
template <int DA, int DC>
__device__ void bp_add(const BP<DA>& a, double s, BP<DC>& c) {
  const int SA = BP<DA>::S, SC = BP<DC>::S;
  if (a.deg > c.deg) c.deg = a.deg;
  for (int i = 0; i <= a.deg; ++i)
    for (int j = 0; i + j <= a.deg; ++j) c.c[i * SC + j] = fma(s, a.c[i * SA + j], c.c[i * SC + j]);
}
template <int D>
__device__ double bp_eval(const BP<D>& p, double u, double v) {
  const int S = BP<D>::S;
  double acc = 0.0;
  for (int i = p.deg; i >= 0; --i) {
    double s = 0.0;
    for (int j = p.deg - i; j >= 0; --j) s = fma(s, v, p.c[i * S + j]);
    acc = fma(acc, u, s);
  }
  return acc;
}
template <int D>
__device__ void bp_slices(const BP<D>& p, int du, double v, double* out) {  // a_i(v), i = 0..du
  const int S = BP<D>::S;
  for (int i = 0; i <= du; ++i) {
    double s = 0.0;
    if (i <= p.deg)
      for (int j = p.deg - i; j >= 0; --j) s = fma(s, v, p.c[i * S + j]);
    out[i] = s;
  }
}

template <int D>
struct BV {
  BP<D> x, y, z;
};
// vector helpers: BV<DC> r = a . b etc.
template <int DA, int DB, int DC>
__device__ void bv_dot_acc(const BV<DA>& a, const BV<DB>& b, double s, BP<DC>& c) {
  bp_mul_acc(a.x, b.x, s, c);
  bp_mul_acc(a.y, b.y, s, c);
  bp_mul_acc(a.z, b.z, s, c);
}
template <int DA, int DC>
__device__ void bv_dotc_acc(const BV<DA>& a, d3 b, double s, BP<DC>& c) {
  bp_add(a.x, s * b.x, c);
  bp_add(a.y, s * b.y, c);
  bp_add(a.z, s * b.z, c);
}
// (a x b) for polynomial a and constant b
template <int DA, int DC>
__device__ void bv_cross_c(const BV<DA>& a, d3 b, BV<DC>& r) {
  bp_zero(r.x, a.x.deg);
  bp_zero(r.y, a.x.deg);
  bp_zero(r.z, a.x.deg);
  bp_add(a.y, b.z, r.x); bp_add(a.z, -b.y, r.x);
  bp_add(a.z, b.x, r.y); bp_add(a.x, -b.z, r.y);
  bp_add(a.x, b.y, r.z); bp_add(a.y, -b.x, r.z);
}
// r = a x b, both polynomial
template <int DA, int DB, int DC>
__device__ void bv_cross(const BV<DA>& a, const BV<DB>& b, BV<DC>& r) {
  const int d = a.x.deg + b.x.deg;
  bp_zero(r.x, d);
  bp_zero(r.y, d);
  bp_zero(r.z, d);
  bp_mul_acc(a.y, b.z, 1.0, r.x); bp_mul_acc(a.z, b.y, -1.0, r.x);
  bp_mul_acc(a.z, b.x, 1.0, r.y); bp_mul_acc(a.x, b.z, -1.0, r.y);
  bp_mul_acc(a.x, b.y, 1.0, r.z); bp_mul_acc(a.y, b.x, -1.0, r.z);
}

// ------------------------------------------------------------------ system
// chain X1 X2 with X = R (reflection) / T (refraction): V1T = vertex 1 refracts, V2T = vertex 2 refracts
template <bool V1T, bool V2T>
struct Sys2 {
  static constexpr int DK = V1T ? 7 : 3;  // deg kappa = deg d~_1 (Eq. 17: 3; Eqs. 19-20 cleared: 7)
  static constexpr int DU = DK + 1;       // deg u~, v~
  static constexpr int DA = 2 * DK + 3;   // deg a: 9 (R.), 17 (T.)
  // deg b: product form (d~.N2)(D2.T2)+..: DK+DU+2DU; square form D2^2 P^2: 2DU + 2(DK+DU)
  static constexpr int DB = V2T ? 2 * DU + 2 * (DK + DU) : (DK + DU) + 2 * DU;  // RR 15, RT 22, TR 31, TT 46
  BP<DA> a;
  BP<DB> b;
  BP<DU> U, V;
  BP<DK> K;
  double eta0, eta1, eta2;
  bool relabel;
  uint32_t flags;
  int da, db, n;
};

struct Tri2 {
  d3 p[3], n[3];
  __device__ d3 e1() const { return p[1] - p[0]; }
  __device__ d3 e2() const { return p[2] - p[0]; }
  __device__ d3 g() const { return cross(p[1] - p[0], p[2] - p[0]); }
  __device__ d3 X(double u, double v) const { return p[0] + u * (p[1] - p[0]) + v * (p[2] - p[0]); }
  __device__ d3 N(double u, double v) const { return n[0] + u * (n[1] - n[0]) + v * (n[2] - n[0]); }
  __device__ d3 c() const { return (1.0 / 3.0) * (p[0] + p[1] + p[2]); }
};

// piecewise rational sqrt surrogate (Eq. 20): literal copy of tests/golden/sqrt_table.txt (our fit, R8)
__constant__ double c_sqrt_tab[6][5] = {
    {0, 0.00042432536375417839, 0.00089999999999879705, 154.92902483814683, 5615.7008147954339},
    {0.00042432536375417839, 0.0077313602416299448, 0.013714746392967799, 21.253136166194601, 135.24944765874642},
    {0.0077313602416299448, 0.051793068389647277, 0.04635497395617269, 6.7900571325924943, 14.594946360257405},
    {0.051793068389647277, 0.21636853563098274, 0.10736470812718857, 3.006160575603614, 2.9223382765562778},
    {0.21636853563098274, 0.68268233146982271, 0.20527897991137517, 1.5904325277264706, 0.82650456712266585},
    {0.68268233146982271, 1, 0.30276242425651556, 1.0984677499357838, 0.40129928835931156}};

template <bool V1T, bool V2T>
__device__ bool build_system2(d3 x0, d3 x3, const Tri2& T1, const Tri2& T2in, const SolveParams& prm,
                              Sys2<V1T, V2T>& S) {
  using Sy = Sys2<V1T, V2T>;
  S.flags = 0;
  const bool front0 = dot(x0 - T1.p[0], T1.g()) > 0;
  S.eta0 = front0 ? prm.eta_front : prm.eta_back;
  S.eta1 = V1T ? (front0 ? prm.eta_back : prm.eta_front) : S.eta0;
  const d3 c1 = T1.c();
  const bool c1front = dot(c1 - T2in.p[0], T2in.g()) > 0;
  S.eta2 = V2T ? (c1front ? prm.eta_back : prm.eta_front) : S.eta1;
  // reading R1 at x_2 with x_{k-1} = centroid of T_1
  const d3 nc = T2in.N(1.0 / 3.0, 1.0 / 3.0);
  const d3 lc = cross(x3 - c1, nc);
  const double ln = norm(lc);
  if (!(ln > 1e-12 * norm(x3 - c1) * norm(nc))) S.flags |= SPOLY_FLAG_DEGENERATE;
  S.relabel = false;
  d3 ell = mk3(1, 0, 0);
  if (!V2T) {
    if (ln > 0) {
      const d3 e1 = T2in.e1(), e2 = T2in.e2();
      S.relabel = fabs(dot(e1, lc)) / (norm(e1) * ln) < fabs(dot(e2, lc)) / (norm(e2) * ln);
    }
  } else if (ln > 0) {
    ell = (1.0 / ln) * lc;
  }
  Tri2 T2 = T2in;
  if (S.relabel) {
    T2.p[1] = T2in.p[2]; T2.p[2] = T2in.p[1];
    T2.n[1] = T2in.n[2]; T2.n[2] = T2in.n[1];
  }
  // X1 = p0 + u e1 + v e2, N1 = n0 + u m1 + v m2, D0 = X1 - x0   (Eqs. 1-2)
  const d3 e1 = T1.e1(), e2 = T1.e2(), m1 = T1.n[1] - T1.n[0], m2 = T1.n[2] - T1.n[0];
  BV<1> X1, N1, D0;
  bp_linear(X1.x, T1.p[0].x, e1.x, e2.x); bp_linear(X1.y, T1.p[0].y, e1.y, e2.y); bp_linear(X1.z, T1.p[0].z, e1.z, e2.z);
  bp_linear(N1.x, T1.n[0].x, m1.x, m2.x); bp_linear(N1.y, T1.n[0].y, m1.y, m2.y); bp_linear(N1.z, T1.n[0].z, m1.z, m2.z);
  const d3 q = T1.p[0] - x0;
  bp_linear(D0.x, q.x, e1.x, e2.x); bp_linear(D0.y, q.y, e1.y, e2.y); bp_linear(D0.z, q.z, e1.z, e2.z);
  constexpr int DK = Sy::DK;
  BV<DK> Dt;
  {
    BP<2> dn, nn;
    bp_zero(dn, 2);
    bp_zero(nn, 2);
    bv_dot_acc(D0, N1, 1.0, dn);
    bv_dot_acc(N1, N1, 1.0, nn);
    bp_zero(Dt.x, DK); bp_zero(Dt.y, DK); bp_zero(Dt.z, DK);
    if (!V1T) {
      // Eq. 17: d~ = -2 (d0 . n) n + d0 n^2
      bp_mul_acc(dn, N1.x, -2.0, Dt.x); bp_mul_acc(dn, N1.y, -2.0, Dt.y); bp_mul_acc(dn, N1.z, -2.0, Dt.z);
      bp_mul_acc(nn, D0.x, 1.0, Dt.x); bp_mul_acc(nn, D0.y, 1.0, Dt.y); bp_mul_acc(nn, D0.z, 1.0, Dt.z);
    } else {
      // Eqs. 18-20 with sqrt(beta) ~ sqrt(s) (c0 s + c1 beta) / (s + d1 beta), denominator cleared
      const double ep = S.eta0 / S.eta1;
      double nmax = 0, dmax = 0;
      for (int j = 0; j < 3; ++j) {
        nmax = fmax(nmax, dot(T1.n[j], T1.n[j]));
        dmax = fmax(dmax, dot(T1.p[j] - x0, T1.p[j] - x0));
      }
      const double s = nmax * dmax;
      const d3 ncen = T1.N(1.0 / 3.0, 1.0 / 3.0), dcen = T1.X(1.0 / 3.0, 1.0 / 3.0) - x0;
      const double cnn = dot(ncen, ncen), cdd = dot(dcen, dcen), cdn = dot(dcen, ncen);
      const double cbeta = cnn * cdd - ep * ep * (cnn * cdd - cdn * cdn);
      const double xb = fmin(1.0, fmax(0.0, cbeta / s));
      int piece = 5;
      for (int i = 5; i >= 0; --i)
        if (xb <= c_sqrt_tab[i][1]) piece = i;
      const double sigma = cdn < 0 ? 1.0 : -1.0;
      BP<2> dd;
      bp_zero(dd, 2);
      bv_dot_acc(D0, D0, 1.0, dd);
      BP<4> beta, nd, dn2;
      bp_zero(beta, 4);
      bp_zero(nd, 4);
      bp_zero(dn2, 4);
      bp_mul_acc(nn, dd, 1.0, nd);
      bp_mul_acc(dn, dn, 1.0, dn2);
      bp_add(nd, 1.0 - ep * ep, beta);  // beta = nn dd - ep^2 (nn dd - dn^2)   (Eq. 19)
      bp_add(dn2, ep * ep, beta);
      BP<4> den, sq;
      bp_zero(den, 4);
      bp_zero(sq, 4);
      bp_add(beta, c_sqrt_tab[piece][4], den);
      den.c[0] += s;
      bp_add(beta, c_sqrt_tab[piece][3], sq);
      sq.c[0] += c_sqrt_tab[piece][2] * s;
      // tang = nn D0 - dn N1 (deg 3)
      BV<3> tang;
      bp_zero(tang.x, 3); bp_zero(tang.y, 3); bp_zero(tang.z, 3);
      bp_mul_acc(nn, D0.x, 1.0, tang.x); bp_mul_acc(dn, N1.x, -1.0, tang.x);
      bp_mul_acc(nn, D0.y, 1.0, tang.y); bp_mul_acc(dn, N1.y, -1.0, tang.y);
      bp_mul_acc(nn, D0.z, 1.0, tang.z); bp_mul_acc(dn, N1.z, -1.0, tang.z);
      const double k2 = -sigma * sqrt(s);
      bp_mul_acc(den, tang.x, ep, Dt.x); bp_mul_acc(sq, N1.x, k2, Dt.x);
      bp_mul_acc(den, tang.y, ep, Dt.y); bp_mul_acc(sq, N1.y, k2, Dt.y);
      bp_mul_acc(den, tang.z, ep, Dt.z); bp_mul_acc(sq, N1.z, k2, Dt.z);
    }
  }
  // rational coordinate mapping onto T_2 (Eqs. 13-16)
  const d3 f1 = T2.e1(), f2 = T2.e2(), r0 = T2.n[0], g1 = T2.n[1] - T2.n[0], g2 = T2.n[2] - T2.n[0];
  BV<1> Sv;  // x_1 - p_{2,0}
  const d3 sq0 = T1.p[0] - T2.p[0];
  bp_linear(Sv.x, sq0.x, e1.x, e2.x); bp_linear(Sv.y, sq0.y, e1.y, e2.y); bp_linear(Sv.z, sq0.z, e1.z, e2.z);
  BV<DK> Dxf2;
  bv_cross_c(Dt, f2, Dxf2);
  constexpr int DU = Sy::DU;
  bp_zero(S.U, DU);
  bv_dot_acc(Dxf2, Sv, 1.0, S.U);  // u~ = (d~ x e22) . (x1 - p20)
  bp_zero(S.K, DK);
  bv_dotc_acc(Dxf2, f1, 1.0, S.K);  // kappa = (d~ x e22) . e21
  {
    // v~ = ((x1 - p20) x e21) . d~
    BV<1> Sxf1;
    bv_cross_c(Sv, f1, Sxf1);
    bp_zero(S.V, DU);
    bv_dot_acc(Sxf1, Dt, 1.0, S.V);
  }
  // kappa x_2 and kappa n_2
  BV<DU> X2, N2;
  bp_zero(X2.x, DU); bp_zero(X2.y, DU); bp_zero(X2.z, DU);
  bp_zero(N2.x, DU); bp_zero(N2.y, DU); bp_zero(N2.z, DU);
  bp_add(S.K, T2.p[0].x, X2.x); bp_add(S.U, f1.x, X2.x); bp_add(S.V, f2.x, X2.x);
  bp_add(S.K, T2.p[0].y, X2.y); bp_add(S.U, f1.y, X2.y); bp_add(S.V, f2.y, X2.y);
  bp_add(S.K, T2.p[0].z, X2.z); bp_add(S.U, f1.z, X2.z); bp_add(S.V, f2.z, X2.z);
  bp_add(S.K, r0.x, N2.x); bp_add(S.U, g1.x, N2.x); bp_add(S.V, g2.x, N2.x);
  bp_add(S.K, r0.y, N2.y); bp_add(S.U, g1.y, N2.y); bp_add(S.V, g2.y, N2.y);
  bp_add(S.K, r0.z, N2.z); bp_add(S.U, g1.z, N2.z); bp_add(S.V, g2.z, N2.z);
  // a = ((X2 - K X1) x (x3 - X1)) . N2   (Eq. 6 at x_2, Eq. 23 first line)
  {
    BV<DU> W;  // X2 - K X1 (deg DK + 1)
    bp_zero(W.x, DU); bp_zero(W.y, DU); bp_zero(W.z, DU);
    bp_add(X2.x, 1.0, W.x); bp_mul_acc(S.K, X1.x, -1.0, W.x);
    bp_add(X2.y, 1.0, W.y); bp_mul_acc(S.K, X1.y, -1.0, W.y);
    bp_add(X2.z, 1.0, W.z); bp_mul_acc(S.K, X1.z, -1.0, W.z);
    BV<1> Y;  // x3 - X1
    const d3 y0 = x3 - T1.p[0];
    bp_linear(Y.x, y0.x, -e1.x, -e2.x); bp_linear(Y.y, y0.y, -e1.y, -e2.y); bp_linear(Y.z, y0.z, -e1.z, -e2.z);
    BV<DU + 1> C;
    bv_cross(W, Y, C);
    bp_zero(S.a, Sy::DA);
    bv_dot_acc(C, N2, 1.0, S.a);
  }
  // D2 = K x3 - X2 (kappa d_2)
  BV<DU> D2;
  bp_zero(D2.x, DU); bp_zero(D2.y, DU); bp_zero(D2.z, DU);
  bp_add(S.K, x3.x, D2.x); bp_add(X2.x, -1.0, D2.x);
  bp_add(S.K, x3.y, D2.y); bp_add(X2.y, -1.0, D2.y);
  bp_add(S.K, x3.z, D2.z); bp_add(X2.z, -1.0, D2.z);
  bp_zero(S.b, Sy::DB);
  if (!V2T) {
    // b = (d~.N2)(D2.T2) + (d~.T2)(D2.N2), T2 = N2 x e21   (Eq. 12 with d~_1, Eq. 23)
    BV<DU> Tt;
    bv_cross_c(N2, f1, Tt);
    BP<DK + DU> p1, p3;
    BP<2 * DU> p2, p4;
    bp_zero(p1, DK + DU); bp_zero(p2, 2 * DU); bp_zero(p3, DK + DU); bp_zero(p4, 2 * DU);
    bv_dot_acc(Dt, N2, 1.0, p1);
    bv_dot_acc(D2, Tt, 1.0, p2);
    bv_dot_acc(Dt, Tt, 1.0, p3);
    bv_dot_acc(D2, N2, 1.0, p4);
    bp_mul_acc(p1, p2, 1.0, S.b);
    bp_mul_acc(p3, p4, 1.0, S.b);
  } else {
    // b = eta1^2 D2^2 ((d~ x N2).l)^2 - eta2^2 d~^2 ((D2 x N2).l)^2   (Eq. 9 at x_2)
    BP<DK + DU> P;
    BP<2 * DU> Q;
    {
      BV<DK + DU> C;
      bv_cross(Dt, N2, C);
      bp_zero(P, DK + DU);
      bv_dotc_acc(C, ell, 1.0, P);
    }
    {
      BV<2 * DU> C;
      bv_cross(D2, N2, C);
      bp_zero(Q, 2 * DU);
      bv_dotc_acc(C, ell, 1.0, Q);
    }
    BP<2 * DU> d22;
    bp_zero(d22, 2 * DU);
    bv_dot_acc(D2, D2, 1.0, d22);
    BP<2 * DK> dt2;
    bp_zero(dt2, 2 * DK);
    bv_dot_acc(Dt, Dt, 1.0, dt2);
    {
      BP<2 * (DK + DU)> P2;
      bp_zero(P2, 2 * (DK + DU));
      bp_mul_acc(P, P, 1.0, P2);
      bp_mul_acc(d22, P2, S.eta1 * S.eta1, S.b);
    }
    {
      BP<4 * DU> Q2;
      bp_zero(Q2, 4 * DU);
      bp_mul_acc(Q, Q, 1.0, Q2);
      bp_mul_acc(dt2, Q2, -S.eta2 * S.eta2, S.b);
    }
  }
  // normalise and truncate (R6)
  double ma = 0, mb = 0;
  const int SA = BP<Sy::DA>::S, SB = BP<Sy::DB>::S;
  for (int i = 0; i <= S.a.deg; ++i)
    for (int j = 0; i + j <= S.a.deg; ++j) ma = fmax(ma, fabs(S.a.c[i * SA + j]));
  for (int i = 0; i <= S.b.deg; ++i)
    for (int j = 0; i + j <= S.b.deg; ++j) mb = fmax(mb, fabs(S.b.c[i * SB + j]));
  if (!(ma > 0) || !(mb > 0)) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  const double ia = 1.0 / ma, ib = 1.0 / mb;
  S.da = 0;
  S.db = 0;
  double f = 1.0;
  for (int i = 0; i <= S.a.deg; ++i, f *= 1.1) {
    double m = 0;
    for (int j = 0; i + j <= S.a.deg; ++j) {
      S.a.c[i * SA + j] *= ia;
      m = fmax(m, fabs(S.a.c[i * SA + j]));
    }
    if (m * f > prm.tau_trunc) S.da = i;
  }
  f = 1.0;
  for (int i = 0; i <= S.b.deg; ++i, f *= 1.1) {
    double m = 0;
    for (int j = 0; i + j <= S.b.deg; ++j) {
      S.b.c[i * SB + j] *= ib;
      m = fmax(m, fabs(S.b.c[i * SB + j]));
    }
    if (m * f > prm.tau_trunc) S.db = i;
  }
  for (int i = S.da + 1; i <= S.a.deg; ++i)
    for (int j = 0; i + j <= S.a.deg; ++j) S.a.c[i * SA + j] = 0.0;
  for (int i = S.db + 1; i <= S.b.deg; ++i)
    for (int j = 0; i + j <= S.b.deg; ++j) S.b.c[i * SB + j] = 0.0;
  S.n = max(S.da, S.db);
  if (S.n == 0) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  return true;
}

// det R(v) (Eq. 24) by the Chionh recurrence + Gaussian elimination with partial pivoting (max |.|,
// lowest index on ties); returns the sign and log|det|
template <bool V1T, bool V2T>
__device__ int det_sign_at(const Sys2<V1T, V2T>& S, double v, double* logabs, double* M /* n*n scratch */) {
  constexpr int NS = Sys2<V1T, V2T>::DB + 2;
  double as[NS], bs[NS];
  const int n = S.n;
  bp_slices(S.a, n, v, as);
  bp_slices(S.b, n, v, bs);
  for (int i = S.da + 1; i <= n; ++i) as[i] = 0.0;
  for (int i = S.db + 1; i <= n; ++i) bs[i] = 0.0;
  as[n + 1] = bs[n + 1] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double t = as[i] * bs[j + 1] - bs[i] * as[j + 1];
      if (i > 0 && j + 1 < n) t += M[(i - 1) * n + j + 1];
      M[i * n + j] = t;
    }
  int sign = 1;
  double lg = 0.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = fabs(M[c * n + c]);
    for (int r = c + 1; r < n; ++r)
      if (fabs(M[r * n + c]) > best) {
        best = fabs(M[r * n + c]);
        piv = r;
      }
    if (best == 0.0) {
      *logabs = -INFINITY;
      return 0;
    }
    if (piv != c) {
      sign = -sign;
      for (int l = c; l < n; ++l) {
        const double t = M[c * n + l];
        M[c * n + l] = M[piv * n + l];
        M[piv * n + l] = t;
      }
    }
    const double d = M[c * n + c];
    if (d < 0) sign = -sign;
    lg += log(fabs(d));
    const double inv = 1.0 / d;
    for (int r = c + 1; r < n; ++r) {
      const double fr = M[r * n + c] * inv;
      if (fr != 0.0)
        for (int l = c + 1; l < n; ++l) M[r * n + l] = fma(-fr, M[c * n + l], M[r * n + l]);
    }
  }
  *logabs = lg;
  return sign;
}

// ------------------------------------------------------------------ path space
__device__ __forceinline__ bool refract_dir(d3 d, d3 n, double ei, double eo, d3* out) {
  const double ep = ei / eo;
  double ci = -dot(d, n);
  if (ci < 0) {
    n = -1.0 * n;
    ci = -ci;
  }
  const double k = 1.0 - ep * ep * (1.0 - ci * ci);
  if (k < 0) return false;
  *out = ep * d + (ep * ci - sqrt(k)) * n;
  return true;
}
__device__ __forceinline__ bool scatter_dir(bool refract, d3 d, d3 n, double ei, double eo, d3* out) {
  if (!refract) {
    *out = d - (2.0 * dot(d, n)) * n;
    return true;
  }
  return refract_dir(d, n, ei, eo, out);
}
__device__ __forceinline__ bool plane_hit(d3 o, d3 d, const Tri2& T, double* u, double* v, double* t) {
  const d3 e1 = T.e1(), e2 = T.e2();
  const d3 P = cross(d, e2);
  const double det = dot(e1, P);
  if (det == 0.0) return false;
  const d3 s = o - T.p[0];
  *u = dot(s, P) / det;
  const d3 Q = cross(s, e1);
  *v = dot(d, Q) / det;
  *t = dot(e2, Q) / det;
  return true;
}
__device__ __forceinline__ double resid(d3 xp, d3 x, d3 xn, d3 n, double ep_, double en) {
  const d3 dp = normalize(x - xp), dn = normalize(xn - x), nh = normalize(n);
  const d3 h = en * dn - ep_ * dp;
  return norm(cross(h, nh)) / fmax(norm(h), 1e-3 * (ep_ + en));
}
__device__ __forceinline__ bool sides(bool refract, d3 xp, d3 x, d3 xn, d3 n, d3 g) {
  const double spn = dot(xp - x, n), snn = dot(xn - x, n), spg = dot(xp - x, g), sng = dot(xn - x, g);
  if (!(spn * spg > 0)) return false;
  if (!refract) return spn * snn > 0 && spg * sng > 0;
  return spn * snn < 0 && spg * sng < 0;
}

struct Chain2 {
  bool r1, r2;  // refraction at vertex 1 / 2
  double eta[3];
  Tri2 T1, T2;
  d3 x0, x3;
};
// exact forward shooting (c13): G = two components of (w2^ - target^) in the frame (f1, f2)
__device__ bool shoot2(const Chain2& C, double u1, double v1, d3 f1, d3 f2, double G[2], double* u2, double* v2) {
  const d3 x1 = C.T1.X(u1, v1);
  const d3 n1 = normalize(C.T1.N(u1, v1));
  d3 w1;
  if (!scatter_dir(C.r1, normalize(x1 - C.x0), n1, C.eta[0], C.eta[1], &w1)) return false;
  double t;
  if (!plane_hit(x1, w1, C.T2, u2, v2, &t) || !(t > 0)) return false;
  const d3 x2 = x1 + t * w1;
  const d3 n2 = normalize(C.T2.N(*u2, *v2));
  d3 w2;
  if (!scatter_dir(C.r2, normalize(w1), n2, C.eta[1], C.eta[2], &w2)) return false;
  const d3 dw = normalize(w2) - normalize(C.x3 - x2);
  G[0] = dot(dw, f1);
  G[1] = dot(dw, f2);
  return true;
}
__device__ void frame_of(d3 w, d3* a, d3* b) {
  const d3 ax = fabs(w.x) < 0.6 ? mk3(1, 0, 0) : (fabs(w.y) < 0.6 ? mk3(0, 1, 0) : mk3(0, 0, 1));
  *a = normalize(cross(w, ax));
  *b = cross(w, *a);
}
// light-side trace to the plane through x0 perpendicular to dref (c15)
__device__ bool light_trace2(const Chain2& C, d3 dref, d3 c1, d3 c2, d3 omega, double out[2]) {
  d3 o = C.x3, d = omega;
  for (int i = 1; i >= 0; --i) {
    const Tri2& T = i ? C.T2 : C.T1;
    double u, v, t;
    if (!plane_hit(o, d, T, &u, &v, &t) || !(t > 0)) return false;
    const d3 x = o + t * d;
    const d3 n = normalize(T.N(u, v));
    d3 nd;
    if (!scatter_dir(i ? C.r2 : C.r1, d, n, C.eta[i + 1], C.eta[i], &nd)) return false;
    o = x;
    d = normalize(nd);
  }
  const double den = dot(d, dref);
  if (den == 0.0) return false;
  const double t = dot(C.x0 - o, dref) / den;
  const d3 p = o + t * d - C.x0;
  out[0] = dot(p, c1);
  out[1] = dot(p, c2);
  return true;
}
__device__ double jacobian2(const Chain2& C, d3 x1, d3 x2) {
  const d3 dref = normalize(C.x0 - x1);
  d3 c1, c2, b1, b2;
  frame_of(dref, &c1, &c2);
  const d3 w = normalize(x2 - C.x3);
  frame_of(w, &b1, &b2);
  double j[2][2];
  for (int k = 0; k < 2; ++k) {
    const d3 b = k ? b2 : b1;
    double dh[2], dq[2];
    for (int pass = 0; pass < 2; ++pass) {
      const double h = pass ? 0.5e-5 : 1e-5;
      double p[2], m[2];
      if (!light_trace2(C, dref, c1, c2, normalize(w + h * b), p) ||
          !light_trace2(C, dref, c1, c2, normalize(w - h * b), m))
        return -1.0;
      double* o = pass ? dq : dh;
      o[0] = (p[0] - m[0]) / (2 * h);
      o[1] = (p[1] - m[1]) / (2 * h);
    }
    j[k][0] = (4 * dq[0] - dh[0]) / 3;
    j[k][1] = (4 * dq[1] - dh[1]) / 3;
  }
  return fabs(j[0][0] * j[1][1] - j[0][1] * j[1][0]);
}

// ------------------------------------------------------------------ kernel
template <bool V1T, bool V2T>
__global__ void __launch_bounds__(64) k2_solve(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                               uint64_t npairs, const TriRec* __restrict__ tris,
                                               const double* __restrict__ ep, const double* __restrict__ inten,
                                               SolveParams prm, SolSink S) {
  using Sy = Sys2<V1T, V2T>;
  constexpr int MAXN = Sy::DB;
  constexpr int MAXV = 40;
  uint32_t cnt[C_NUM];
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = gw * 32; base < npairs; base += nw * 32) {
    const uint64_t pi = base + lane;
    const bool active = pi < npairs;
    uint32_t flags = 0;
    int nsol = 0;
    double su[4][4], scontrib[4];
    float sres[4];
    uint32_t sslot[4];
    if (active) {
      const uint32_t q = pq[pi];
      Chain2 C;
      load_tri(tris, pt[2 * pi], C.T1.p, C.T1.n);
      load_tri(tris, pt[2 * pi + 1], C.T2.p, C.T2.n);
      const double* e = ep + 6ull * q;
      C.x0 = mk3(e[0], e[1], e[2]);
      C.x3 = mk3(e[3], e[4], e[5]);
      C.r1 = V1T;
      C.r2 = V2T;
      cnt[C_PAIRS]++;
      Sy Sys;
      const bool ok = build_system2<V1T, V2T>(C.x0, C.x3, C.T1, C.T2, prm, Sys);
      flags |= Sys.flags;
      C.eta[0] = Sys.eta0;
      C.eta[1] = Sys.eta1;
      C.eta[2] = Sys.eta2;
      if (ok) {
        cnt[C_SYSTEMS]++;
        // algorithmic FLOPs (kFLOP units): coefficient phase (dense products of the Eq. 13-23 chain,
        // counted in DESIGN.md §5: RR 17k, RT 40k, TR 150k, TT 400k) + per determinant evaluation:
        // slices 2 (sum of the a_i, b_i lengths, i <= n) + Chionh 3 n^2 + GE (2/3) n^3
        const double build_f = (!V1T && !V2T) ? 17e3 : (!V1T ? 40e3 : (!V2T ? 150e3 : 400e3));
        double slice_terms = 0;
        for (int i = 0; i <= Sys.n; ++i)
          slice_terms += (i <= Sys.da ? Sy::DA - i + 1 : 0) + (i <= Sys.db ? Sy::DB - i + 1 : 0);
        const double nn = (double)Sys.n;
        const double eval_f = 2.0 * slice_terms + 3.0 * nn * nn + (2.0 / 3.0) * nn * nn * nn;
        double kflop_acc = build_f;
        // ---- 100-piece determinant-sign scan
        double M[MAXN * MAXN];
        const int P = prm.pieces;
        double vroots[MAXV];
        int nv = 0;
        int s_prev = 0, last_change = -10;
        double lg_prev = -INFINITY, lg_prev2 = -INFINITY;
        int s_cur;
        double lg_cur;
        s_cur = det_sign_at<V1T, V2T>(Sys, 0.0, &lg_cur, M);
        kflop_acc += eval_f;
        for (int j = 0; j <= P; ++j) {
          int s_next = 0;
          double lg_next = -INFINITY;
          if (j < P) {
            s_next = det_sign_at<V1T, V2T>(Sys, (double)(j + 1) / P, &lg_next, M);
            kflop_acc += eval_f;
          }
          // near-tangent: |det(v_j)| < 1e-9 max(neighbours)
          const double nb = fmax(lg_prev, lg_next);
          if (lg_cur < log(1e-9) + nb) flags |= SPOLY_FLAG_NEAR_TANGENT;
          if (s_cur == 0) {
            if (nv < MAXV) vroots[nv++] = (double)j / P;
          } else if (j < P && s_next != 0 && s_next != s_cur) {
            if (j - last_change == 1) flags |= SPOLY_FLAG_NEAR_TANGENT;
            last_change = j;
            double lo = (double)j / P, hi = (double)(j + 1) / P;
            for (int it = 0; it < prm.scan_bisect_iters; ++it) {
              const double m = 0.5 * (lo + hi);
              double l2;
              const int sm = det_sign_at<V1T, V2T>(Sys, m, &l2, M);
              kflop_acc += eval_f;
              if (sm == 0) {
                lo = hi = m;
                break;
              }
              if (sm == s_cur)
                lo = m;
              else
                hi = m;
            }
            if (nv < MAXV) vroots[nv++] = 0.5 * (lo + hi);
          }
          lg_prev2 = lg_prev;
          lg_prev = lg_cur;
          s_prev = s_cur;
          s_cur = s_next;
          lg_cur = lg_next;
        }
        (void)s_prev;
        (void)lg_prev2;
        cnt[C_KFLOP] += (uint32_t)(kflop_acc * 1e-3);
        cnt[C_VROOTS] += nv;
        // ---- path phase
        constexpr int NA = Sy::DB + 1;
        for (int iv = 0; iv < nv; ++iv) {
          const double vs = vroots[iv];
          double Acoef[NA];
          bp_slices(Sys.a, Sys.da, vs, Acoef);
          int dA = Sys.da;
          double amax = 0;
          for (int i = 0; i <= dA; ++i) amax = fmax(amax, fabs(Acoef[i]));
          if (!(amax >= 1e-12)) {
            bp_slices(Sys.b, Sys.db, vs, Acoef);
            dA = Sys.db;
            amax = 0;
            for (int i = 0; i <= dA; ++i) amax = fmax(amax, fabs(Acoef[i]));
            if (!(amax >= 1e-12)) {
              flags |= SPOLY_FLAG_DEGENERATE;
              continue;
            }
          }
          while (dA > 0 && Acoef[dA] == 0.0) --dA;
          double us[MAXV];
          int nu = 0;
          if (dA == 1) {
            us[nu++] = -Acoef[0] / Acoef[1];
          } else if (dA == 2) {
            const double a0 = Acoef[0], a1 = Acoef[1], a2 = Acoef[2];
            double disc = a1 * a1 - 4 * a2 * a0;
            const double sc = a1 * a1 + 4 * fabs(a2 * a0);
            if (fabs(disc) <= 1e-8 * sc) flags |= SPOLY_FLAG_NEAR_TANGENT;
            if (!(disc < -1e-12 * sc)) {
              if (disc < 0) disc = 0;
              const double qq = -0.5 * (a1 + copysign(sqrt(disc), a1));
              if (qq == 0.0) {
                us[nu++] = 0.0;
              } else {
                double r1 = qq / a2, r2 = a0 / qq;
                if (r1 > r2) {
                  const double t = r1;
                  r1 = r2;
                  r2 = t;
                }
                us[nu++] = r1;
                if (r2 - r1 >= 1e-7) us[nu++] = r2;
              }
            }
          } else if (dA > 2) {
            RootSet<NA> Ru;
            isolate_roots<NA>(Acoef, dA, -0.1, 1.1, 1e-7, Ru);
            for (int i = 0; i < Ru.n && nu < MAXV; ++i)
              if (nu == 0 || Ru.x[i] - us[nu - 1] >= 1e-7) us[nu++] = Ru.x[i];
          }
          for (int iu = 0; iu < nu; ++iu) {
            cnt[C_CANDIDATES]++;
            const double ur = us[iu], vr = vs;
            const double kap = bp_eval(Sys.K, ur, vr), ut = bp_eval(Sys.U, ur, vr), vt = bp_eval(Sys.V, ur, vr);
            double u2 = ut / kap, v2 = vt / kap;
            if (!(fabs(kap) > 0) || !isfinite(u2) || !isfinite(v2)) {
              cnt[C_REJ_KAPPA]++;
              continue;
            }
            if (Sys.relabel) {
              const double t = u2;
              u2 = v2;
              v2 = t;
            }
            const double dm = 1e-3;
            if (!(ur >= -dm && vr >= -dm && ur + vr <= 1 + dm && u2 >= -dm && v2 >= -dm && u2 + v2 <= 1 + dm)) {
              cnt[C_REJ_DOMAIN]++;
              continue;
            }
            d3 x1 = C.T1.X(ur, vr), x2 = C.T2.X(u2, v2);
            double r1 = resid(C.x0, x1, x2, C.T1.N(ur, vr), C.eta[0], C.eta[1]);
            double r2 = resid(x1, x2, C.x3, C.T2.N(u2, v2), C.eta[1], C.eta[2]);
            if (!(fmax(r1, r2) < prm.theta_admit)) {
              cnt[C_REJ_CONSTRAINT]++;
              continue;
            }
            // polish: <= polish_iters Newton steps on the exact shooting residual, keep if |G| decreases
            d3 f1, f2;
            frame_of(normalize(C.x3 - x2), &f1, &f2);
            double uu = ur, vv = vr, G[2], uu2 = u2, vv2 = v2;
            bool okp = shoot2(C, uu, vv, f1, f2, G, &uu2, &vv2);
            double Jm[4] = {0, 0, 0, 0};
            for (int it = 0; okp && it < prm.polish_iters; ++it) {
              const double h = 1e-7;
              double Gp[2], Gm[2], t1, t2;
              if (!shoot2(C, uu + h, vv, f1, f2, Gp, &t1, &t2) || !shoot2(C, uu - h, vv, f1, f2, Gm, &t1, &t2)) break;
              Jm[0] = (Gp[0] - Gm[0]) / (2 * h);
              Jm[2] = (Gp[1] - Gm[1]) / (2 * h);
              if (!shoot2(C, uu, vv + h, f1, f2, Gp, &t1, &t2) || !shoot2(C, uu, vv - h, f1, f2, Gm, &t1, &t2)) break;
              Jm[1] = (Gp[0] - Gm[0]) / (2 * h);
              Jm[3] = (Gp[1] - Gm[1]) / (2 * h);
              const double det = Jm[0] * Jm[3] - Jm[1] * Jm[2];
              if (det == 0.0) break;
              const double du = -(Jm[3] * G[0] - Jm[1] * G[1]) / det;
              const double dv = -(-Jm[2] * G[0] + Jm[0] * G[1]) / det;
              double Gn[2], nu2, nv2;
              if (!shoot2(C, uu + du, vv + dv, f1, f2, Gn, &nu2, &nv2)) break;
              if (!(hypot(Gn[0], Gn[1]) < hypot(G[0], G[1]))) break;
              uu += du;
              vv += dv;
              G[0] = Gn[0];
              G[1] = Gn[1];
              uu2 = nu2;
              vv2 = nv2;
            }
            if (!okp) {
              cnt[C_REJ_CONSTRAINT]++;
              continue;
            }
            const double ed = prm.eps_domain;
            if (!(uu >= -ed && vv >= -ed && uu + vv <= 1 + ed && uu2 >= -ed && vv2 >= -ed && uu2 + vv2 <= 1 + ed)) {
              cnt[C_REJ_DOMAIN]++;
              continue;
            }
            x1 = C.T1.X(uu, vv);
            x2 = C.T2.X(uu2, vv2);
            const d3 n1 = C.T1.N(uu, vv), n2 = C.T2.N(uu2, vv2);
            r1 = resid(C.x0, x1, x2, n1, C.eta[0], C.eta[1]);
            r2 = resid(x1, x2, C.x3, n2, C.eta[1], C.eta[2]);
            const double rho = fmax(r1, r2);
            if (!(rho < prm.theta_final)) {
              cnt[C_REJ_CONSTRAINT]++;
              continue;
            }
            if (!sides(C.r1, C.x0, x1, x2, n1, C.T1.g()) || !sides(C.r2, x1, x2, C.x3, n2, C.T2.g())) {
              cnt[C_REJ_SIDE]++;
              continue;
            }
            if (C.r2) {  // eta consistency: x_1 on the side of T_2 whose IOR is eta_1
              const double se = dot(x1 - C.T2.p[0], C.T2.g()) > 0 ? prm.eta_front : prm.eta_back;
              if (se != C.eta[1]) {
                cnt[C_REJ_SIDE]++;
                continue;
              }
            }
            if (rho >= 1e-7) flags |= SPOLY_FLAG_RESIDUAL;
            const double e1d = fmin(fmin(uu, vv), 1 - uu - vv), e2d = fmin(fmin(uu2, vv2), 1 - uu2 - vv2);
            if (e1d <= prm.eps_flag || e2d <= prm.eps_flag) flags |= SPOLY_FLAG_BOUNDARY;
            if (fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]) < 1e-6 * hypot(Jm[0], Jm[1]) * hypot(Jm[2], Jm[3]))
              flags |= SPOLY_FLAG_NEAR_TANGENT;
            bool dup = false;
            for (int s = 0; s < nsol; ++s)
              if (fabs(su[s][0] - uu) < 1e-7 && fabs(su[s][1] - vv) < 1e-7) dup = true;
            if (dup) {
              cnt[C_REJ_SIDE]++;
              continue;
            }
            if (nsol < 4) {
              const double J = jacobian2(C, x1, x2);
              const double I = inten ? inten[q] : 1.0;
              su[nsol][0] = uu;
              su[nsol][1] = vv;
              su[nsol][2] = uu2;
              su[nsol][3] = vv2;
              scontrib[nsol] = J > 0 ? I / J : 0.0;
              sres[nsol] = (float)rho;
              sslot[nsol] = (uint32_t)nsol;  // processing order: deterministic
              nsol++;
              cnt[C_ADMISSIBLE]++;
            }
          }
        }
      }
    }
    // emission (warp-aggregated, all lanes)
    {
      const bool hf = active && flags != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, hf);
      if (bal) {
        unsigned long long fb = 0;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) fb = atomicAdd(S.count + 1, (unsigned long long)__popc(bal));
        fb = __shfl_sync(0xffffffffu, fb, leader);
        if (hf) {
          const unsigned long long p = fb + __popc(bal & ((1u << lane) - 1u));
          if (p < S.fcapacity) {
            S.fkey[p] = pi;
            S.fflags[p] = flags;
          }
        }
      }
      uint32_t n = active ? (uint32_t)nsol : 0u, incl = n;
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tot) {
        unsigned long long b = 0;
        if (lane == 31) b = atomicAdd(S.count, (unsigned long long)tot);
        b = __shfl_sync(0xffffffffu, b, 31);
        for (uint32_t s = 0; s < n; ++s) {
          const unsigned long long p = b + incl - n + s;
          if (p < S.capacity) {
            S.key[p] = ((unsigned long long)pi << 6) | sslot[s];
            for (int c = 0; c < 4; ++c) S.bary[4 * p + c] = su[s][c];
            S.contrib[p] = scontrib[s];
            S.resid[p] = sres[s];
          }
        }
      }
    }
  }
  for (int i = 0; i < C_NUM; ++i) {
    uint32_t v = cnt[i];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0 && v) atomicAdd(S.counters + i, (unsigned long long)v);
  }
}

void launch_solve_k2(int v1t, int v2t, const uint32_t* pq, const uint32_t* pt, uint64_t npairs, const DeviceMesh& M,
                     const double* ep, const double* inten, const SolveParams& prm, const SolSink& S, int nsm,
                     cudaStream_t st) {
  if (!npairs) return;
  const int threads = 64;
  const uint64_t want = (npairs + threads - 1) / threads;
  const uint64_t cap = (uint64_t)nsm * 8;
  const int g = (int)(want < cap ? want : cap);
  if (v1t && v2t)
    k2_solve<true, true><<<g, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, inten, prm, S);
  else if (v1t)
    k2_solve<true, false><<<g, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, inten, prm, S);
  else if (v2t)
    k2_solve<false, true><<<g, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, inten, prm, S);
  else
    k2_solve<false, false><<<g, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, inten, prm, S);
}

}  // namespace spoly
