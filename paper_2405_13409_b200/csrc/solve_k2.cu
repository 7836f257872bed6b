// Two-bounce solve, chains "RR" (Eq. 23), "RT", "TR" and "TT" (Eqs. 13-20; square form at a refracting x_2,
// product form at a reflecting one; Table 3 rows).  One (query, triangle pair) per group
// of G lanes (G = 16 for RR, whose Bezout order is <= 15; 32 otherwise), FP64:
//
//   coefficient phase : rational coordinate mapping u_2 = (u~, v~)/kappa (Eqs. 13-16) of the scaled
//                       direction d~_1 (Eq. 17 reflection; Eqs. 18-20 refraction with the piecewise rational
//                       sqrt surrogate, reading R8), then a = Eq. 6 at x_2 and b = Eq. 12 (product form) /
//                       Eq. 9 (square form), denominators cleared; every bivariate product is computed by
//                       the group in shared memory (wpoly.cuh), then normalised + truncated (R6)
//   elimination       : Bezout matrix of Eq. 24 at v, columns by the Chionh recurrence across lanes
//   roots             : sign of det R(v_j) at v_j = j/100 by register-resident Gaussian elimination with
//                       partial pivoting (one row per lane), 10 bisections per sign-changing piece
//
//   path phase        : (lane 0) u-roots of a(., v*) on [-0.1, 1.1], mapping to u_2, raw admission
//                       (theta_admit), <= 3 Newton steps on the exact shooting residual, final
//                       Eq. 3 validation, sides, flags, contribution I / J (J by central differences of the
//                       light-side trace, Richardson), emission.
#include "kernels.cuh"
#include "poly_dev.cuh"
#include "wpoly.cuh"

#include <algorithm>
#include <cstdio>

namespace spoly {

#ifdef SPOLY_PROF_BUILD  // section timing of the two-bounce build (clock64 per system, lane 0; diagnostic only)
__device__ unsigned long long g_bprof[16];
#define BPROF_INIT long long bprof_t = clock64();
#define BPROF(k)                                                   \
  do {                                                             \
    const long long bprof_n = clock64();                           \
    if (g.lane == 0) atomicAdd(&g_bprof[k], (unsigned long long)(bprof_n - bprof_t)); \
    bprof_t = bprof_n;                                             \
  } while (0)
#else
#define BPROF_INIT
#define BPROF(k)
#endif

struct Tri2 {
  d3 p[3], n[3];
  __device__ d3 e1() const { return p[1] - p[0]; }
  __device__ d3 e2() const { return p[2] - p[0]; }
  __device__ d3 g() const { return cross(p[1] - p[0], p[2] - p[0]); }
  __device__ d3 X(double u, double v) const { return p[0] + u * (p[1] - p[0]) + v * (p[2] - p[0]); }
  __device__ d3 N(double u, double v) const { return n[0] + u * (n[1] - n[0]) + v * (n[2] - n[0]); }
  __device__ d3 c() const { return (1.0 / 3.0) * (p[0] + p[1] + p[2]); }
};

// piecewise rational sqrt surrogate (Eq. 20): literal copy of tests/golden/sqrt_table.txt (our fit, R8); the
// same literal fills the device table and the host copy spoly_sqrt_table() returns, and the tests compare
// both (the device one read back from constant memory) with the golden file
#define SPOLY_SQRT_TAB                                                                                            \
  {{0, 0.00042432536375417839, 0.00089999999999879705, 154.92902483814683, 5615.7008147954339},                 \
   {0.00042432536375417839, 0.0077313602416299448, 0.013714746392967799, 21.253136166194601, 135.24944765874642}, \
   {0.0077313602416299448, 0.051793068389647277, 0.04635497395617269, 6.7900571325924943, 14.594946360257405},    \
   {0.051793068389647277, 0.21636853563098274, 0.10736470812718857, 3.006160575603614, 2.9223382765562778},       \
   {0.21636853563098274, 0.68268233146982271, 0.20527897991137517, 1.5904325277264706, 0.82650456712266585},      \
   {0.68268233146982271, 1, 0.30276242425651556, 1.0984677499357838, 0.40129928835931156}}
__constant__ double c_sqrt_tab[6][5] = SPOLY_SQRT_TAB;
static const double h_sqrt_tab[6][5] = SPOLY_SQRT_TAB;

cudaError_t k2_sqrt_table(int from_device, double* out30) {
  if (from_device) return cudaMemcpyFromSymbol(out30, c_sqrt_tab, sizeof(h_sqrt_tab));
  for (int i = 0; i < 30; ++i) out30[i] = h_sqrt_tab[i / 5][i % 5];
  return cudaSuccess;
}

#ifndef SPOLY_TT_ARENA
// TT: room for P^2 and Q^2 side by side (one batched product, then b in one two-term pass); 2 x 27.2 KB per block,
// 4 blocks per SM (the register budget's limit) still fit the 228 KB of shared memory
#define SPOLY_TT_ARENA 3400
#endif
// polynomial degrees of the chain X1 X2 (X = R reflection / T refraction)
template <bool V1T, bool V2T>
struct Deg2 {
  static constexpr int DK = V1T ? 7 : 3;  // deg kappa = deg d~_1 (Eq. 17: 3; Eqs. 19-20 cleared: 7)
  static constexpr int DU = DK + 1;       // deg u~, v~
  static constexpr int DA = 2 * DK + 3;   // deg a: 9 (R.), 17 (T.)
  // deg b: product form (d~.N2)(D2.T2)+..: DK+DU+2DU; square form D2^2 P^2: 2DU + 2(DK+DU)
  static constexpr int DB = V2T ? 2 * DU + 2 * (DK + DU) : (DK + DU) + 2 * DU;  // RR 15, RT 22, TR 31, TT 46
  static constexpr int G = (DB <= 15) ? 16 : 32;                               // lanes per system
  // shared-memory arena per group (doubles): persistent a, b, U, V, K + the build temporaries (peak) +
  // the v-root list; the n > 32 determinant scratch reuses the temporaries (TT only)
  static constexpr int ARENA = (!V1T && !V2T) ? 640 : (!V1T ? 768 : (!V2T ? 1984 : SPOLY_TT_ARENA));
};

struct Sys2w {
  WP a, b, U, V, K;
  double eta0, eta1, eta2;
  int tb;  // b's effective total degree (reading R29)
  bool relabel;
  uint32_t flags;
  int da, db, n;
};

// coefficient phase, group-cooperative (same construction as the oracle's)
template <bool V1T, bool V2T, int G>
__device__ bool build_w(const Grp<G>& g, Arena& ar, d3 x0, d3 x3, const Tri2& T1, const Tri2& T2in,
                        const SolveParams& prm, Sys2w& S) {
  using D = Deg2<V1T, V2T>;
  constexpr int DK = D::DK, DU = D::DU;
  BPROF_INIT
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
  // persistent polynomials first
  S.a = ar.poly(D::DA);
  S.b = ar.poly(D::DB);
  S.U = ar.poly(DU);
  S.V = ar.poly(DU);
  S.K = ar.poly(DK);
  const int mark = ar.top;
  // X1 = p0 + u e1 + v e2, N1 = n0 + u m1 + v m2, D0 = X1 - x0   (Eqs. 1-2)
  const d3 e1 = T1.e1(), e2 = T1.e2(), m1 = T1.n[1] - T1.n[0], m2 = T1.n[2] - T1.n[0];
  WV X1 = ar.vec(1), N1 = ar.vec(1), D0 = ar.vec(1);
  wlinear3(g, X1, T1.p[0], e1, e2);
  wlinear3(g, N1, T1.n[0], m1, m2);
  wlinear3(g, D0, T1.p[0] - x0, e1, e2);
  WP dn = ar.poly(2), nn = ar.poly(2);
  wdot(g, dn, D0, N1, 1.0, false);
  wdot(g, nn, N1, N1, 1.0, false);
  BPROF(0);
  WV Dt = ar.vec(DK);
  if (!V1T) {
    // Eq. 17: d~ = -2 (d0 . n) n + d0 n^2
#ifndef SPOLY_NO_BATCH
    wmul2x3(g, Dt, wv_rep(dn), N1, -2.0, wv_rep(nn), D0, 1.0, false);
#else
    wmul2(g, Dt.x, dn, N1.x, -2.0, nn, D0.x, 1.0, false);
    wmul2(g, Dt.y, dn, N1.y, -2.0, nn, D0.y, 1.0, false);
    wmul2(g, Dt.z, dn, N1.z, -2.0, nn, D0.z, 1.0, false);
#endif
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
    WP dd = ar.poly(2), nd = ar.poly(4), dn2 = ar.poly(4), beta = ar.poly(4), den = ar.poly(4), sq = ar.poly(4);
    wdot(g, dd, D0, D0, 1.0, false);
    wmul1(g, nd, nn, dd, 1.0, false);
    wmul1(g, dn2, dn, dn, 1.0, false);
    wlin2(g, beta, nd, 1.0 - ep * ep, dn2, ep * ep, false);  // beta = nn dd - ep^2 (nn dd - dn^2)  (Eq. 19)
    wlin1(g, den, beta, c_sqrt_tab[piece][4], false);
    wadd0(g, den, s);
    wlin1(g, sq, beta, c_sqrt_tab[piece][3], false);
    wadd0(g, sq, c_sqrt_tab[piece][2] * s);
    WV tang = ar.vec(3);  // nn D0 - dn N1
#ifndef SPOLY_NO_BATCH
    wmul2x3(g, tang, wv_rep(nn), D0, 1.0, wv_rep(dn), N1, -1.0, false);
#else
    wmul2(g, tang.x, nn, D0.x, 1.0, dn, N1.x, -1.0, false);
    wmul2(g, tang.y, nn, D0.y, 1.0, dn, N1.y, -1.0, false);
    wmul2(g, tang.z, nn, D0.z, 1.0, dn, N1.z, -1.0, false);
#endif
    const double k2 = -sigma * sqrt(s);
#ifndef SPOLY_NO_BATCH
    wmul2x3(g, Dt, wv_rep(den), tang, ep, wv_rep(sq), N1, k2, false);
#else
    wmul2(g, Dt.x, den, tang.x, ep, sq, N1.x, k2, false);
    wmul2(g, Dt.y, den, tang.y, ep, sq, N1.y, k2, false);
    wmul2(g, Dt.z, den, tang.z, ep, sq, N1.z, k2, false);
#endif
  }
  BPROF(1);
  // rational coordinate mapping onto T_2 (Eqs. 13-16)
  const d3 f1 = T2.e1(), f2 = T2.e2(), r0 = T2.n[0], g1 = T2.n[1] - T2.n[0], g2 = T2.n[2] - T2.n[0];
  const bool face2 = T2.n[1].x == r0.x && T2.n[1].y == r0.y && T2.n[1].z == r0.z && T2.n[2].x == r0.x &&
                     T2.n[2].y == r0.y && T2.n[2].z == r0.z;
  WV Sv = ar.vec(1);  // x_1 - p_{2,0}
  wlinear3(g, Sv, T1.p[0] - T2.p[0], e1, e2);
  WV Dxf2 = ar.vec(DK);
  wcross_c(g, Dxf2, Dt, f2);
  wlin3(g, S.K, Dxf2.x, f1.x, Dxf2.y, f1.y, Dxf2.z, f1.z, false);     // kappa = (d~ x e22) . e21
  WV Sxf1 = ar.vec(1);
  wcross_c(g, Sxf1, Sv, f1);
#ifndef SPOLY_NO_BATCH
  {  // u~ = (d~ x e22) . (x1 - p20), v~ = ((x1 - p20) x e21) . d~, side by side
    const WP c[2] = {S.U, S.V};
    const WP a[2][3] = {{Dxf2.x, Dxf2.y, Dxf2.z}, {Sxf1.x, Sxf1.y, Sxf1.z}};
    const WP b[2][3] = {{Sv.x, Sv.y, Sv.z}, {Dt.x, Dt.y, Dt.z}};
    const double sc[2][3] = {{1, 1, 1}, {1, 1, 1}};
    wmul_batch<G, 3, 2>(g, c, a, b, sc, false);
  }
#else
  wdot(g, S.U, Dxf2, Sv, 1.0, false);                                 // u~ = (d~ x e22) . (x1 - p20)
  wdot(g, S.V, Sxf1, Dt, 1.0, false);                                 // v~ = ((x1 - p20) x e21) . d~
#endif
  // kappa x_2 and kappa n_2
  WV X2 = ar.vec(DU), N2 = ar.vec(DU);
  wlin3(g, X2.x, S.K, T2.p[0].x, S.U, f1.x, S.V, f2.x, false);
  wlin3(g, X2.y, S.K, T2.p[0].y, S.U, f1.y, S.V, f2.y, false);
  wlin3(g, X2.z, S.K, T2.p[0].z, S.U, f1.z, S.V, f2.z, false);
  if (face2) {
    // face mode (n_2 = n_{2,0} constant): kappa n_2 would be kappa n_{2,0}, a factor kappa common
    // to a and b (det R == 0 identically), so the constant normal enters instead (reading R22)
    for (int i = g.lane; i < tri_n(DU); i += G) {
      N2.x.c[i] = i == 0 ? r0.x : 0.0;
      N2.y.c[i] = i == 0 ? r0.y : 0.0;
      N2.z.c[i] = i == 0 ? r0.z : 0.0;
    }
    g.sync();
  } else {
    wlin3(g, N2.x, S.K, r0.x, S.U, g1.x, S.V, g2.x, false);
    wlin3(g, N2.y, S.K, r0.y, S.U, g1.y, S.V, g2.y, false);
    wlin3(g, N2.z, S.K, r0.z, S.U, g1.z, S.V, g2.z, false);
  }
  BPROF(2);
  // a = ((X2 - K X1) x (x3 - X1)) . N2   (Eq. 6 at x_2, Eq. 23 first line)
  {
    const int m2 = ar.top;
    WV W = ar.vec(DU);
#ifndef SPOLY_NO_BATCH
    wlin1(g, W.x, X2.x, 1.0, false);
    wlin1(g, W.y, X2.y, 1.0, false);
    wlin1(g, W.z, X2.z, 1.0, false);
    wmul1x3(g, W, wv_rep(S.K), X1, -1.0, true);
#else
    wlin1(g, W.x, X2.x, 1.0, false); wmul1(g, W.x, S.K, X1.x, -1.0, true);
    wlin1(g, W.y, X2.y, 1.0, false); wmul1(g, W.y, S.K, X1.y, -1.0, true);
    wlin1(g, W.z, X2.z, 1.0, false); wmul1(g, W.z, S.K, X1.z, -1.0, true);
#endif
    WV Y = ar.vec(1);
    wlinear3(g, Y, x3 - T1.p[0], -1.0 * e1, -1.0 * e2);
    WV Cc = ar.vec(DU + 1);
#ifndef SPOLY_NO_BATCH
    wmul2x3(g, Cc, WV{W.y, W.z, W.x}, WV{Y.z, Y.x, Y.y}, 1.0, WV{W.z, W.x, W.y}, WV{Y.y, Y.z, Y.x}, -1.0, false);
#else
    wcross(g, Cc, W, Y);
#endif
    wdot(g, S.a, Cc, N2, 1.0, false);
    ar.top = m2;
  }
  BPROF(3);
  // D2 = K x3 - X2 (kappa d_2)
  WV D2 = ar.vec(DU);
  wlin2(g, D2.x, S.K, x3.x, X2.x, -1.0, false);
  wlin2(g, D2.y, S.K, x3.y, X2.y, -1.0, false);
  wlin2(g, D2.z, S.K, x3.z, X2.z, -1.0, false);
  // only d~, N2, D2 are live from here: compact them to the bottom of the temporary region
  {
    double* dst = S.K.c + tri_n(DK);
    dst = wmovev(g, Dt, dst);
    dst = wmovev(g, N2, dst);
    dst = wmovev(g, D2, dst);
    ar.top = (int)(dst - ar.base);
  }
  if (!V2T) {
    // b = (d~.N2)(D2.T2) + (d~.T2)(D2.N2), T2 = N2 x e21   (Eq. 12 with d~_1, Eq. 23)
    WV Tt = ar.vec(DU);
    wcross_c(g, Tt, N2, f1);
    WP p1 = ar.poly(DK + DU), p2 = ar.poly(2 * DU), p3 = ar.poly(DK + DU), p4 = ar.poly(2 * DU);
#ifndef SPOLY_NO_BATCH
    wdot4(g, p1, Dt, N2, p2, D2, Tt, p3, Dt, Tt, p4, D2, N2);
#else
    wdot(g, p1, Dt, N2, 1.0, false);
    wdot(g, p2, D2, Tt, 1.0, false);
    wdot(g, p3, Dt, Tt, 1.0, false);
    wdot(g, p4, D2, N2, 1.0, false);
#endif
    wmul2(g, S.b, p1, p2, 1.0, p3, p4, 1.0, false);
  } else {
    // b = eta1^2 D2^2 ((d~ x N2).l)^2 - eta2^2 d~^2 ((D2 x N2).l)^2   (Eq. 9 at x_2); (A x N2).l = A.(N2 x l)
    WV Nl = ar.vec(DU);
    wcross_c(g, Nl, N2, ell);
    WP P = ar.poly(DK + DU), Q = ar.poly(2 * DU), d22 = ar.poly(2 * DU), dt2 = ar.poly(2 * DK);
#ifndef SPOLY_NO_BATCH
    wdot4(g, P, Dt, Nl, Q, D2, Nl, d22, D2, D2, dt2, Dt, Dt);
#else
    wdot(g, P, Dt, Nl, 1.0, false);
    wdot(g, Q, D2, Nl, 1.0, false);
    wdot(g, d22, D2, D2, 1.0, false);
    wdot(g, dt2, Dt, Dt, 1.0, false);
#endif
    {  // only P, Q, D2^2, d~^2 are live from here
      double* dst = S.K.c + tri_n(DK);
      wmove(g, P, dst);
      dst += tri_n(P.d);
      wmove(g, Q, dst);
      dst += tri_n(Q.d);
      wmove(g, d22, dst);
      dst += tri_n(d22.d);
      wmove(g, dt2, dst);
      dst += tri_n(dt2.d);
      ar.top = (int)(dst - ar.base);
    }
    BPROF(4);
#ifndef SPOLY_NO_BATCH
    if (D::ARENA - ar.top >= tri_n(2 * (DK + DU)) + tri_n(4 * DU)) {
      // P^2 and Q^2 side by side, then b = eta1^2 d22 P^2 - eta2^2 dt2 Q^2 in one two-term pass (the same fma
      // sequence per coefficient as two passes)
      WP P2 = ar.poly(2 * (DK + DU)), Q2 = ar.poly(4 * DU);
      {
        const WP c[2] = {P2, Q2};
        const WP a[2][1] = {{P}, {Q}}, b[2][1] = {{P}, {Q}};
        const double sc[2][1] = {{1.0}, {1.0}};
        wmul_batch<G, 1, 2>(g, c, a, b, sc, false);
      }
      wmul2(g, S.b, d22, P2, S.eta1 * S.eta1, dt2, Q2, -S.eta2 * S.eta2, false);
    } else
#endif
    {
      WP PQ2 = ar.poly(4 * DU);
      WP P2{PQ2.c, 2 * (DK + DU)};
      wmul1(g, P2, P, P, 1.0, false);
      wmul1(g, S.b, d22, P2, S.eta1 * S.eta1, false);
      wmul1(g, PQ2, Q, Q, 1.0, false);
      wmul1(g, S.b, dt2, PQ2, -S.eta2 * S.eta2, true);
    }
  }
  BPROF(5);
  ar.top = mark;
  if (ar.overflow) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  // normalise and truncate (R6)
  const int na = tri_n(S.a.d), nb = tri_n(S.b.d);
  double ma = 0, mb = 0;
  for (int i = g.lane; i < na; i += G) ma = fmax(ma, fabs(S.a.c[i]));
  for (int i = g.lane; i < nb; i += G) mb = fmax(mb, fabs(S.b.c[i]));
  ma = g.max_(ma);
  mb = g.max_(mb);
  if (!(ma > 0) || !(mb > 0)) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  const double ia = 1.0 / ma, ib = 1.0 / mb;
  for (int i = g.lane; i < na; i += G) S.a.c[i] *= ia;
  for (int i = g.lane; i < nb; i += G) S.b.c[i] *= ib;
  g.sync();
  int da = 0, db = 0;
  for (int i = g.lane; i <= S.a.d; i += G) {
    double m = 0, f = 1.0;
    for (int j = 0; j <= S.a.d - i; ++j) m = fmax(m, fabs(S.a.c[poff(S.a.d, i) + j]));
    for (int t = 0; t < i; ++t) f *= 1.1;
    if (m * f > prm.tau_trunc) da = max(da, i);
  }
  for (int i = g.lane; i <= S.b.d; i += G) {
    double m = 0, f = 1.0;
    for (int j = 0; j <= S.b.d - i; ++j) m = fmax(m, fabs(S.b.c[poff(S.b.d, i) + j]));
    for (int t = 0; t < i; ++t) f *= 1.1;
    if (m * f > prm.tau_trunc) db = max(db, i);
  }
  S.da = g.imax(da);
  S.db = g.imax(db);
  S.n = max(S.da, S.db);
  BPROF(6);
#ifdef SPOLY_NO_TB
  S.tb = S.b.d;
#else
  {
    // reading R29: b's effective total degree T: its terms of total degree above T are bounded, on |u|, |v| <= 1.1,
    // by 2^-56 of max |b_ij| (= 1 after the normalisation); the scan evaluates each row only up to T
    double* mb = ar.raw(S.b.d + 1);
    wmass(g, S.b, mb);
    double tail;
    S.tb = trunc_degree(mb, S.b.d, 0x1p-56, &tail);
    g.sync();
    ar.top = mark;
  }
#endif
  BPROF(7);
  if (S.n == 0) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  return true;
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



// ------------------------------------------------------------------ per-pair system records (HBM)
// Written by the build kernel, read by the scan and path kernels.  Coefficients are stored transposed,
// [j * NR + i] = coefficient of u^i v^j (zero above the truncated u-degree and beyond the row), so the lane
// that owns row i reads consecutive addresses with its neighbours.
constexpr int kMaxV2 = 208;  // v-roots + c14 probes kept per pair: 100 pieces give <= 101 of each (more: TRUNCATED)
template <bool V1T, bool V2T>
struct Rec2 {
  using D = Deg2<V1T, V2T>;
  static constexpr int NR = D::DB <= 15 ? 16 : (D::DB <= 31 ? 32 : 48);
  static constexpr int VR = 16;  // header: eta0, eta1, eta2, relabel, flags, da, db, n, ok, nv
  static constexpr int AT = VR + kMaxV2;
  static constexpr int BT = AT + (D::DA + 1) * NR;
  static constexpr int U = BT + (D::DB + 1) * NR;
  static constexpr int V = U + tri_n(D::DU);
  static constexpr int K = V + tri_n(D::DU);
  static constexpr int STRIDE = (K + tri_n(D::DK) + 7) & ~7;
};
enum { H_ETA0 = 0, H_ETA1, H_ETA2, H_RELABEL, H_FLAGS, H_DA, H_DB, H_N, H_OK, H_NV, H_TB };
constexpr int kMaxSol2 = 8;  // admissible chains kept per pair (more: SPOLY_FLAG_TRUNCATED)

__device__ __forceinline__ void load_chain(const TriRec* __restrict__ tris, const uint32_t* __restrict__ pt,
                                           const double* __restrict__ ep, uint32_t q, uint64_t pi, Chain2& C) {
  load_tri(tris, pt[2 * pi], C.T1.p, C.T1.n);
  load_tri(tris, pt[2 * pi + 1], C.T2.p, C.T2.n);
  const double* e = ep + 6ull * q;
  C.x0 = mk3(e[0], e[1], e[2]);
  C.x3 = mk3(e[3], e[4], e[5]);
}

__device__ __forceinline__ void emit_flags(const SolSink& S, uint64_t pi, uint32_t flags) {
  const unsigned long long p = atomicAdd(S.count + 1, 1ull);
  if (p < S.fcapacity) {
    S.fkey[p] = pi;
    S.fflags[p] = flags;
  }
}

template <int G>
__device__ __forceinline__ void group_counters(const Grp<G>& g, const uint32_t* cnt, const SolSink& S) {
  for (int i = 0; i < C_NUM; ++i) {
    uint32_t v = (g.lane == 0) ? cnt[i] : 0u;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(S.counters + i, (unsigned long long)v);
  }
}

// ---- kernel 1: coefficient phase (group per pair, shared-memory arena), record write
constexpr int kBuildWarps = 2;
template <bool V1T, bool V2T>
__host__ __device__ constexpr int build_group() {
#ifdef SPOLY_BUILD_G16
  return 16;
#else
  return Deg2<V1T, V2T>::G;
#endif
}
#ifndef SPOLY_BUILD_MINB
#define SPOLY_BUILD_MINB 4  // 4 x 64 threads: up to 255 registers (5 blocks fit the TT arena but cap them at 168: spills)
#endif
template <bool V1T, bool V2T>
__global__ void __launch_bounds__(kBuildWarps * 32, SPOLY_BUILD_MINB) k2_build(const uint32_t* __restrict__ pq,
                                                            const uint32_t* __restrict__ pt, uint64_t p0,
                                                            uint64_t np, const TriRec* __restrict__ tris,
                                                            const double* __restrict__ ep, SolveParams prm,
                                                            double* __restrict__ recs, SolSink S,
                                                            unsigned long long* __restrict__ next) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  constexpr int G = build_group<V1T, V2T>(), GPW = 32 / G;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, gi = (threadIdx.x & 31) / G;
  Grp<G> g;
  g.lane = (threadIdx.x & 31) % G;
  g.mask = G == 32 ? 0xffffffffu : (0xffffu << (16 * gi));
  double* base = smem + (size_t)(warp * GPW + gi) * D::ARENA;
  uint32_t cnt[C_NUM];
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  while (true) {
    unsigned long long r = 0;
    if (g.lane == 0) r = atomicAdd(next, 1ull);
    r = g.bcast(r, 0);
    if (r >= np) break;
    const uint64_t pi = p0 + r;
    Chain2 C;
    load_chain(tris, pt, ep, pq[pi], pi, C);
    cnt[C_PAIRS]++;
    Arena ar{base, 0, D::ARENA, false};
    Sys2w Sy;
    const bool ok = build_w<V1T, V2T, G>(g, ar, C.x0, C.x3, C.T1, C.T2, prm, Sy);
    BPROF_INIT
    double* rec = recs + r * R::STRIDE;
    if (g.lane == 0) {
      rec[H_ETA0] = Sy.eta0;
      rec[H_ETA1] = Sy.eta1;
      rec[H_ETA2] = Sy.eta2;
      rec[H_RELABEL] = Sy.relabel ? 1.0 : 0.0;
      rec[H_FLAGS] = (double)Sy.flags;
      rec[H_DA] = ok ? Sy.da : 0;
      rec[H_DB] = ok ? Sy.db : 0;
      rec[H_N] = ok ? Sy.n : 0;
      rec[H_OK] = ok ? 1.0 : 0.0;
      rec[H_NV] = 0.0;
      rec[H_TB] = ok ? Sy.tb : 0;
    }
    if (ok) {
      cnt[C_SYSTEMS]++;
      for (int idx = g.lane; idx < (D::DA + 1) * R::NR; idx += G) {
        const int j = idx / R::NR, i = idx % R::NR;
        rec[R::AT + idx] = (i <= Sy.da && i + j <= D::DA) ? Sy.a.c[poff(D::DA, i) + j] : 0.0;
      }
      for (int idx = g.lane; idx < (D::DB + 1) * R::NR; idx += G) {
        const int j = idx / R::NR, i = idx % R::NR;
        rec[R::BT + idx] = (i <= Sy.db && i + j <= D::DB) ? Sy.b.c[poff(D::DB, i) + j] : 0.0;
      }
      for (int idx = g.lane; idx < tri_n(D::DU); idx += G) {
        rec[R::U + idx] = Sy.U.c[idx];
        rec[R::V + idx] = Sy.V.c[idx];
      }
      for (int idx = g.lane; idx < tri_n(D::DK); idx += G) rec[R::K + idx] = Sy.K.c[idx];
    }
    g.sync();
    BPROF(8);
  }
  group_counters(g, cnt, S);
}

// ---- binning by determinant order: one scan launch per order class keeps a single fully unrolled
// elimination variant per kernel (mixed variants thrashed the instruction cache: 28% no_instruction stalls)
template <int G>
__host__ __device__ constexpr int nc_of_class(int c) {
  return G == 16 ? (c == 0 ? 8 : (c == 1 ? 12 : 16)) : (c < 6 ? 12 + 4 * c : 0);
}
template <int G>
__device__ __forceinline__ int class_of(bool ok, int n) {
  if (!ok) return 0;
  if (G == 16) return n <= 8 ? 0 : (n <= 12 ? 1 : 2);
  return n <= 12 ? 0 : (n <= 16 ? 1 : (n <= 20 ? 2 : (n <= 24 ? 3 : (n <= 28 ? 4 : (n <= 32 ? 5 : 6)))));
}
constexpr int kMaxClasses = 8;

template <bool V1T, bool V2T>
__global__ void __launch_bounds__(256) k2_bin(uint64_t np, const double* __restrict__ recs,
                                              uint32_t* __restrict__ clist, unsigned long long* __restrict__ ccount) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; b < np;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = b + lane;
    int cls = -1;
    if (r < np) {
      const double* rec = recs + r * R::STRIDE;
      cls = class_of<D::G>(rec[H_OK] != 0.0, (int)rec[H_N]);
    }
    for (int c = 0; c < kMaxClasses; ++c) {
      const unsigned m = __ballot_sync(0xffffffffu, cls == c);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(ccount + c, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (cls == c) clist[(uint64_t)c * np + base + __popc(m & lt)] = (uint32_t)r;
    }
  }
}

// ---- kernel 2: 100-piece determinant-sign scan + bisection, group per pair of one order
// class: NC > 0 register determinant of that class; NC = 0 orders above 32 (shared-memory determinant)
constexpr int kScanWarps = 4;
// resident blocks per SM the register budget must allow: the scan is latency-bound (dependent shuffles and
// FP64 chains), so occupancy matters more than the compiler's unconstrained register use (252 for TT)
__host__ __device__ constexpr int scan_min_blocks(int nc) { return nc == 0 ? 1 : (nc <= 16 ? 4 : (nc <= 24 ? 3 : 2)); }
// lanes per system in the scan: a class with order <= 16 needs 16 rows, so two systems share a warp (the build's
// group is 32 wide for the chains whose b has more than 16 u-rows)
template <bool V1T, bool V2T>
__host__ __device__ constexpr int scan_group(int nc) {
#ifdef SPOLY_SCAN_G32
  return Deg2<V1T, V2T>::G;
#else
  return (nc > 0 && nc <= 16) ? 16 : Deg2<V1T, V2T>::G;
#endif
}
template <bool V1T, bool V2T, int NC>
__global__ void __launch_bounds__(kScanWarps * 32, scan_min_blocks(NC)) k2_scan(uint64_t p0, uint64_t np, SolveParams prm,
                                                          const uint32_t* __restrict__ vrange,
                                                          double* __restrict__ recs, SolSink S,
                                                          const uint32_t* __restrict__ clist,
                                                          const unsigned long long* __restrict__ ccount,
                                                          uint32_t* __restrict__ plist,
                                                          unsigned long long* __restrict__ pcount,
                                                          unsigned long long* __restrict__ next) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  constexpr int G = scan_group<V1T, V2T>(NC), GPW = 32 / G;
  constexpr bool BIG = NC == 0;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, gi = (threadIdx.x & 31) / G;
  Grp<G> g;
  g.lane = (threadIdx.x & 31) % G;
  g.mask = G == 32 ? 0xffffffffu : (0xffffu << (16 * gi));
  double* scratch = smem + (size_t)(warp * GPW + gi) * (BIG ? (2 * (R::NR + 2) + R::NR * R::NR) : 0);
  uint32_t cnt[C_NUM];
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const unsigned long long nlist = *ccount;
  while (true) {
    unsigned long long li = 0;
    if (g.lane == 0) li = atomicAdd(next, 1ull);
    li = g.bcast(li, 0);
    if (li >= nlist) break;
    const uint64_t r = clist[li];
    double* rec = recs + r * R::STRIDE;
    const bool ok = rec[H_OK] != 0.0;
    const int n = (int)rec[H_N];
    uint32_t flags = (uint32_t)rec[H_FLAGS];
    int nv = 0;
    if (ok) {
      if (BIG) cnt[C_BIG_SCAN]++;
      const int da = (int)rec[H_DA], db = (int)rec[H_DB];
      const double* AT = rec + R::AT;
      const double* BT = rec + R::BT;
      // algorithmic FLOPs (kFLOP units): coefficient phase (dense products of the Eq. 13-23 chain,
      // RR 17k, RT 40k, TR 150k, TT 400k) + per determinant evaluation: slices 2 (sum of the
      // a_i, b_i lengths, i <= n) + Chionh 3 n^2 + GE (2/3) n^3
      const double build_f = (!V1T && !V2T) ? 17e3 : (!V1T ? 40e3 : (!V2T ? 150e3 : 400e3));
      const int tb = (int)rec[H_TB];  // b's total degree after the cut (reading R29): row l has tb - l + 1 terms
      double slice_terms = 0;
      for (int i = 0; i <= n; ++i)
        slice_terms += (i <= da ? D::DA - i + 1 : 0) + (i <= db && i <= tb ? tb - i + 1 : 0);
      const double nn = (double)n;
      const double eval_f = 2.0 * slice_terms + 3.0 * nn * nn + (2.0 / 3.0) * nn * nn * nn;
      double kflop_acc = build_f;
      auto det = [&](double v, double* lg) -> int {
        kflop_acc += eval_f;
        if (BIG) return wdet_sign_smem<G, R::NR>(g, AT, D::DA, BT, tb, n, v, lg, scratch, scratch + 2 * (n + 2));
        return wdet_T<G, R::NR, NC>(g, AT, D::DA, BT, tb, n, v, lg);
      };
      const int P = prm.pieces;
      // reading R25: only the pieces that overlap the v-range of T_1's surviving cull cells, +1 piece each side
      // (a chain elsewhere is excluded by the sound cull predicate); samples j in [jlo, jhi] on the same grid
      int jlo = 0, jhi = P;
      if (vrange) {
        const uint32_t lo = vrange[2 * (p0 + r)], hi = vrange[2 * (p0 + r) + 1];
        jlo = max(0, (int)((lo * (uint32_t)P) / 32u) - 1);
        jhi = min(P, (int)((hi * (uint32_t)P + 31u) / 32u) + 1);
        if (jhi < jlo) jhi = jlo;
      }
      int nprobe = 0;
      double lg_prev = -INFINITY, lg_cur;
      int s_cur = det((double)jlo / P, &lg_cur);
      for (int j = jlo; j <= jhi; ++j) {
        int s_next = 0;
        double lg_next = -INFINITY;
        if (j < jhi) s_next = det((double)(j + 1) / P, &lg_next);
        // c14: |det(v_j)| < 1e-9 max(neighbours), a root within ~1e-11 of the sample: a near-tangency condition the
        // path kernel probes (stored as v_j + 2 among the v-roots; reading R11); one that does not fit flags
        const double nb = fmax(lg_prev, lg_next);
        if (lg_cur < log(1e-9) + nb) {
          if (nv < kMaxV2) {
            if (g.lane == 0) rec[R::VR + nv] = 2.0 + (double)j / P;
            nv++;
            nprobe++;
          } else {
            flags |= SPOLY_FLAG_NEAR_TANGENT;
          }
        }
        if (s_cur == 0) {
          if (nv < kMaxV2) {
            if (g.lane == 0) rec[R::VR + nv] = (double)j / P;
            nv++;
          } else {
            flags |= SPOLY_FLAG_TRUNCATED;
            cnt[C_TRUNCATED]++;
          }
        } else if (j < jhi && s_next != 0 && s_next != s_cur) {
          double lo = (double)j / P, hi = (double)(j + 1) / P;
          for (int it = 0; it < prm.scan_bisect_iters; ++it) {
            const double m = 0.5 * (lo + hi);
            double l2;
            const int sm = det(m, &l2);
            if (sm == 0) {
              lo = hi = m;
              break;
            }
            if (sm == s_cur)
              lo = m;
            else
              hi = m;
          }
          if (nv < kMaxV2) {
            if (g.lane == 0) rec[R::VR + nv] = 0.5 * (lo + hi);
            nv++;
          } else {
            flags |= SPOLY_FLAG_TRUNCATED;
            cnt[C_TRUNCATED]++;
          }
        }
        lg_prev = lg_cur;
        s_cur = s_next;
        lg_cur = lg_next;
      }
      cnt[C_KFLOP] += (uint32_t)(kflop_acc * 1e-3);
      cnt[C_VROOTS] += nv - nprobe;
    }
    if (g.lane == 0) {
      rec[H_NV] = nv;
      if (flags) emit_flags(S, p0 + r, flags);
      if (nv) {
        const unsigned long long k = atomicAdd(pcount, 1ull);
        plist[k] = (uint32_t)r;
      }
    }
    g.sync();
  }
  group_counters(g, cnt, S);
}

// ---- kernel 2 (multi-sample form, orders <= 16): one system per warp, D = 32 / L determinants at once (wdet_quad).
// The samples j = jlo..jhi are evaluated D at a time and walked in order with exactly the sequential scan's
// decisions (c14 probe, exact zero, sign change), so the v-root list is the same list in the same order.  Each
// sign-changing piece is then bisected by multisection: the 2^m - 1 nested midpoints of the bracket (m <= log2 D
// levels per round, the values sequential bisection would compute along any path) are evaluated at once and the
// bisection path is walked through their signs: the same final bracket as 10 sequential bisections.
template <int NC>
struct QuadCfg {
  static constexpr int L = NC <= 8 ? 2 : 4;
  static constexpr int D = 32 / L;
  static constexpr int LV = D >= 8 ? 3 : (D >= 4 ? 2 : 1);  // bisection levels per multisection round
};
template <bool V1T, bool V2T, int NC>
__global__ void __launch_bounds__(kScanWarps * 32, 2) k2_scan_q(uint64_t p0, uint64_t np, SolveParams prm,
                                                               const uint32_t* __restrict__ vrange,
                                                               double* __restrict__ recs, SolSink S,
                                                               const uint32_t* __restrict__ clist,
                                                               const unsigned long long* __restrict__ ccount,
                                                               uint32_t* __restrict__ plist,
                                                               unsigned long long* __restrict__ pcount,
                                                               unsigned long long* __restrict__ next) {
  using D2 = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  using Q = QuadCfg<NC>;
  constexpr int L = Q::L, ND = Q::D;
  __shared__ uint32_t pend_s[kScanWarps][kMaxV2];  // pending bisections: j (16) | slot (8) | sign (1)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane / L;
  uint32_t* pend = pend_s[warp];
  uint32_t cnt[C_NUM];
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const unsigned long long nlist = *ccount;
  const double P = (double)prm.pieces;
  while (true) {
    unsigned long long li = 0;
    if (lane == 0) li = atomicAdd(next, 1ull);
    li = __shfl_sync(0xffffffffu, li, 0);
    if (li >= nlist) break;
    const uint64_t r = clist[li];
    double* rec = recs + r * R::STRIDE;
    const bool ok = rec[H_OK] != 0.0;
    const int n = (int)rec[H_N];
    uint32_t flags = (uint32_t)rec[H_FLAGS];
    int nv = 0;
    if (ok) {
      const int da = (int)rec[H_DA], db = (int)rec[H_DB];
      const double* AT = rec + R::AT;
      const double* BT = rec + R::BT;
      const double build_f = (!V1T && !V2T) ? 17e3 : (!V1T ? 40e3 : (!V2T ? 150e3 : 400e3));
      const int tb = (int)rec[H_TB];
      double slice_terms = 0;
      for (int i = 0; i <= n; ++i)
        slice_terms += (i <= da ? D2::DA - i + 1 : 0) + (i <= db && i <= tb ? tb - i + 1 : 0);
      const double nn = (double)n;
      const double eval_f = 2.0 * slice_terms + 3.0 * nn * nn + (2.0 / 3.0) * nn * nn * nn;
      int ndet = 0;  // determinant evaluations of the sequential algorithm (FLOP model)
      const int Pi = prm.pieces;
      int jlo = 0, jhi = Pi;
      if (vrange) {
        const uint32_t lo = vrange[2 * (p0 + r)], hi = vrange[2 * (p0 + r) + 1];
        jlo = max(0, (int)((lo * (uint32_t)Pi) / 32u) - 1);
        jhi = min(Pi, (int)((hi * (uint32_t)Pi + 31u) / 32u) + 1);
        if (jhi < jlo) jhi = jlo;
      }
      int nprobe = 0, npend = 0;
      // walk state: sample jc (pending its successor), its sign / log|det|, and the predecessor's log|det|
      int jc = jlo - 1, s_cur = 0;
      double lg_cur = -INFINITY, lg_prev = -INFINITY;
      auto visit = [&](int j, int s_next, double lg_next) {  // decisions of sample j (uniform over the warp)
        const double nb = fmax(lg_prev, lg_next);
        if (lg_cur < log(1e-9) + nb) {
          if (nv < kMaxV2) {
            if (lane == 0) rec[R::VR + nv] = 2.0 + (double)j / P;
            nv++;
            nprobe++;
          } else {
            flags |= SPOLY_FLAG_NEAR_TANGENT;
          }
        }
        if (s_cur == 0) {
          if (nv < kMaxV2) {
            if (lane == 0) rec[R::VR + nv] = (double)j / P;
            nv++;
          } else {
            flags |= SPOLY_FLAG_TRUNCATED;
            cnt[C_TRUNCATED]++;
          }
        } else if (j < jhi && s_next != 0 && s_next != s_cur) {
          if (nv < kMaxV2) {
            if (lane == 0) pend[npend] = ((uint32_t)j << 16) | ((uint32_t)nv << 1) | (s_cur > 0 ? 1u : 0u);
            npend++;
            nv++;
          } else {
            flags |= SPOLY_FLAG_TRUNCATED;
            cnt[C_TRUNCATED]++;
          }
        }
      };
      for (int base = jlo; base <= jhi; base += ND) {
        const int j = min(base + q, jhi);
        double lgq;
        const int sq = wdet_quad<L, NC, R::NR>(AT, D2::DA, BT, tb, n, (double)j / P, &lgq);
#pragma unroll
        for (int k = 0; k < ND; ++k) {
          if (base + k > jhi) break;
          const int sk = __shfl_sync(0xffffffffu, sq, L * k);
          const double lk = __shfl_sync(0xffffffffu, lgq, L * k);
          ndet++;
          if (jc >= jlo) visit(jc, sk, lk);
          lg_prev = lg_cur;
          s_cur = sk;
          lg_cur = lk;
          jc = base + k;
        }
      }
      visit(jc, 0, -INFINITY);  // the last sample (jc == jhi): no successor
      __syncwarp();
      // multisection of the pending sign changes (sequential order of discovery)
      for (int b = 0; b < npend; ++b) {
        const uint32_t e = pend[b];
        const int j = (int)(e >> 16), slot = (int)((e >> 1) & 255u), sc = (e & 1u) ? 1 : -1;
        double lo = (double)j / P, hi = (double)(j + 1) / P;
        bool hit = false;
        for (int it = 0; it < prm.scan_bisect_iters && !hit;) {
          const int lv = min(Q::LV, prm.scan_bisect_iters - it);
          const int M = 1 << lv;  // bracket cut into M parts: points 1..M-1
          // nested midpoints X[0..M] (X[0] = lo, X[M] = hi), as sequential bisection computes them
          double X[9];
          X[0] = lo;
          X[M] = hi;
#pragma unroll
          for (int st = 8; st >= 2; st >>= 1) {
            const int h = st * M / 8;
            if (h < 2) continue;
            for (int a = 0; a + h <= M; a += h) X[a + h / 2] = 0.5 * (X[a] + X[a + h]);
          }
          const int pi = 1 + (q % (M - 1));  // quads beyond M - 1 repeat a point (results unused)
          double lgm;
          const int sm_q = wdet_quad<L, NC, R::NR>(AT, D2::DA, BT, tb, n, X[pi], &lgm);
          int sg[9];
#pragma unroll
          for (int k = 1; k < 8; ++k) sg[k] = __shfl_sync(0xffffffffu, sm_q, L * ((k - 1) % ND));
          // the bisection path through the evaluated points (quad k - 1 evaluated point k)
          int a = 0, c = M;
          for (int l = 0; l < lv; ++l) {
            const int m = (a + c) >> 1;
            int sv = 0;
#pragma unroll
            for (int k = 1; k < 8; ++k)
              if (k == m) sv = sg[k];
            ndet++;
            it++;
            if (sv == 0) {
              lo = hi = X[m];
              hit = true;
              break;
            }
            if (sv == sc)
              a = m;
            else
              c = m;
          }
          if (!hit) {
            lo = X[a];
            hi = X[c];
          }
        }
        if (lane == 0) rec[R::VR + slot] = 0.5 * (lo + hi);
      }
      cnt[C_KFLOP] += (uint32_t)((build_f + ndet * eval_f) * 1e-3);
      cnt[C_VROOTS] += nv - nprobe;
    }
    if (lane == 0) {
      rec[H_NV] = nv;
      if (flags) emit_flags(S, p0 + r, flags);
      if (nv) {
        const unsigned long long k = atomicAdd(pcount, 1ull);
        plist[k] = (uint32_t)r;
      }
    }
    __syncwarp();
  }
  Grp<32> g;
  g.lane = lane;
  g.mask = 0xffffffffu;
  group_counters(g, cnt, S);
}

// back-substitution (c11): u-roots of a(., v) -- b(., v) when a(., v) == 0 -- on [-0.1, 1.1]; a
// quadratic with |disc| <= 1e-8 scale reports its double root in *udouble (a c14 condition, probed), else NaN
template <bool V1T, bool V2T>
__device__ int k2_back_sub(const double* AT, const double* BT, int da, int db, double vs, double* us, double* udouble,
                           uint32_t* flags) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  constexpr int NA = D::DB + 1;
  *udouble = __longlong_as_double(0x7ff8000000000000ll);
  double Acoef[NA];
  int dA = da;
  double amax = 0;
  for (int i = 0; i <= dA; ++i) {
    Acoef[i] = rowT<R::NR>(AT, D::DA, i, vs);
    amax = fmax(amax, fabs(Acoef[i]));
  }
  if (!(amax >= 1e-12)) {
    dA = db;
    amax = 0;
    for (int i = 0; i <= dA; ++i) {
      Acoef[i] = rowT<R::NR>(BT, D::DB, i, vs);
      amax = fmax(amax, fabs(Acoef[i]));
    }
    if (!(amax >= 1e-12)) {
      *flags |= SPOLY_FLAG_DEGENERATE;
      return 0;
    }
  }
  while (dA > 0 && Acoef[dA] == 0.0) --dA;
  int nu = 0;
  if (dA == 1) {
    us[nu++] = -Acoef[0] / Acoef[1];
  } else if (dA == 2) {
    const double a0 = Acoef[0], a1 = Acoef[1], a2 = Acoef[2];
    double disc = a1 * a1 - 4 * a2 * a0;
    const double sc = a1 * a1 + 4 * fabs(a2 * a0);
    if (fabs(disc) <= 1e-8 * sc) *udouble = -a1 / (2 * a2);
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
    for (int i = 0; i < Ru.n; ++i)
      if (nu == 0 || Ru.x[i] - us[nu - 1] >= 1e-7) us[nu++] = Ru.x[i];  // Ru.n <= dA < NA
  }
  return nu;
}

// c13 polish: <= iters Newton steps on the exact shooting residual (central differences, h = 1e-7),
// a step kept only if |G| decreases; Jm receives the last Jacobian (zero if none was formed)
__device__ bool polish2(const Chain2& C, int iters, d3 f1, d3 f2, double& uu, double& vv, double& uu2, double& vv2,
                        double Jm[4]) {
  double Gs[2];
  Jm[0] = Jm[1] = Jm[2] = Jm[3] = 0.0;
  const bool okp = shoot2(C, uu, vv, f1, f2, Gs, &uu2, &vv2);
  for (int it = 0; okp && it < iters; ++it) {
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
    const double du = -(Jm[3] * Gs[0] - Jm[1] * Gs[1]) / det;
    const double dv = -(-Jm[2] * Gs[0] + Jm[0] * Gs[1]) / det;
    double Gn[2], nu2, nv2;
    if (!shoot2(C, uu + du, vv + dv, f1, f2, Gn, &nu2, &nv2)) break;
    if (!(hypot(Gn[0], Gn[1]) < hypot(Gs[0], Gs[1]))) break;
    uu += du;
    vv += dv;
    Gs[0] = Gn[0];
    Gs[1] = Gn[1];
    uu2 = nu2;
    vv2 = nv2;
  }
  return okp;
}

__device__ __forceinline__ bool in_tri(double u, double v, double e) { return u >= -e && v >= -e && u + v <= 1 + e; }

// c14 probe (reading R11): does the near-tangency condition at (u1, v1) sit at an (almost) admissible chain?  Within
// kProbeDomain of both triangles, polished (moving at most kProbeMove), still within kProbeDomain, residual below
// theta_final.  Ghost double roots of the square form fail it and raise no flag.
constexpr double kProbeDomain2 = 1e-3, kProbeMove = 1e-2;
__device__ bool probe2(const Chain2& C, const SolveParams& prm, const WP& Up, const WP& Vp, const WP& Kp, bool relabel,
                       double u1, double v1) {
  const double kap = wp_eval(Kp, u1, v1);
  double u2 = wp_eval(Up, u1, v1) / kap, v2 = wp_eval(Vp, u1, v1) / kap;
  if (!(fabs(kap) > 0) || !isfinite(u2) || !isfinite(v2)) return false;
  if (relabel) {
    const double t = u2;
    u2 = v2;
    v2 = t;
  }
  if (!in_tri(u1, v1, kProbeDomain2) || !in_tri(u2, v2, kProbeDomain2)) return false;
  d3 f1, f2;
  frame_of(normalize(C.x3 - C.T2.X(u2, v2)), &f1, &f2);
  double uu = u1, vv = v1, uu2 = u2, vv2 = v2, Jm[4];
  if (!polish2(C, prm.polish_iters, f1, f2, uu, vv, uu2, vv2, Jm)) return false;
  if (fmax(fabs(uu - u1), fabs(vv - v1)) > kProbeMove) return false;
  if (!in_tri(uu, vv, kProbeDomain2) || !in_tri(uu2, vv2, kProbeDomain2)) return false;
  const d3 x1 = C.T1.X(uu, vv), x2 = C.T2.X(uu2, vv2);
  const double r1 = resid(C.x0, x1, x2, C.T1.N(uu, vv), C.eta[0], C.eta[1]);
  const double r2 = resid(x1, x2, C.x3, C.T2.N(uu2, vv2), C.eta[1], C.eta[2]);
  return fmax(r1, r2) < prm.theta_final;
}

// ---- kernel 3: path phase (thread per pair with v-roots): back-substitution, polish, validation,
// contribution, emission (slot = processing order within the pair, deterministic after the sort)
template <bool V1T, bool V2T>
__global__ void __launch_bounds__(128) k2_path(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                               uint64_t p0, const TriRec* __restrict__ tris,
                                               const double* __restrict__ ep, const double* __restrict__ inten,
                                               SolveParams prm, const double* __restrict__ recs, SolSink S,
                                               const uint32_t* __restrict__ plist,
                                               const unsigned long long* __restrict__ pcount) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  uint32_t cnt[C_NUM];
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const unsigned long long total = *pcount;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = plist[t];
    const uint64_t pi = p0 + r;
    const double* rec = recs + r * R::STRIDE;
    const uint32_t q = pq[pi];
    Chain2 C;
    load_chain(tris, pt, ep, q, pi, C);
    C.r1 = V1T;
    C.r2 = V2T;
    C.eta[0] = rec[H_ETA0];
    C.eta[1] = rec[H_ETA1];
    C.eta[2] = rec[H_ETA2];
    const bool relabel = rec[H_RELABEL] != 0.0;
    const int da = (int)rec[H_DA], db = (int)rec[H_DB], nv = (int)rec[H_NV];
    const double* AT = rec + R::AT;
    const double* BT = rec + R::BT;
    const WP Up{const_cast<double*>(rec + R::U), D::DU}, Vp{const_cast<double*>(rec + R::V), D::DU},
        Kp{const_cast<double*>(rec + R::K), D::DK};
    uint32_t flags = 0;
    bool tangent = false;  // a probed c14 condition sits at an admissible chain (NEAR_TANGENT, reading R11)
    int nsol = 0;
    double su[kMaxSol2][4], scontrib[kMaxSol2];
    float sres[kMaxSol2];
    constexpr int NA = D::DB + 1;
    for (int iv = 0; iv < nv; ++iv) {
      const double ve = rec[R::VR + iv];
      const bool is_probe = ve >= 2.0;  // a scan sample with |det| ~ 0 (stored as v + 2)
      const double vs = is_probe ? ve - 2.0 : ve;
      double us[NA], ud;
      uint32_t fl = 0;
      const int nu = k2_back_sub<V1T, V2T>(AT, BT, da, db, vs, us, &ud, &fl);
      if (is_probe) {
        for (int iu = 0; iu < nu && !tangent; ++iu) tangent = probe2(C, prm, Up, Vp, Kp, relabel, us[iu], vs);
        continue;
      }
      flags |= fl;
      if (!tangent && !isnan(ud)) tangent = probe2(C, prm, Up, Vp, Kp, relabel, ud, vs);
      for (int iu = 0; iu < nu; ++iu) {
        cnt[C_CANDIDATES]++;
        const double ur = us[iu], vr = vs;
        const double kap = wp_eval(Kp, ur, vr), ut = wp_eval(Up, ur, vr), vt = wp_eval(Vp, ur, vr);
        double u2 = ut / kap, v2 = vt / kap;
        if (!(fabs(kap) > 0) || !isfinite(u2) || !isfinite(v2)) {
          cnt[C_REJ_KAPPA]++;
          continue;
        }
        if (relabel) {
          const double t = u2;
          u2 = v2;
          v2 = t;
        }
        const double dm = 1e-3;
        if (!(in_tri(ur, vr, dm) && in_tri(u2, v2, dm))) {
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
        double uu = ur, vv = vr, uu2 = u2, vv2 = v2, Jm[4];
        if (!polish2(C, prm.polish_iters, f1, f2, uu, vv, uu2, vv2, Jm)) {
          cnt[C_REJ_CONSTRAINT]++;
          continue;
        }
        const double ed = prm.eps_domain;
        if (!(in_tri(uu, vv, ed) && in_tri(uu2, vv2, ed))) {
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
        if (nsol >= kMaxSol2) {  // per-pair capacity: flagged, never silent
          flags |= SPOLY_FLAG_TRUNCATED;
          cnt[C_TRUNCATED]++;
        } else {
          const double J = jacobian2(C, x1, x2);
          const double I = inten ? inten[q] : 1.0;
          su[nsol][0] = uu;
          su[nsol][1] = vv;
          su[nsol][2] = uu2;
          su[nsol][3] = vv2;
          scontrib[nsol] = J > 0 ? I / J : 0.0;
          sres[nsol] = (float)rho;
          nsol++;
          cnt[C_ADMISSIBLE]++;
        }
      }
    }
    if (tangent) flags |= SPOLY_FLAG_NEAR_TANGENT;
    // emission: flag record, then the solutions in processing order (deterministic slot)
    if (flags) {
      const unsigned long long p = atomicAdd(S.count + 1, 1ull);
      if (p < S.fcapacity) {
        S.fkey[p] = pi;
        S.fflags[p] = flags;
      }
    }
    if (nsol) {
      const unsigned long long b = atomicAdd(S.count, (unsigned long long)nsol);
      for (int s = 0; s < nsol; ++s) {
        const unsigned long long p = b + s;
        if (p < S.capacity) {
          S.key[p] = ((unsigned long long)pi << 6) | (unsigned)s;
          for (int c = 0; c < 4; ++c) S.bary[4 * p + c] = su[s][c];
          S.contrib[p] = scontrib[s];
          S.resid[p] = sres[s];
        }
      }
    }
  }
  for (int i = 0; i < C_NUM; ++i) {
    uint32_t v = cnt[i];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(S.counters + i, (unsigned long long)v);
  }
}

template <bool V1T, bool V2T>
static void launch_k2(const uint32_t* pq, const uint32_t* pt, const uint32_t* vr, uint64_t npairs, const DeviceMesh& M,
                      const double* ep,
                      const double* inten, const SolveParams& prm, const SolSink& S, K2Scratch& W, int nsm,
                      cudaStream_t st) {
  using D = Deg2<V1T, V2T>;
  using R = Rec2<V1T, V2T>;
  constexpr int G = D::G;
  const size_t sh_build = (size_t)kBuildWarps * (32 / build_group<V1T, V2T>()) * D::ARENA * sizeof(double);
  const size_t sh_big = (size_t)kScanWarps * (32 / G) * (2 * (R::NR + 2) + R::NR * R::NR) * sizeof(double);
  // the attribute is per device: set it on every launch (cheap; a process-wide "done" flag would skip it on a
  // second context's device, and is not thread-safe)
  cudaFuncSetAttribute(k2_build<V1T, V2T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_build);
  cudaFuncSetAttribute(k2_scan<V1T, V2T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_big);
  int occ_b = 0, occ_s = 0, occ_p = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, k2_build<V1T, V2T>, kBuildWarps * 32, sh_build);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k2_scan<V1T, V2T, nc_of_class<G>(0)>, kScanWarps * 32, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, k2_path<V1T, V2T>, 128, 0);
  occ_b = occ_b < 1 ? 1 : occ_b;
  occ_s = occ_s < 1 ? 1 : occ_s;
  occ_p = occ_p < 1 ? 1 : occ_p;
  const uint64_t chunk = W.rec_cap / R::STRIDE;
  // counters: [0] build fetch, [1] path list count, [8 + c] class counts, [16 + c] class fetch
  unsigned long long* cc = W.ctr + 8;
  unsigned long long* cn = W.ctr + 16;
  for (uint64_t p0 = 0; p0 < npairs; p0 += chunk) {
    const uint64_t np = npairs - p0 < chunk ? npairs - p0 : chunk;
    cudaMemsetAsync(W.ctr, 0, 24 * sizeof(unsigned long long), st);
    const uint64_t gb = (uint64_t)kBuildWarps * (32 / build_group<V1T, V2T>()), gs = (uint64_t)kScanWarps * (32 / G);
    const uint64_t gs16 = (uint64_t)kScanWarps * 2;  // classes of order <= 16 run two systems per warp
    const int bs16 = (int)std::min<uint64_t>((np + gs16 - 1) / gs16, (uint64_t)nsm * occ_s);
    const int bb = (int)std::min<uint64_t>((np + gb - 1) / gb, (uint64_t)nsm * occ_b);
    const int bs = (int)std::min<uint64_t>((np + gs - 1) / gs, (uint64_t)nsm * occ_s);
    const int bp = (int)std::min<uint64_t>((np + 127) / 128, (uint64_t)nsm * occ_p);
    k2_build<V1T, V2T><<<bb, kBuildWarps * 32, sh_build, st>>>(pq, pt, p0, np, M.tris, ep, prm, W.rec, S, W.ctr);
    k2_bin<V1T, V2T><<<(int)std::min<uint64_t>((np + 255) / 256, (uint64_t)nsm * 8), 256, 0, st>>>(np, W.rec, W.clist,
                                                                                                   cc);
    const uint32_t* L = W.clist;
#ifdef SPOLY_SCAN_QUAD
    {  // classes of order <= 16: multi-sample scan, one system per warp (C4: 1.78 -> 2.29 s: the restricted v-ranges
       // (R25) are short, so most of the D parallel samples and the multisection points are wasted)
      const int bq = (int)std::min<uint64_t>((np + kScanWarps - 1) / kScanWarps, (uint64_t)nsm * 4);
      k2_scan_q<V1T, V2T, nc_of_class<G>(0)><<<bq, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L, cc, W.plist, W.ctr + 1, cn);
      k2_scan_q<V1T, V2T, nc_of_class<G>(1)><<<bq, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + np, cc + 1, W.plist, W.ctr + 1, cn + 1);
      if (G == 16)
        k2_scan_q<V1T, V2T, nc_of_class<G>(2)><<<bq, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 2 * np, cc + 2, W.plist, W.ctr + 1, cn + 2);
      else
        k2_scan<V1T, V2T, nc_of_class<G>(2)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 2 * np, cc + 2, W.plist, W.ctr + 1, cn + 2);
      if (G != 16) {
        k2_scan<V1T, V2T, nc_of_class<G>(3)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 3 * np, cc + 3, W.plist, W.ctr + 1, cn + 3);
        k2_scan<V1T, V2T, nc_of_class<G>(4)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 4 * np, cc + 4, W.plist, W.ctr + 1, cn + 4);
        k2_scan<V1T, V2T, nc_of_class<G>(5)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 5 * np, cc + 5, W.plist, W.ctr + 1, cn + 5);
        W.launches += 3;
        if (D::DB > 32) {
          k2_scan<V1T, V2T, 0><<<nsm, kScanWarps * 32, sh_big, st>>>(p0, np, prm, vr, W.rec, S, L + 6 * np, cc + 6, W.plist, W.ctr + 1, cn + 6);
          W.launches += 1;
        }
      }
      W.launches += 3;
    }
#else
    if (G == 16) {
      k2_scan<V1T, V2T, nc_of_class<G>(0)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L, cc, W.plist, W.ctr + 1, cn);
      k2_scan<V1T, V2T, nc_of_class<G>(1)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + np, cc + 1, W.plist, W.ctr + 1, cn + 1);
      k2_scan<V1T, V2T, nc_of_class<G>(2)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 2 * np, cc + 2, W.plist, W.ctr + 1, cn + 2);
      W.launches += 3;
    } else {
      k2_scan<V1T, V2T, nc_of_class<G>(0)><<<bs16, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L, cc, W.plist, W.ctr + 1, cn);
      k2_scan<V1T, V2T, nc_of_class<G>(1)><<<bs16, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + np, cc + 1, W.plist, W.ctr + 1, cn + 1);
      k2_scan<V1T, V2T, nc_of_class<G>(2)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 2 * np, cc + 2, W.plist, W.ctr + 1, cn + 2);
      k2_scan<V1T, V2T, nc_of_class<G>(3)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 3 * np, cc + 3, W.plist, W.ctr + 1, cn + 3);
      k2_scan<V1T, V2T, nc_of_class<G>(4)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 4 * np, cc + 4, W.plist, W.ctr + 1, cn + 4);
      k2_scan<V1T, V2T, nc_of_class<G>(5)><<<bs, kScanWarps * 32, 0, st>>>(p0, np, prm, vr, W.rec, S, L + 5 * np, cc + 5, W.plist, W.ctr + 1, cn + 5);
      W.launches += 6;
      if (D::DB > 32) {
        k2_scan<V1T, V2T, 0><<<nsm, kScanWarps * 32, sh_big, st>>>(p0, np, prm, vr, W.rec, S, L + 6 * np, cc + 6, W.plist, W.ctr + 1, cn + 6);
        W.launches += 1;
      }
    }
#endif
    k2_path<V1T, V2T><<<bp, 128, 0, st>>>(pq, pt, p0, M.tris, ep, inten, prm, W.rec, S, W.plist, W.ctr + 1);
    W.launches += 3;
  }
}

uint64_t k2_record_bytes(int v1t, int v2t) {
  if (v1t && v2t) return Rec2<true, true>::STRIDE * sizeof(double);
  if (v1t) return Rec2<true, false>::STRIDE * sizeof(double);
  if (v2t) return Rec2<false, true>::STRIDE * sizeof(double);
  return Rec2<false, false>::STRIDE * sizeof(double);
}

void launch_solve_k2(int v1t, int v2t, const uint32_t* pq, const uint32_t* pt, const uint32_t* vr, uint64_t npairs,
                     const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                     const SolSink& S, K2Scratch& W, int nsm, cudaStream_t st) {
  if (!npairs) return;

  if (v1t && v2t)
    launch_k2<true, true>(pq, pt, vr, npairs, M, ep, inten, prm, S, W, nsm, st);
  else if (v1t)
    launch_k2<true, false>(pq, pt, vr, npairs, M, ep, inten, prm, S, W, nsm, st);
  else if (v2t)
    launch_k2<false, true>(pq, pt, vr, npairs, M, ep, inten, prm, S, W, nsm, st);
  else
    launch_k2<false, false>(pq, pt, vr, npairs, M, ep, inten, prm, S, W, nsm, st);
#ifdef SPOLY_PROF_BUILD
  unsigned long long h[16];
  cudaStreamSynchronize(st);
  if (cudaMemcpyFromSymbol(h, g_bprof, sizeof(h)) == cudaSuccess) {
    fprintf(stderr, "k2_build section clocks (cumulative, lane 0):");
    for (int i = 0; i < 9; ++i) fprintf(stderr, " %d:%.3e", i, (double)h[i]);
    fprintf(stderr, "\n");
  }
#endif
}

}  // namespace spoly
