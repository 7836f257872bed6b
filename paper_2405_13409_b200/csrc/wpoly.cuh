// Group-cooperative (16 or 32 lanes) dense bivariate polynomial algebra in shared memory, and the
// register-resident determinant of the Bezout matrix (Eq. 24) used by the two-bounce solve.
//
// Storage: a polynomial of degree d is packed row by row in u-degree, c[poff(d, i) + j] = coefficient of
// u^i v^j (i + j <= d), T(d) = (d + 1)(d + 2) / 2 doubles.  Every output coefficient is produced by exactly
// one lane (gather form), so no atomics and a fixed summation order (deterministic).
#pragma once
#include "common.cuh"
#include "poly_dev.cuh"

namespace spoly {

template <int G>
struct Grp {
  int lane;       // 0 .. G-1 within the group
  unsigned mask;  // lanes of the group within the warp
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  template <class T>
  __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(mask, v, src, G); }
  template <class T>
  __device__ __forceinline__ T down(T v, int d) const { return __shfl_down_sync(mask, v, d, G); }
  template <class T>
  __device__ __forceinline__ T xor_(T v, int d) const { return __shfl_xor_sync(mask, v, d, G); }
  __device__ __forceinline__ double max_(double v) const {
    for (int o = G / 2; o; o >>= 1) v = fmax(v, xor_(v, o));
    return v;
  }
  __device__ __forceinline__ int imax(int v) const {
    for (int o = G / 2; o; o >>= 1) v = max(v, xor_(v, o));
    return v;
  }
};

__host__ __device__ constexpr int tri_n(int d) { return (d + 1) * (d + 2) / 2; }
__device__ __forceinline__ int poff(int d, int i) { return i * (2 * d + 3 - i) / 2; }

struct WP {
  double* c;
  int d;
};
struct WV {
  WP x, y, z;
};

// per-group bump allocator over the shared-memory arena (uniform across the group)
struct Arena {
  double* base;
  int top, cap;
  bool overflow;
  __device__ WP poly(int d) {
    WP p{base + top, d};
    top += tri_n(d);
    if (top > cap) {
      overflow = true;
      top = cap - tri_n(d) > 0 ? cap - tri_n(d) : 0;  // keep pointers in bounds; result discarded
      p.c = base + top;
      top += tri_n(d);
    }
    return p;
  }
  __device__ WV vec(int d) { return {poly(d), poly(d), poly(d)}; }
  __device__ double* raw(int n) {
    double* p = base + top;
    top += n;
    if (top > cap) {
      overflow = true;
      top -= n;
      p = base;
    }
    return p;
  }
};

// advance the packed (i, j) position of output degree d by `step` coefficients
__device__ __forceinline__ void padv(int d, int step, int& i, int& j) {
  j += step;
  while (i <= d && j > d - i) {
    j -= d - i + 1;
    ++i;
  }
}

// advance the (row i, chunk start j0) position of output degree d by `step` chunks of W coefficients
template <int W>
__device__ __forceinline__ void tadv(int d, int step, int& i, int& j0) {
  while (step > 0 && i <= d) {
    const int left = (d - i + 1 - j0 + W - 1) / W;  // chunks from j0 to the end of row i
    if (step < left) {
      j0 += step * W;
      step = 0;
    } else {
      step -= left;
      ++i;
      j0 = 0;
    }
  }
}

// inlined at every call site (an out-of-line copy per (G, K), -DSPOLY_WMUL_INLINE="__device__ __noinline__",
// measured 10% slower on C4 despite ncu's instruction-fetch stalls)
#ifndef SPOLY_WMUL_W
#define SPOLY_WMUL_W 8  // output coefficients per lane chunk (A/B: 4)
#endif
#ifndef SPOLY_WMUL_SMALL_DC
#define SPOLY_WMUL_SMALL_DC 12  // 4-wide chunks below this output degree; A/B on C4: none 1.81 s, 12 1.73 s, 20 1.74 s
#endif
#ifndef SPOLY_WMUL_INLINE
#define SPOLY_WMUL_INLINE __device__ __forceinline__
#endif
// c = sum_k s_k a_k b_k  (+ c if acc); every product term with i + j <= c.d is produced.
// Register-windowed gather (W = 8): a lane owns W consecutive coefficients (i, j0..j0+W-1) of one output row; for
// every operand row pair (p, i - p) it walks q once, so each a coefficient is loaded once for the W outputs
// and the b operands slide through a W-register window (one new load per step): 2 shared-memory loads per W
// FMAs instead of 2 per FMA.  Out-of-row b positions read as 0 (predicated), so the W outputs may share the
// union of their q ranges.
template <int K, int W>
SPOLY_WMUL_INLINE void wmul_core(int lane, int stride, WP c, const WP (&a)[K], const WP (&b)[K], const double (&s)[K],
                                 bool acc) {
  const int dc = c.d;
  int i = 0, j0 = 0;
  tadv<W>(dc, lane, i, j0);
  while (i <= dc) {
    const int rowlen = dc - i + 1;
    double* cp = c.c + poff(dc, i);
    double out[W];
#pragma unroll
    for (int k = 0; k < W; ++k) out[k] = (acc && j0 + k < rowlen) ? cp[j0 + k] : 0.0;
#pragma unroll  // (rolled, the operand descriptors go to local memory: C4 build +8%)
    for (int kk = 0; kk < K; ++kk) {
      const int da = a[kk].d, db = b[kk].d;
      double t[W];
#pragma unroll
      for (int k = 0; k < W; ++k) t[k] = 0.0;
      const int p0 = max(0, i - db), p1 = min(i, da);
      for (int p = p0; p <= p1; ++p) {
        const int blen = db - (i - p);  // b row i - p holds indices 0..blen
        const double* ap = a[kk].c + poff(da, p);
        const double* bp = b[kk].c + poff(db, i - p);
        const int qlo = max(0, j0 - blen), qhi = min(j0 + W - 1, da - p);
        if (qlo > qhi) continue;
#ifndef SPOLY_WMUL_SLIDE
        // register-blocked: 8 a coefficients x 15 b coefficients -> 64 FMAs per block of q, all register
        // indices static (no sliding-window moves); positions outside a row read as 0
        for (int qb = qlo; qb <= qhi; qb += W) {
          double av[W], bw[2 * W - 1];
#pragma unroll
          for (int m = 0; m < W; ++m) av[m] = (qb + m <= qhi) ? ap[qb + m] : 0.0;
#pragma unroll
          for (int r = 0; r < 2 * W - 1; ++r) {
            const int jb = j0 - qb - (W - 1) + r;
            bw[r] = ((unsigned)jb <= (unsigned)blen) ? bp[jb] : 0.0;
          }
#pragma unroll
          for (int m = 0; m < W; ++m)
#pragma unroll
            for (int k = 0; k < W; ++k) t[k] = fma(av[m], bw[k - m + W - 1], t[k]);
        }
#else
        double w[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const int jb = j0 + k - qlo;
          w[k] = (jb >= 0 && jb <= blen) ? bp[jb] : 0.0;
        }
        for (int q = qlo; q <= qhi; ++q) {
          const double av = ap[q];
#pragma unroll
          for (int k = 0; k < W; ++k) t[k] = fma(av, w[k], t[k]);
#pragma unroll
          for (int k = W - 1; k > 0; --k) w[k] = w[k - 1];
          const int jb = j0 - q - 1;  // <= blen - 1 because q >= qlo >= j0 - blen
          w[0] = jb >= 0 ? bp[jb] : 0.0;
        }
#endif
      }
#pragma unroll
      for (int k = 0; k < W; ++k) out[k] = fma(s[kk], t[k], out[k]);
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (j0 + k < rowlen) cp[j0 + k] = out[k];
    tadv<W>(dc, stride, i, j0);
  }
}
template <int G, int K, int W>
__device__ __forceinline__ void wmul_w(const Grp<G>& g, WP c, const WP (&a)[K], const WP (&b)[K], const double (&s)[K],
                                       bool acc) {
  wmul_core<K, W>(g.lane, G, c, a, b, s, acc);
  g.sync();
}
// outputs with few coefficients use 4-wide chunks, so more lanes get one (the build's small products left most of
// the group idle with 8-wide chunks); the large products keep 8-wide register blocks
template <int G, int K>
__device__ __forceinline__ void wmul(const Grp<G>& g, WP c, const WP (&a)[K], const WP (&b)[K], const double (&s)[K],
                                     bool acc) {
#if SPOLY_WMUL_SMALL_DC > 0
  if (c.d < SPOLY_WMUL_SMALL_DC) {
    wmul_w<G, K, 4>(g, c, a, b, s, acc);
    return;
  }
#endif
  wmul_w<G, K, SPOLY_WMUL_W>(g, c, a, b, s, acc);
}
// NB independent products at once, G / NB lanes each (lane l works on product l / (G / NB)): the build's medium
// products have fewer 8-wide output chunks than lanes, and NB of them side by side fill the group with one sync.
// A product with c.d < 0 is a placeholder (no chunks).  Each output chunk is still computed once by the same
// arithmetic as wmul's.
__device__ __forceinline__ WP sel_wp(bool p, WP x, WP y) {
  WP r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %2, 0;\n\tselp.b64 %0, %3, %4, q;\n\tselp.b32 %1, %5, %6, q;\n\t}"
      : "=l"(r.c), "=r"(r.d) : "r"((int)p), "l"(x.c), "l"(y.c), "r"(x.d), "r"(y.d));
  return r;
}
__device__ __forceinline__ double sel_d(bool p, double x, double y) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\tselp.f64 %0, %2, %3, q;\n\t}" : "=d"(r) : "r"((int)p), "d"(x), "d"(y));
  return r;
}
template <int G, int K, int NB>
__device__ __forceinline__ void wmul_batch(const Grp<G>& g, const WP (&c)[NB], const WP (&a)[NB][K],
                                           const WP (&b)[NB][K], const double (&s)[NB][K], bool acc) {
  constexpr int SG = G / NB;
  const int job = g.lane / SG;
  WP cc = c[0], aa[K], bb[K];
  double ss[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    aa[k] = a[0][k];
    bb[k] = b[0][k];
    ss[k] = s[0][k];
  }
#pragma unroll
  for (int q = 1; q < NB; ++q) {
    const bool m = job == q;
    cc = sel_wp(m, c[q], cc);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      aa[k] = sel_wp(m, a[q][k], aa[k]);
      bb[k] = sel_wp(m, b[q][k], bb[k]);
      ss[k] = sel_d(m, s[q][k], ss[k]);
    }
  }
#if SPOLY_WMUL_SMALL_DC > 0
  if (c[0].d < SPOLY_WMUL_SMALL_DC)
    wmul_core<K, 4>(g.lane % SG, SG, cc, aa, bb, ss, acc);
  else
#endif
    wmul_core<K, SPOLY_WMUL_W>(g.lane % SG, SG, cc, aa, bb, ss, acc);
  g.sync();
}
template <int G>
__device__ __forceinline__ void wmul1x3(const Grp<G>& g, const WV& R, const WV& A, const WV& B, double s0, bool acc) {
  const WP none{R.x.c, -1};
  const WP c[4] = {R.x, R.y, R.z, none};
  const WP a[4][1] = {{A.x}, {A.y}, {A.z}, {A.x}};
  const WP b[4][1] = {{B.x}, {B.y}, {B.z}, {B.x}};
  const double s[4][1] = {{s0}, {s0}, {s0}, {s0}};
  wmul_batch<G, 1, 4>(g, c, a, b, s, acc);
}
// three (or four) dot products c_q = s_q A_q . B_q side by side
template <int G>
__device__ __forceinline__ void wdot4(const Grp<G>& g, WP c0, const WV& A0, const WV& B0, WP c1, const WV& A1, const WV& B1,
                                      WP c2, const WV& A2, const WV& B2, WP c3, const WV& A3, const WV& B3) {
  const WP c[4] = {c0, c1, c2, c3};
  const WP a[4][3] = {{A0.x, A0.y, A0.z}, {A1.x, A1.y, A1.z}, {A2.x, A2.y, A2.z}, {A3.x, A3.y, A3.z}};
  const WP b[4][3] = {{B0.x, B0.y, B0.z}, {B1.x, B1.y, B1.z}, {B2.x, B2.y, B2.z}, {B3.x, B3.y, B3.z}};
  const double s[4][3] = {{1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {1, 1, 1}};
  wmul_batch<G, 3, 4>(g, c, a, b, s, false);
}
// the three components of sum_k s_k a_k(x) b_k(x) (x = x, y, z) side by side: R.x = s0 a0.x b0.x + s1 a1.x b1.x etc.
// with per-component operands given as WVs (a WP repeated in all three for a scalar factor)
template <int G>
__device__ __forceinline__ void wmul2x3(const Grp<G>& g, const WV& R, const WV& A0, const WV& B0, double s0,
                                        const WV& A1, const WV& B1, double s1, bool acc) {
  const WP none{R.x.c, -1};
  const WP c[4] = {R.x, R.y, R.z, none};
  const WP a[4][2] = {{A0.x, A1.x}, {A0.y, A1.y}, {A0.z, A1.z}, {A0.x, A1.x}};
  const WP b[4][2] = {{B0.x, B1.x}, {B0.y, B1.y}, {B0.z, B1.z}, {B0.x, B1.x}};
  const double s[4][2] = {{s0, s1}, {s0, s1}, {s0, s1}, {s0, s1}};
  wmul_batch<G, 2, 4>(g, c, a, b, s, acc);
}
__device__ __forceinline__ WV wv_rep(WP p) { return {p, p, p}; }

template <int G>
__device__ __forceinline__ void wmul1(const Grp<G>& g, WP c, WP a, WP b, double s, bool acc) {
  const WP A[1] = {a}, B[1] = {b};
  const double Sc[1] = {s};
  wmul<G, 1>(g, c, A, B, Sc, acc);
}
template <int G>
__device__ __forceinline__ void wmul2(const Grp<G>& g, WP c, WP a0, WP b0, double s0, WP a1, WP b1, double s1,
                                      bool acc) {
  const WP A[2] = {a0, a1}, B[2] = {b0, b1};
  const double Sc[2] = {s0, s1};
  wmul<G, 2>(g, c, A, B, Sc, acc);
}
// c (+)= s (A . B)
template <int G>
__device__ __forceinline__ void wdot(const Grp<G>& g, WP c, const WV& A, const WV& B, double s, bool acc) {
  const WP a[3] = {A.x, A.y, A.z}, b[3] = {B.x, B.y, B.z};
  const double Sc[3] = {s, s, s};
  wmul<G, 3>(g, c, a, b, Sc, acc);
}

// c = sum_k s_k a_k (+ c if acc), a_k of degree <= anything (terms beyond c.d dropped)
template <int G, int K>
__device__ void wlin(const Grp<G>& g, WP c, const WP (&a)[K], const double (&s)[K], bool acc) {
  const int dc = c.d, n = tri_n(dc);
  int i = 0, j = 0;
  padv(dc, g.lane, i, j);
  for (int idx = g.lane; idx < n; idx += G) {
    double sum = acc ? c.c[idx] : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (i + j <= a[k].d) sum = fma(s[k], a[k].c[poff(a[k].d, i) + j], sum);
    c.c[idx] = sum;
    padv(dc, G, i, j);
  }
  g.sync();
}
template <int G>
__device__ __forceinline__ void wlin1(const Grp<G>& g, WP c, WP a, double s, bool acc) {
  const WP A[1] = {a};
  const double Sc[1] = {s};
  wlin<G, 1>(g, c, A, Sc, acc);
}
template <int G>
__device__ __forceinline__ void wlin2(const Grp<G>& g, WP c, WP a0, double s0, WP a1, double s1, bool acc) {
  const WP A[2] = {a0, a1};
  const double Sc[2] = {s0, s1};
  wlin<G, 2>(g, c, A, Sc, acc);
}
template <int G>
__device__ __forceinline__ void wlin3(const Grp<G>& g, WP c, WP a0, double s0, WP a1, double s1, WP a2, double s2,
                                      bool acc) {
  const WP A[3] = {a0, a1, a2};
  const double Sc[3] = {s0, s1, s2};
  wlin<G, 3>(g, c, A, Sc, acc);
}
// c.c[0] += x
template <int G>
__device__ __forceinline__ void wadd0(const Grp<G>& g, WP c, double x) {
  if (g.lane == 0) c.c[0] += x;
  g.sync();
}
// linear polynomial c0 + cu u + cv v
template <int G>
__device__ __forceinline__ void wlinear(const Grp<G>& g, WP c, double c0, double cu, double cv) {
  if (g.lane == 0) {
    c.c[0] = c0;  // (0, 0)
    c.c[1] = cv;  // (0, 1)
    c.c[2] = cu;  // (1, 0)
  }
  g.sync();
}
template <int G>
__device__ __forceinline__ void wlinear3(const Grp<G>& g, WV& V, d3 c0, d3 cu, d3 cv) {
  if (g.lane == 0) {
    V.x.c[0] = c0.x; V.x.c[1] = cv.x; V.x.c[2] = cu.x;
    V.y.c[0] = c0.y; V.y.c[1] = cv.y; V.y.c[2] = cu.y;
    V.z.c[0] = c0.z; V.z.c[1] = cv.z; V.z.c[2] = cu.z;
  }
  g.sync();
}
// R = A x b for a constant vector b
template <int G>
__device__ __forceinline__ void wcross_c(const Grp<G>& g, const WV& R, const WV& A, d3 b) {
  wlin2(g, R.x, A.y, b.z, A.z, -b.y, false);
  wlin2(g, R.y, A.z, b.x, A.x, -b.z, false);
  wlin2(g, R.z, A.x, b.y, A.y, -b.x, false);
}
// R = A x B
template <int G>
__device__ __forceinline__ void wcross(const Grp<G>& g, const WV& R, const WV& A, const WV& B) {
  wmul2(g, R.x, A.y, B.z, 1.0, A.z, B.y, -1.0, false);
  wmul2(g, R.y, A.z, B.x, 1.0, A.x, B.z, -1.0, false);
  wmul2(g, R.z, A.x, B.y, 1.0, A.y, B.x, -1.0, false);
}

// move a polynomial to a lower address of the arena (ascending chunks: safe for overlapping ranges)
template <int G>
__device__ void wmove(const Grp<G>& g, WP& p, double* dst) {
  const int n = tri_n(p.d);
  if (dst == p.c) return;
  for (int b0 = 0; b0 < n; b0 += G) {
    const int i = b0 + g.lane;
    const double v = i < n ? p.c[i] : 0.0;
    g.sync();
    if (i < n) dst[i] = v;
    g.sync();
  }
  p.c = dst;
}
template <int G>
__device__ __forceinline__ double* wmovev(const Grp<G>& g, WV& V, double* dst) {
  wmove(g, V.x, dst);
  dst += tri_n(V.x.d);
  wmove(g, V.y, dst);
  dst += tri_n(V.y.d);
  wmove(g, V.z, dst);
  return dst + tri_n(V.z.d);
}

// ------------------------------------------------------------------ total-degree mass bounds (reading R29)
// m[s] = sum_{i+j=s} |c_ij|, s = 0..p.d (lane s; a sum of products obeys m_{ab}[s] <= sum m_a[s1] m_b[s - s1])
template <int G>
__device__ __forceinline__ void wmass(const Grp<G>& g, const WP& p, double* m) {
  for (int s = g.lane; s <= p.d; s += G) {
    double t = 0.0;
    for (int i = 0; i <= s; ++i) t += fabs(p.c[poff(p.d, i) + s - i]);
    m[s] = t;
  }
  g.sync();
}
// out[s] = sum_{s1} x[s1] y[s - s1], s = 0..nx + ny (upper bound of the product's masses)
template <int G>
__device__ __forceinline__ void mconv(const Grp<G>& g, double* out, const double* x, int nx, const double* y, int ny) {
  for (int s = g.lane; s <= nx + ny; s += G) {
    double t = 0.0;
    for (int s1 = max(0, s - ny); s1 <= min(s, nx); ++s1) t = fma(x[s1], y[s - s1], t);
    out[s] = t;
  }
  g.sync();
}
// smallest T with sum_{s > T} m[s] 1.1^s <= thr (the dropped terms' bound on |u|, |v| <= 1.1, the back-substitution
// range); *tail receives that bound for T.  Uniform over the group (every lane scans m).
__device__ __forceinline__ int trunc_degree(const double* m, int d, double thr, double* tail) {
  double w = 1.0;
  for (int s = 0; s < d; ++s) w *= 1.1;  // 1.1^d
  double acc = 0.0;
  int T = d;
  for (int s = d; s >= 1; --s) {
    const double nacc = acc + m[s] * w;
    if (!(nacc <= thr)) break;
    acc = nacc;
    T = s - 1;
    w *= 1.0 / 1.1;
  }
  *tail = acc;
  return T;
}

// ------------------------------------------------------------------ scalar evaluation (one lane)
__device__ __forceinline__ double wp_row(const WP& p, int i, double v) {  // sum_j c_ij v^j
  const double* r = p.c + poff(p.d, i);
  double s = 0.0;
  for (int j = p.d - i; j >= 0; --j) s = fma(s, v, r[j]);
  return s;
}
__device__ __forceinline__ double wp_eval(const WP& p, double u, double v) {
  double acc = 0.0;
  for (int i = p.d; i >= 0; --i) acc = fma(acc, u, wp_row(p, i, v));
  return acc;
}

// ------------------------------------------------------------------ determinant of R(v) (Eq. 24)
// Slices a_l(v), b_l(v) (lane l; rows above the truncated degrees are stored as zero), Bezout columns by
// the Chionh recurrence B_ij = B_{i-1,j+1} + a_i b_{j+1} - b_i a_{j+1} (lane j holds column j; the matrix
// is symmetric, so the columns are the rows of B^T and det B^T = det B), then Gaussian elimination with
// partial pivoting by rows held in registers: the pivot row is chosen by a group max over the live rows
// (|x| quantised to 15 mantissa bits, lowest row on ties), broadcast by shuffles, never moved ("virtual"
// pivoting; the permutation sign is the parity of the unused rows above each pivot).  Returns sign(det)
// (0 for a zero pivot) and log|det| in *lg.  NC >= n is a compile-time bound (columns >= n are zero, so
// the update loops need no predicates); lanes >= n hold zero rows.
__device__ __forceinline__ void renorm(double& mant, int& ex) {
  const int hi = __double2hiint(mant);
  ex += ((hi >> 20) & 0x7ff) - 1022;
  mant = __hiloint2double((hi & 0x800fffff) | 0x3fe00000, __double2loint(mant));
}

template <int G, int NC>
__device__ int wdet_rows(const Grp<G>& g, double as, double bs, double aj1, double bj1, int n, double* lg) {
  const int l = g.lane;
  double col[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const double ai = g.bcast(as, i), bi = g.bcast(bs, i);
    double prev = g.down(i ? col[i - 1] : 0.0, 1);  // B_{i-1, j+1}
    if (i == 0 || l + 1 >= n) prev = 0.0;
    col[i] = (i < n) ? prev + (ai * bj1 - bi * aj1) : 0.0;
  }
  const bool live = l < n;
  unsigned used = 0u;
  int sign = 1;
  double mant = 1.0;
  int ex = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    if (c >= n) break;
    const bool cand = live && !((used >> l) & 1u);
    unsigned key = 0u;
    if (cand) key = (((unsigned)__double2hiint(fabs(col[c]))) & ~31u) | (unsigned)(31 - l);
    if (G == 32)
      key = __reduce_max_sync(0xffffffffu, key);  // one REDUX instead of a 5-step shuffle butterfly
    else
      for (int o = G / 2; o; o >>= 1) key = max(key, g.xor_(key, o));
    if ((key >> 5) == 0u) {
      *lg = -INFINITY;
      return 0;
    }
    const int p = 31 - (int)(key & 31u);
    const double piv = g.bcast(col[c], p);
    if ((__popc(~used & ((1u << p) - 1u)) & 1) ^ (piv < 0)) sign = -sign;
    mant *= fabs(piv);
    renorm(mant, ex);
    used |= 1u << p;
    const double lm = (cand && l != p) ? col[c] * fast_rcp(piv) : 0.0;
#pragma unroll
    for (int jj = c + 1; jj < NC; ++jj) col[jj] = fma(-lm, g.bcast(col[jj], p), col[jj]);
  }
  *lg = log(mant) + ex * 0.69314718055994530942;
  return sign;
}

// slice of row l at v from a transposed coefficient block AT[j * NR + l] (zero beyond the row)
template <int NR>
// D: the polynomial's total degree, so row l holds the terms j <= D - l (higher positions are structural zeros)
__device__ __forceinline__ double rowT(const double* __restrict__ AT, int D, int l, double v) {
  double s = 0.0;
  for (int j = D - l; j >= 0; --j) s = fma(s, v, __ldg(AT + j * NR + l));
  return s;
}

#ifndef SPOLY_WDET_INLINE
// one out-of-line copy per class: the scan calls it from three sites (first sample, next sample, bisection);
// A/B: C5 solve 2.01 -> 1.85 s (instruction-cache misses of the 20-row class), C4 -0.5%, bit-identical
#define SPOLY_WDET_INLINE __device__ __noinline__
#endif
// det sign for n <= G from the transposed blocks (the group evaluates the slices, lane l row l)
template <int G, int NR, int NCF = 0>
SPOLY_WDET_INLINE int wdet_T(const Grp<G>& g, const double* AT, int DA, const double* BT, int DB, int n, double v,
                      double* lg) {
  const int l = g.lane;
  const double as = rowT<NR>(AT, DA, l, v), bs = rowT<NR>(BT, DB, l, v);
  double aj1 = g.down(as, 1), bj1 = g.down(bs, 1);  // slices j + 1
  if (l == G - 1) {  // slice G is only needed when n == G (rows >= NR do not exist)
    constexpr int RG = G < NR ? G : 0;
    const bool need = G < NR && n >= G;
    aj1 = need ? rowT<NR>(AT, DA, RG, v) : 0.0;
    bj1 = need ? rowT<NR>(BT, DB, RG, v) : 0.0;
  }
  if (NCF) return wdet_rows<G, (NCF > 0 ? NCF : 8)>(g, as, bs, aj1, bj1, n, lg);  // fixed class (binned launch)
  if (G == 16) {
    if (n <= 8) return wdet_rows<G, 8>(g, as, bs, aj1, bj1, n, lg);
    if (n <= 12) return wdet_rows<G, 12>(g, as, bs, aj1, bj1, n, lg);
    return wdet_rows<G, 16>(g, as, bs, aj1, bj1, n, lg);
  }
  if (n <= 12) return wdet_rows<G, 12>(g, as, bs, aj1, bj1, n, lg);
  if (n <= 16) return wdet_rows<G, 16>(g, as, bs, aj1, bj1, n, lg);
  if (n <= 20) return wdet_rows<G, 20>(g, as, bs, aj1, bj1, n, lg);
  if (n <= 24) return wdet_rows<G, 24>(g, as, bs, aj1, bj1, n, lg);
  if (n <= 28) return wdet_rows<G, 28>(g, as, bs, aj1, bj1, n, lg);
  return wdet_rows<G, 32>(g, as, bs, aj1, bj1, n, lg);
}

// Several determinants per warp (the scan's samples of one system): L lanes per determinant ("quad" for L = 4),
// D = 32 / L determinants at once, lane t of a quad holding the columns r = t + L k (k < NC / L) of the symmetric
// Bezout matrix in registers.  The arithmetic per matrix entry is the same as wdet_rows' (slices by rowT, the
// Chionh recurrence, virtual partial pivoting on the quantised |x| with the lowest row on ties, one fma per entry
// and step), so every determinant's sign and log|det| are those wdet_rows computes; the communication per
// shuffle instruction serves D determinants instead of one.  All quads execute every step (n is the system's, so
// uniform); a quad whose determinant hit a zero pivot keeps stepping with its result frozen.
// a == b ? x : y through PTX selp (a plain select chain over a register array is turned into a dynamically
// indexed local-memory load by the compiler)
__device__ __forceinline__ double sel_eq(int a, int b, double x, double y) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\tselp.f64 %0, %3, %4, p;\n\t}"
      : "=d"(r) : "r"(a), "r"(b), "d"(x), "d"(y));
  return r;
}

template <int L, int NC, int NR>
__device__ __noinline__ int wdet_quad(const double* __restrict__ AT, int DA, const double* __restrict__ BT, int DB, int n, double v,
                         double* lg) {
  constexpr int RPL = (NC + L - 1) / L;   // columns per lane
  constexpr int SPL = (NC + L) / L;       // slices 0..NC per lane (i = t + L k)
  const int lane = threadIdx.x & 31, t = lane % L, qb = lane - t;
  // slices a_i(v), b_i(v), i = t + L k <= NC (rows >= NR are absent: zero)
  double sa[SPL], sb[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    const int i = t + L * k;
    const bool have = i <= NC && i < NR;
    sa[k] = have ? rowT<NR>(AT, DA, have ? i : 0, v) : 0.0;
    sb[k] = have ? rowT<NR>(BT, DB, have ? i : 0, v) : 0.0;
  }
  // a_{r+1}, b_{r+1} of each own column r = t + L k: slice r + 1 lives on lane (t + 1) % L, slot k (+1 if t = L-1)
  double aj1[RPL], bj1[RPL];
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int src = qb + (t + 1) % L;
    const double xa = __shfl_sync(0xffffffffu, sa[k], src), xb = __shfl_sync(0xffffffffu, sb[k], src);
    const double ya = (k + 1 < SPL) ? __shfl_sync(0xffffffffu, sa[k + 1 < SPL ? k + 1 : k], src) : 0.0;
    const double yb = (k + 1 < SPL) ? __shfl_sync(0xffffffffu, sb[k + 1 < SPL ? k + 1 : k], src) : 0.0;
    aj1[k] = (t + 1 < L) ? xa : ya;
    bj1[k] = (t + 1 < L) ? xb : yb;
  }
  double col[RPL][NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const double ai = __shfl_sync(0xffffffffu, sa[i / L], qb + i % L);
    const double bi = __shfl_sync(0xffffffffu, sb[i / L], qb + i % L);
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      // B_{i-1, r+1}: entry i - 1 of column r + 1 (lane (t + 1) % L, slot k, or slot k + 1 from lane 0)
      double prev = 0.0;
      if (i > 0) {
        const int src = qb + (t + 1) % L;
        const double x = __shfl_sync(0xffffffffu, col[k][i - 1], src);
        const double y = (k + 1 < RPL) ? __shfl_sync(0xffffffffu, col[k + 1 < RPL ? k + 1 : k][i - 1], src) : 0.0;
        prev = (t + 1 < L) ? x : y;
      }
      const int r = t + L * k;
      if (i == 0 || r + 1 >= n) prev = 0.0;
      col[k][i] = (i < n) ? prev + (ai * bj1[k] - bi * aj1[k]) : 0.0;
    }
  }
  unsigned used = 0u;
  int sign = 1, dead = 0;
  double mant = 1.0;
  int ex = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    if (c >= n) continue;  // uniform: n is the system's (no break: keeps the loop fully unrolled)
    bool cand[RPL];
    unsigned key = 0u;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int r = t + L * k;
      cand[k] = r < n && !((used >> r) & 1u);
      if (cand[k]) key = max(key, (((unsigned)__double2hiint(fabs(col[k][c]))) & ~31u) | (unsigned)(31 - r));
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
    if ((key >> 5) == 0u) dead = 1;
    const int p = 31 - (int)(key & 31u);
    const int owner = qb + p % L, kp = p / L;
    double sel = col[0][c];
#pragma unroll
    for (int k = 1; k < RPL; ++k) sel = sel_eq(kp, k, col[k][c], sel);
    const double piv = __shfl_sync(0xffffffffu, sel, owner);
    if (!dead) {
      if ((__popc(~used & ((1u << p) - 1u)) & 1) ^ (piv < 0)) sign = -sign;
      mant *= fabs(piv);
      renorm(mant, ex);
      used |= 1u << p;
    }
    const double rp = dead ? 0.0 : fast_rcp(piv);
    double lm[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) lm[k] = (cand[k] && t + L * k != p && !dead) ? col[k][c] * rp : 0.0;
#pragma unroll
    for (int jj = c + 1; jj < NC; ++jj) {
      double sj = col[0][jj];
#pragma unroll
      for (int k = 1; k < RPL; ++k) sj = sel_eq(kp, k, col[k][jj], sj);
      const double pj = __shfl_sync(0xffffffffu, sj, owner);
#pragma unroll
      for (int k = 0; k < RPL; ++k) col[k][jj] = fma(-lm[k], pj, col[k][jj]);
    }
  }
  if (dead) {
    *lg = -INFINITY;
    return 0;
  }
  *lg = log(mant) + ex * 0.69314718055994530942;
  return sign;
}

// Same determinant for n > G (rare: numerical TT orders above 32): matrix in the shared-memory scratch M
// (n*n doubles), rows built by the recurrence, elimination lane-parallel over columns.
template <int G, int NR>
__device__ int wdet_sign_smem(const Grp<G>& g, const double* AT, int DA, const double* BT, int DB, int n, double v,
                              double* lg, double* sl /* 2 (n + 2) */, double* M) {
  double* as = sl;
  double* bs = sl + n + 2;
  for (int i = g.lane; i <= n + 1; i += G) {
    as[i] = (i <= n && i < NR) ? rowT<NR>(AT, DA, i, v) : 0.0;
    bs[i] = (i <= n && i < NR) ? rowT<NR>(BT, DB, i, v) : 0.0;
  }
  g.sync();
  for (int i = 0; i < n; ++i) {
    for (int j = g.lane; j < n; j += G) {
      double t = as[i] * bs[j + 1] - bs[i] * as[j + 1];
      if (i > 0 && j + 1 < n) t += M[(i - 1) * n + j + 1];
      M[i * n + j] = t;
    }
    g.sync();
  }
  int sign = 1;
  double mant = 1.0;
  int ex = 0;
  for (int c = 0; c < n; ++c) {
    double best = -1.0;
    int piv = c;
    for (int r = c + g.lane; r < n; r += G) {
      const double x = fabs(M[r * n + c]);
      if (x > best) {
        best = x;
        piv = r;
      }
    }
    for (int o = G / 2; o; o >>= 1) {
      const double ob = g.xor_(best, o);
      const int op = g.xor_(piv, o);
      if (ob > best || (ob == best && op < piv)) {
        best = ob;
        piv = op;
      }
    }
    if (!(best > 0.0)) {
      *lg = -INFINITY;
      g.sync();
      return 0;
    }
    if (piv != c) {
      sign = -sign;
      for (int l2 = c + g.lane; l2 < n; l2 += G) {
        const double t = M[c * n + l2];
        M[c * n + l2] = M[piv * n + l2];
        M[piv * n + l2] = t;
      }
      g.sync();
    }
    const double d = M[c * n + c];
    if (d < 0) sign = -sign;
    int e;
    mant = frexp(mant * fabs(d), &e);
    ex += e;
    for (int r = c + 1; r < n; ++r) {
      const double fr = M[r * n + c] / d;
      g.sync();
      if (fr != 0.0)
        for (int l2 = c + 1 + g.lane; l2 < n; l2 += G) M[r * n + l2] = fma(-fr, M[c * n + l2], M[r * n + l2]);
    }
    g.sync();
  }
  *lg = log(mant) + ex * 0.69314718055994530942;
  return sign;
}

}  // namespace spoly
