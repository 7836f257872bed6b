// Device polynomial helpers for the fused solve kernels: fixed-size, fully unrolled, FP64.
// Univariate p(v) = sum_i c[i] v^i; bivariate grids G[i][j] = coeff of u^i v^j (i+j <= D).
#pragma once
#include "common.cuh"

namespace spoly {

template <int N>
__device__ __forceinline__ double horner(const double* c, double x) {
  double s = c[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) s = fma(s, x, c[i]);
  return s;
}

// runtime-degree Horner (deg <= N-1), unrolled with predication
template <int N>
__device__ __forceinline__ double horner_rt(const double* c, int deg, double x) {
  double s = 0.0;
#pragma unroll
  for (int i = N - 1; i >= 0; --i)
    if (i <= deg) s = fma(s, x, c[i]);
  return s;
}

// C[0..NA+NB-2] (+)= s * A[0..NA-1] * B[0..NB-1]
template <int NA, int NB>
__device__ __forceinline__ void pmul_acc(const double* A, const double* B, double s, double* C) {
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const double a = s * A[i];
#pragma unroll
    for (int j = 0; j < NB; ++j) C[i + j] = fma(a, B[j], C[i + j]);
  }
}

// bivariate product: C (degree DA+DB grid, stride SC) += s * A (DA, stride SA) * B (DB, stride SB)
template <int DA, int DB, int SA, int SB, int SC>
__device__ __forceinline__ void bmul_acc(const double* A, const double* B, double s, double* C) {
#pragma unroll
  for (int i = 0; i <= DA; ++i)
#pragma unroll
    for (int j = 0; i + j <= DA; ++j) {
      const double a = s * A[i * SA + j];
#pragma unroll
      for (int k = 0; k <= DB; ++k)
#pragma unroll
        for (int l = 0; k + l <= DB; ++l) C[(i + k) * SC + (j + l)] = fma(a, B[k * SB + l], C[(i + k) * SC + (j + l)]);
    }
}

template <int D, int S>
__device__ __forceinline__ void bscale(double* G, double s) {
#pragma unroll
  for (int i = 0; i <= D; ++i)
#pragma unroll
    for (int j = 0; i + j <= D; ++j) G[i * S + j] *= s;
}
// per-u-row max |c_ij| in one pass (rm[i]) and the overall max (return value).  Scaling by s > 0 is monotone
// under rounding, so max_j fl(|c_ij| s) = fl(rm[i] s): the numerical u-degree of the scaled grid can be taken
// from the unscaled row maxima (bit-identical to taking the maxima after scaling; one max pass instead of two)
template <int D, int S>
__device__ __forceinline__ double browmax(const double* G, double* rm) {
  double m = 0.0;
#pragma unroll
  for (int i = 0; i <= D; ++i) {
    double r = 0.0;
#pragma unroll
    for (int j = 0; i + j <= D; ++j) r = dmax(r, fabs(G[i * S + j]));
    rm[i] = r;
    m = dmax(m, r);
  }
  return m;
}
// numerical u-degree of the grid scaled by s: max{i : max_j |s c_ij| 1.1^i > tau}, from the
// unscaled row maxima (see browmax)
template <int D>
__device__ __forceinline__ int bnum_udeg_rows(const double* rm, double s, double tau) {
  int d = 0;
  double f = 1.0;
#pragma unroll
  for (int i = 0; i <= D; ++i) {
    if ((rm[i] * s) * f > tau) d = i;
    f *= 1.1;
  }
  return d;
}
template <int D, int S>
__device__ __forceinline__ void btrunc_u(double* G, int d) {
#pragma unroll
  for (int i = 0; i <= D; ++i)
#pragma unroll
    for (int j = 0; i + j <= D; ++j)
      if (i > d) G[i * S + j] = 0.0;
}
// evaluate G(u, v) and its partials
template <int D, int S>
__device__ __forceinline__ void beval(const double* G, double u, double v, double* f, double* fu, double* fv) {
  // slices s_i(v) and s_i'(v), then Horner in u
  double s[D + 1], sd[D + 1];
#pragma unroll
  for (int i = 0; i <= D; ++i) {
    double acc = 0.0, dacc = 0.0;
#pragma unroll
    for (int j = D - i; j >= 0; --j) {
      dacc = fma(dacc, v, acc);
      acc = fma(acc, v, G[i * S + j]);
    }
    s[i] = acc;
    sd[i] = dacc;
  }
  double p = 0.0, pu = 0.0, pv = 0.0;
#pragma unroll
  for (int i = D; i >= 0; --i) {
    pu = fma(pu, u, p);
    p = fma(p, u, s[i]);
    pv = fma(pv, u, sd[i]);
  }
  *f = p;
  *fu = pu;
  *fv = pv;
}
// slice values a_i(v) for i = 0..D
template <int D, int S>
__device__ __forceinline__ void bslices_at(const double* G, double v, double* out) {
#pragma unroll
  for (int i = 0; i <= D; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = D - i; j >= 0; --j) acc = fma(acc, v, G[i * S + j]);
    out[i] = acc;
  }
}

// ---------------------------------------------------------------------------------------------
// Real roots in [lo, hi] of a polynomial of degree <= N-1 (coefficients c[0..N-1], exact-zero
// trimmed by the caller to degree `deg`), by the paper's derivative recursion:
// roots of p^(k+1) split p^(k) into monotone pieces; each piece with a sign change holds one root.
// Each piece is solved by Newton's method safeguarded by bisection (the GPU formulation of
// Yuksel 2022, cited by the paper at PAPER.md:574), to |step| <= 1e-15 — tighter than the paper's
// 1e-9 bracket threshold, so the roots agree with the oracle's to well inside the parity tolerance.
// Also returns, for the top level (p itself), the critical points' |p| and max_[lo,hi] |p| for the
// near-tangent flag.
template <int N, bool PROBES = false>
struct RootSet {
  double x[N];
  int n;
  double min_crit_ratio;  // min over critical points c in (lo,hi) of |p(c)| / max|p| (1 if none)
  int flags;              // 1: roots closer than eps
  uint32_t terms;         // FMA terms evaluated (FLOP model)
  // PROBES: positions of the c14 near-tangency conditions (reading R11): midpoints of root pairs closer than eps,
  // critical points c with |p(c)| <= 1e-10 max_[lo,hi] |p|
  double probe[PROBES ? 2 * N : 1];
  int nprobe;
};

// falling factorials F[k][i] = i!/(i-k)! (0 for i < k), for the derivative levels p^(k)
static __constant__ double c_falling[16][16] = {
    {1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0},
    {0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0, 9.0, 10.0, 11.0, 12.0, 13.0, 14.0, 15.0},
    {0.0, 0.0, 2.0, 6.0, 12.0, 20.0, 30.0, 42.0, 56.0, 72.0, 90.0, 110.0, 132.0, 156.0, 182.0, 210.0},
    {0.0, 0.0, 0.0, 6.0, 24.0, 60.0, 120.0, 210.0, 336.0, 504.0, 720.0, 990.0, 1320.0, 1716.0, 2184.0, 2730.0},
    {0.0, 0.0, 0.0, 0.0, 24.0, 120.0, 360.0, 840.0, 1680.0, 3024.0, 5040.0, 7920.0, 11880.0, 17160.0, 24024.0, 32760.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 120.0, 720.0, 2520.0, 6720.0, 15120.0, 30240.0, 55440.0, 95040.0, 154440.0, 240240.0, 360360.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 720.0, 5040.0, 20160.0, 60480.0, 151200.0, 332640.0, 665280.0, 1235520.0, 2162160.0, 3603600.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 5040.0, 40320.0, 181440.0, 604800.0, 1663200.0, 3991680.0, 8648640.0, 17297280.0, 32432400.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 40320.0, 362880.0, 1814400.0, 6652800.0, 19958400.0, 51891840.0, 121080960.0, 259459200.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 362880.0, 3628800.0, 19958400.0, 79833600.0, 259459200.0, 726485760.0, 1816214400.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 3628800.0, 39916800.0, 239500800.0, 1037836800.0, 3632428800.0, 10897286400.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 39916800.0, 479001600.0, 3113510400.0, 14529715200.0, 54486432000.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 479001600.0, 6227020800.0, 43589145600.0, 217945728000.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 6227020800.0, 87178291200.0, 653837184000.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 87178291200.0, 1307674368000.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1307674368000.0}};

// reciprocal good to ~1e-15 relative: MUFU.RCP64H seed (rcp.approx.ftz.f64) + two FP64 Newton
// refinements.  The Newton step of the root solver only needs an accurate-enough quotient (the bracket
// guarantees convergence), so the correctly rounded DDIV sequence is not needed.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

// p^(k)(x) and p^(k+1)(x) from the per-level coefficient registers g (p^(k) basis) and h (p^(k+1))
template <int N>
__device__ __forceinline__ double level_eval(const double* g, const double* h, int k, int deg, double x, double* dval) {
  double s = 0.0, d = 0.0;
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    if (i >= k && i <= deg) s = fma(s, x, g[i]);
    if (i >= k + 1 && i <= deg) d = fma(d, x, h[i]);
  }
  *dval = d;
  return s;
}

template <int N>
__device__ __forceinline__ double solve_piece(const double* g, const double* h, int k, int deg, double lo, double hi,
                                              double flo, double fhi, int* its) {
  // secant start inside the bracket, then Newton safeguarded by bisection; |step| <= 1e-12 stops
  // (quadratic convergence: the error after such a step is far below 1e-15)
  double x = lo - flo * (hi - lo) / (fhi - flo);
  if (!(x > lo && x < hi)) x = 0.5 * (lo + hi);
  for (int it = 0; it < 100; ++it) {
    double fp;
    const double f = level_eval<N>(g, h, k, deg, x, &fp);
    if (f == 0.0) {
      *its = it + 1;
      return x;
    }
    if ((f < 0.0) == (flo < 0.0))
      lo = x;
    else
      hi = x;
    double xn = x - f * fast_rcp(fp);
    // convergence before the bracket safeguard (a sub-ulp step may land on the endpoint x just became)
    if (fabs(xn - x) <= 1e-12) {
      *its = it + 1;
      return fmin(fmax(xn, lo), hi);
    }
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
    if (hi - lo <= 1e-15) {
      *its = it + 1;
      return xn;
    }
    x = xn;
  }
  *its = 100;
  return x;
}

// Root of a polynomial that is monotone on [lo, hi] (its derivative is root-free there), degree <= N-1,
// all N coefficients live: full-length unrolled Horner (no per-level predication).  Returns the number
// of roots (0 or 1; an exact zero at an endpoint counts as in the general recursion).
template <int N>
__device__ __forceinline__ int monotone_root(const double* c, double lo, double hi, double* root, uint32_t* terms) {
  double flo = c[N - 1], fhi = c[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) {
    flo = fma(flo, lo, c[i]);
    fhi = fma(fhi, hi, c[i]);
  }
  *terms += 2 * N;
  if (flo == 0.0) {
    *root = lo;
    return 1;
  }
  if (fhi == 0.0) {
    *root = hi;
    return 1;
  }
  if ((flo < 0.0) == (fhi < 0.0)) return 0;
  double a = lo, b = hi;
  double x = a - flo * (b - a) / (fhi - flo);
  if (!(x > a && x < b)) x = 0.5 * (a + b);
  for (int it = 0; it < 100; ++it) {
    double f = c[N - 1], fp = 0.0;
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
      fp = fma(fp, x, f);
      f = fma(f, x, c[i]);
    }
    *terms += 2 * N - 1;
    if (f == 0.0) break;
    if ((f < 0.0) == (flo < 0.0))
      a = x;
    else
      b = x;
    double xn = x - f * fast_rcp(fp);
    // convergence before the bracket safeguard (a sub-ulp step may land on the endpoint x just became)
    if (fabs(xn - x) <= 1e-12) {
      x = fmin(fmax(xn, a), b);
      break;
    }
    if (!(xn > a && xn < b)) xn = 0.5 * (a + b);
    if (b - a <= 1e-15) {
      x = xn;
      break;
    }
    x = xn;
  }
  *root = x;
  return 1;
}

// kstart: a derivative level known to have no root in (lo, hi) (so p^(kstart-1) is monotone there and
// the recursion starts at level kstart-1 with no critical points); kstart < 0 or >= deg-1 runs the plain
// recursion from the linear level deg-1.
template <int N, bool PROBES = false>
__device__ void isolate_roots(const double* c, int deg, double lo, double hi, double eps_close, RootSet<N, PROBES>& R,
                              int kstart = -1) {
  R.terms = 0;
  R.n = 0;
  R.min_crit_ratio = 1.0;
  R.flags = 0;
  R.nprobe = 0;
  double fc[PROBES ? N : 1];  // |p| at the critical points (PROBES)
  if (deg <= 0) return;
  double prev[N];
  int nprev = 0;
  if (kstart < 0 || kstart >= deg - 1) {
    // level deg-1: p^(deg-1)(x) = c_{deg-1} (deg-1)! + c_deg deg! x   (linear: closed form)
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i == deg - 1) a0 = c[i] * c_falling[deg - 1][i];
      if (i == deg) a1 = c[i] * c_falling[deg - 1][i];
    }
    double x = -a0 / a1;
    if (deg == 1) {
      if (x >= lo && x <= hi) R.x[R.n++] = x;
      return;
    }
    if (x > lo && x < hi) prev[nprev++] = x;
    kstart = deg - 1;
  }
  for (int k = kstart - 1; k >= 0; --k) {
    double g[N], h[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      g[i] = c[i] * c_falling[k][i];
      h[i] = g[i] * (double)(i - k);
    }
    double cur[N];
    int ncur = 0;
    double xa = lo, dummy;
    double fa = level_eval<N>(g, h, k, deg, xa, &dummy);
    double fmax_ = fabs(fa), cmin = INFINITY;
    R.terms += (uint32_t)(nprev + 2) * (uint32_t)(deg - k + 1) + 2u * N;
    for (int i = 0; i <= nprev; ++i) {
      double xb = (i < nprev) ? prev[i] : hi;
      double fb = level_eval<N>(g, h, k, deg, xb, &dummy);
      if (k == 0) {
        fmax_ = fmax(fmax_, fabs(fb));
        if (i < nprev) {
          cmin = fmin(cmin, fabs(fb));
          if (PROBES) fc[i] = fabs(fb);
        }
      }
      if (fa == 0.0) {
        cur[ncur++] = xa;
      } else if (fb != 0.0 && ((fa < 0.0) != (fb < 0.0))) {
        int its = 0;
        cur[ncur++] = solve_piece<N>(g, h, k, deg, xa, xb, fa, fb, &its);
        R.terms += (uint32_t)its * (uint32_t)(2 * (deg - k) + 1);
      }
      xa = xb;
      fa = fb;
    }
    if (fa == 0.0) cur[ncur++] = hi;
    if (k == 0) {
      if (nprev > 0 && fmax_ > 0) R.min_crit_ratio = cmin / fmax_;
      for (int i = 0; i < ncur; ++i) {
        if (i > 0 && cur[i] - cur[i - 1] < eps_close) {
          R.flags |= 1;
          if (PROBES) R.probe[R.nprobe++] = 0.5 * (cur[i] + cur[i - 1]);
        }
        R.x[i] = cur[i];
      }
      R.n = ncur;
      if (PROBES)
        for (int i = 0; i < nprev; ++i)
          if (fc[i] <= 1e-10 * fmax_) R.probe[R.nprobe++] = prev[i];
      return;
    }
    nprev = 0;
    for (int i = 0; i < ncur; ++i)
      if (cur[i] > lo && cur[i] < hi) prev[nprev++] = cur[i];
  }
}

}  // namespace spoly
