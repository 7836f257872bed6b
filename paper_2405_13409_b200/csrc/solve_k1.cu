// One-bounce solve, reflection "R" (Eq. 21) and refraction "T" (Eq. 22), split into two kernels so that
// every lane has work:
//
//   k1_phase1 (one thread per (query, triangle) pair, uniform control flow):
//       decisions (readings R1, c7) -> coefficient phase (Eq. 6 a; Eq. 12 b for R, Eq. 9 b for T)
//       -> normalise + truncate (c5) -> elimination phase: r(v) (R: Eq. 24 Bezout + Laplace expansion,
//       PAPER.md:607; T: Res_u(a,b) by pseudo-remainder, reading R5) -> r normalised -> Bernstein
//       root-free level; pairs whose r may have a root in [0,1] are appended to a dense job list.
//   k1_phase2 (one thread per job):
//       univariate roots (derivative recursion) -> back-substitution
//       -> (a,b) refinement (reading R2) -> Eq. 3 validation, sides, flags -> contribution (c15)
//       -> warp-aggregated emission.  The coefficient phase is recomputed from the geometry (same code,
//       bit-identical) instead of being stored.
#include "kernels.cuh"
#include "solve_k1.cuh"

#include <cstdio>

namespace spoly {

template <bool TC>
struct Sys1 {
  static constexpr int DB = TC ? 6 : 4;   // total degree of b (Table 2: square form 6, product form 4)
  static constexpr int NR = TC ? 13 : 10; // coefficients of r(v): degree 12 (T), 9 (R)
  double A[9], B[(DB + 1) * (DB + 1)];
  double eta0, eta1;
  bool relabel;
  uint32_t flags;
  int da, db, n;
};

// decisions + coefficient phase + normalisation/truncation; false when the system is degenerate.
// WITH_B = false builds only a (same arithmetic, bit-identical A) for the candidate pre-pass.
template <bool TC, bool WITH_B = true>
__device__ __forceinline__ bool build_system(d3 x0, d3 x2, const d3 P_in[3], const d3 N_in[3],
                                             const SolveParams& prm, Sys1<TC>& S) {
  constexpr int DB = Sys1<TC>::DB;
  S.flags = 0;
  // reading R1: incidence-plane normal l_c = (x2 - x0) x n(centroid); the tests below are the reading's
  // comparisons squared and cross-multiplied (no square roots or divisions; equal up to rounding at ties)
  const d3 nc = (1.0 / 3.0) * (N_in[0] + N_in[1] + N_in[2]);
  const d3 w0 = x2 - x0;
  const d3 lc = cross(w0, nc);
  const double ln2 = dot(lc, lc);
  if (!(ln2 > 1e-24 * dot(w0, w0) * dot(nc, nc))) S.flags |= SPOLY_FLAG_DEGENERATE;
  const d3 e1o = P_in[1] - P_in[0], e2o = P_in[2] - P_in[0];
  S.relabel = false;
  S.eta0 = S.eta1 = 1.0;
  if (!TC) {
    // product form: t = n x e1 unless e2 is further out of the incidence plane (relabel p1 <-> p2):
    // |e1.lc| / |e1| < |e2.lc| / |e2|
    if (ln2 > 0) {
      const double d1 = dot(e1o, lc), d2 = dot(e2o, lc);
      S.relabel = d1 * d1 * dot(e2o, e2o) < d2 * d2 * dot(e1o, e1o);
    }
  } else {
    // c7: eta_0 from the side of x_0 w.r.t. the triangle's geometric plane; refraction flips the medium
    const bool front = dot(x0 - P_in[0], cross(e1o, e2o)) > 0;
    S.eta0 = front ? prm.eta_front : prm.eta_back;
    S.eta1 = front ? prm.eta_back : prm.eta_front;
  }
  const d3 p0 = P_in[0], p1 = S.relabel ? P_in[2] : P_in[1], p2 = S.relabel ? P_in[1] : P_in[2];
  const d3 n0 = N_in[0], n1 = S.relabel ? N_in[2] : N_in[1], n2 = S.relabel ? N_in[1] : N_in[2];
  const d3 e1 = p1 - p0, e2 = p2 - p0, m1 = n1 - n0, m2 = n2 - n0;
  const d3 q = p0 - x0, w = x2 - x0;
  build_a(q, w, e1, e2, n0, m1, m2, S.A);
  if (WITH_B) {
    if (TC) {
      const double ln = sqrt(ln2);
      const d3 l = ln > 0 ? (1.0 / ln) * lc : mk3(1, 0, 0);
      build_b_T(q, w, e1, e2, n0, m1, m2, l, S.eta0, S.eta1, S.B);
    } else {
      build_b_R(q, w, e1, e2, n0, m1, m2, S.B);
    }
  }
  double rma[3], rmb[DB + 1];
  const double ma = browmax<2, 3>(S.A, rma), mb = WITH_B ? browmax<DB, DB + 1>(S.B, rmb) : 1.0;
  if (!(ma > 0) || !(mb > 0)) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  const double sa = 1.0 / ma, sb = 1.0 / mb;
  bscale<2, 3>(S.A, sa);
  if (WITH_B) bscale<DB, DB + 1>(S.B, sb);
  // numerical u-degree truncation (R6): rarely active for one bounce, so the zeroing is branched around (not
  // predicated over every coefficient)
  S.da = bnum_udeg_rows<2>(rma, sa, prm.tau_trunc);
  if (S.da < 2) btrunc_u<2, 3>(S.A, S.da);
  if (!WITH_B) return true;
  S.db = bnum_udeg_rows<DB>(rmb, sb, prm.tau_trunc);
  if (S.db < (TC ? DB : DB - 1)) btrunc_u<DB, DB + 1>(S.B, S.db);  // R: row 4 is structurally zero already
  S.n = max(S.da, S.db);
  if (S.n == 0) {
    S.flags |= SPOLY_FLAG_DEGENERATE;
    return false;
  }
  return true;
}

// Bernstein form of the quadratic a(u,v) on the triangle (6 control points: corners c00, c00+c10+c20,
// c00+c01+c02 and edge points c00+c10/2, c00+c01/2, c00+(c10+c01+c11)/2); a strict common sign with a
// margin of 1e-4 sum|c| (>> |grad a| * 1e-6) proves a != 0 on the triangle enlarged by 1e-6.
__device__ __forceinline__ bool coplanarity_may_vanish(const double* A) {
  const double c00 = A[0], c01 = A[1], c02 = A[2], c10 = A[3], c11 = A[4], c20 = A[6];
  const double b0 = c00, b1 = c00 + c10 + c20, b2 = c00 + c01 + c02, b3 = c00 + 0.5 * c10, b4 = c00 + 0.5 * c01,
               b5 = c00 + 0.5 * (c10 + c01 + c11);
  const double m = 1e-4 * (fabs(c00) + fabs(c01) + fabs(c02) + fabs(c10) + fabs(c11) + fabs(c20));
  const bool pos = b0 > m && b1 > m && b2 > m && b3 > m && b4 > m && b5 > m;
  const bool neg = b0 < -m && b1 < -m && b2 < -m && b3 < -m && b4 < -m && b5 < -m;
  return !(pos || neg);
}

template <bool TC>
__device__ __forceinline__ void eliminate(const Sys1<TC>& S, double* r) {
  if (TC)
    resultant_T(S.A, S.B, S.da, S.db, r);
  else
    det_R(S.A, S.B, S.n, r);
}

// ---------------------------------------------------------------------------------------------
// warp-aggregated appends (all 32 lanes must call)
__device__ __forceinline__ unsigned long long warp_alloc(unsigned long long* counter, uint32_t n, uint32_t* excl) {
  const int lane = threadIdx.x & 31;
  uint32_t incl = n;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (total) {
    if (lane == 31) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
  }
  *excl = incl - n;
  return base;
}

__device__ __forceinline__ void emit_flag(bool has, uint32_t flags, uint64_t pair, const SolSink& S) {
  uint32_t ex;
  const unsigned long long base = warp_alloc(S.count + 1, has ? 1u : 0u, &ex);
  if (has && base + ex < S.fcapacity) {
    S.fkey[base + ex] = pair;
    S.fflags[base + ex] = flags;
  }
}

__device__ __forceinline__ void flush_counters(const SolSink& S, const uint32_t* cnt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) {
    uint32_t v = cnt[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0 && v) atomicAdd(S.counters + i, (unsigned long long)v);
  }
}

__device__ __forceinline__ void load_pair(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                          const TriRec* __restrict__ tris, const double* __restrict__ ep, uint64_t i,
                                          d3 P[3], d3 N[3], d3& x0, d3& x2, uint32_t& q) {
  q = __ldg(pq + i);
  load_tri(tris, __ldg(pt + i), P, N);
  const double* e = ep + 6ull * q;
  x0 = mk3(__ldg(e), __ldg(e + 1), __ldg(e + 2));
  x2 = mk3(__ldg(e + 3), __ldg(e + 4), __ldg(e + 5));
}

// real roots u of a(., v*) when a is quadratic / linear in u (stable formula, disc clamp; reading R4),
// sorted, merged below 1e-7.  |disc| <= 1e-8 scale (two u-roots about to merge, c14) reports the double root's
// position in *udouble (a near-tangency condition probed by the path kernel, reading R11), else NaN.
__device__ __forceinline__ int quadratic_u_roots(const double al[3], double* ua, double* udouble) {
  int nu = 0;
  *udouble = __longlong_as_double(0x7ff8000000000000ll);
  if (al[2] != 0.0) {
    const double a0 = al[0], a1 = al[1], a2 = al[2];
    double disc = a1 * a1 - 4.0 * a2 * a0;
    const double sc = a1 * a1 + 4.0 * fabs(a2 * a0);
    if (fabs(disc) <= 1e-8 * sc) *udouble = -a1 / (2.0 * a2);
    if (!(disc < -1e-12 * sc)) {
      if (disc < 0) disc = 0;
      const double qq = -0.5 * (a1 + copysign(sqrt(disc), a1));
      if (qq == 0.0) {
        ua[nu++] = 0.0;
      } else {
        double r1 = qq / a2, r2 = a0 / qq;
        if (r1 > r2) {
          const double t = r1;
          r1 = r2;
          r2 = t;
        }
        ua[nu++] = r1;
        if (r2 - r1 >= 1e-7) ua[nu++] = r2;
      }
    }
  } else if (al[1] != 0.0) {
    ua[nu++] = -al[0] / al[1];
  }
  return nu;
}

// phase 1's pre-check only needs the candidates to ~1e-12 (it rejects those > 3e-3 outside the triangle, the
// refinement moves them <= 1e-3): the same stable formula with reciprocals instead of correctly rounded divisions
__device__ __forceinline__ int quadratic_u_roots_precheck(const double al[3], double* ua, bool* near_double) {
  int nu = 0;
  *near_double = false;
  if (al[2] != 0.0) {
    const double a0 = al[0], a1 = al[1], a2 = al[2];
    double disc = a1 * a1 - 4.0 * a2 * a0;
    const double sc = a1 * a1 + 4.0 * fabs(a2 * a0);
    if (fabs(disc) <= 1e-8 * sc) *near_double = true;
    if (!(disc < -1e-12 * sc)) {
      if (disc < 0) disc = 0;
      const double qq = -0.5 * (a1 + copysign(sqrt(disc), a1));
      if (qq == 0.0) {
        ua[nu++] = 0.0;
      } else {
        ua[nu++] = qq * fast_rcp(a2);
        ua[nu++] = a0 * fast_rcp(qq);
      }
    }
  } else if (al[1] != 0.0) {
    ua[nu++] = -al[0] * fast_rcp(al[1]);
  }
  return nu;
}

// the refinement (reading R2) moves u and v by at most 1e-3 each (1 - u - v by 2e-3), so a candidate more than
// 3e-3 outside the simplex can neither become admissible nor land within eps_flag of an edge
__device__ __forceinline__ bool precheck_reject(double us, double vv) {
  return us < -3e-3 || vv < -3e-3 || 1.0 - us - vv < -3e-3;
}

// ---------------------------------------------------------------------------------------------
// resident blocks per SM (A/B on C2, R: 4 -> 5 (<= 96 registers, 156 B spill) took phase 1 2.48 -> 2.38 ms; T spills
// 1.2 KB at 5 and keeps 4)
#ifndef SPOLY_P1_MINB
#define SPOLY_P1_MINB 5
#endif
#ifndef SPOLY_P1_MINB_T
#define SPOLY_P1_MINB_T 4
#endif
#ifdef SPOLY_PATH_MINB
#define SPOLY_PATH_BOUNDS __launch_bounds__(128, SPOLY_PATH_MINB)
#else
#define SPOLY_PATH_BOUNDS __launch_bounds__(128)
#endif
template <bool TC>
__global__ void __launch_bounds__(128, TC ? SPOLY_P1_MINB_T : SPOLY_P1_MINB) k1_phase1(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                                    uint64_t npairs, const TriRec* __restrict__ tris,
                                                    const double* __restrict__ ep, SolveParams prm, SolSink S,
                                                    JobSink J) {
  constexpr int NR = Sys1<TC>::NR;
  uint32_t cnt[C_NUM];
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // block-uniform loop (same pair mapping as a warp-strided loop): the monotone-job append is aggregated
  // over the block's 4 warps, one atomic per 128 pairs (same-address atomics serialise in L2)
  __shared__ uint32_t s_off[4];
  __shared__ unsigned long long s_base;
  // a's 6 coefficients wait in shared memory (not registers) through the elimination and the Bernstein
  // test, until the job slot is known; [coefficient][thread], conflict-free
  __shared__ double s_aj[6][128];
#if defined(SPOLY_P1_WARP_BUFFER)
  __shared__ uint32_t s_wpair[4][64];
  __shared__ double s_wroot[4][64];
  int wbuf_n = 0;  // warp-uniform
#endif
  for (uint64_t bb = (uint64_t)blockIdx.x * blockDim.x; bb < npairs; bb += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = bb + threadIdx.x;
    const bool active = i < npairs;
    bool job = false;
    uint32_t flags = 0, meta = 0;
    double r[NR];
    if (active) {
      d3 P[3], N[3], x0, x2;
      uint32_t q;
      load_pair(pq, pt, tris, ep, i, P, N, x0, x2, q);
      cnt[C_PAIRS]++;
      Sys1<TC> Sys;
      bool ok = build_system<TC>(x0, x2, P, N, prm, Sys);
      flags = Sys.flags;
      if (ok) {
        cnt[C_SYSTEMS]++;
      }
      if (ok && !coplanarity_may_vanish(Sys.A)) {
        // a(u,v) = Eq. 6 has a strict sign on the triangle (enlarged far beyond the 1e-9 domain slack), so
        // no chain exists on this pair: exact early out (no effect on the admissible set)
        ok = false;
      } else if (ok) {
        cnt[C_ELIMS]++;
        s_aj[0][threadIdx.x] = Sys.A[0]; s_aj[1][threadIdx.x] = Sys.A[1]; s_aj[2][threadIdx.x] = Sys.A[2];
        s_aj[3][threadIdx.x] = Sys.A[3]; s_aj[4][threadIdx.x] = Sys.A[4]; s_aj[5][threadIdx.x] = Sys.A[6];
        eliminate<TC>(Sys, r);
        double mr = 0.0;
#pragma unroll
        for (int t = 0; t < NR; ++t) mr = dmax(mr, fabs(r[t]));
        if (!(mr > 0)) {
          flags |= SPOLY_FLAG_DEGENERATE;
        } else {
          const double inv = 1.0 / mr;
#pragma unroll
          for (int t = 0; t < NR; ++t) r[t] *= inv;
          int deg = NR - 1;  // exact structural zeros at the top are rare (face mode, special geometry)
          while (deg > 0 && r[deg] == 0.0) --deg;
          const int kfree = bernstein_root_free_level<NR>(r);
          // kfree == 1: r is monotone on [0,1], so it has a root there iff r(0) and r(1) differ in sign
          // (or one vanishes) -- exact, and it keeps root-free monotone pairs out of the job list
          double r1 = 0.0;
#pragma unroll
          for (int t = NR - 1; t >= 0; --t) r1 += r[t];
          const bool mono_root = !(r[0] * r1 > 0.0);
          if (kfree > 0 && deg > 0 && (kfree > 1 || mono_root)) {
            job = true;
            meta = (uint32_t)kfree | ((uint32_t)deg << 8);
          }
        }
      }
    }
    // ---- monotone jobs (kfree == 1, ~99% of the jobs): the root of r on [0, 1] by the safeguarded Newton
    // iteration of the derivative recursion's monotone piece (reading R13), then the back-substitution
    // pre-check (reading R2's 1e-3 refinement radius): a job whose every candidate lies > 3e-3 outside the triangle
    // and that raises no c14 condition is finished here.  Only (pair, root) of the survivors leaves the kernel
    // (12 B instead of the 128 B job record of round 1).  Lanes iterate independently (3.1 steps on average).
    const bool mono = job && (meta & 0xFF) == 1;
    bool to_path = false, complex_job = false;
    double root = 0.0;
    if (mono) {
      double f1 = 0.0;
#pragma unroll
      for (int t = NR - 1; t >= 0; --t) f1 += r[t];  // r(1)
      const double f0 = r[0];
      cnt[C_EVAL_TERMS] += 2 * NR;
      bool has = true;
      if (f0 == 0.0 || f1 == 0.0) {
        root = f0 == 0.0 ? 0.0 : 1.0;  // exact endpoint root
      } else if ((f0 < 0.0) == (f1 < 0.0)) {
        has = false;  // rounding: no sign change after all
      } else {
        double a = 0.0, b = 1.0, x = -f0 / (f1 - f0);  // secant start
        bool conv = false;
        if (!(x > a && x < b)) x = 0.5;
        for (int it = 0; it < 100; ++it) {
          double f = r[NR - 1], fp = 0.0;
#pragma unroll
          for (int t = NR - 2; t >= 0; --t) {
            fp = fma(fp, x, f);
            f = fma(f, x, r[t]);
          }
          cnt[C_EVAL_TERMS] += 2 * NR - 1;
          if (f == 0.0) break;
          if ((f < 0.0) == (f0 < 0.0))
            a = x;
          else
            b = x;
          double xn = x - f * fast_rcp(fp);
          // convergence is tested before the bracket safeguard: at the root the Newton step is below an ulp and may
          // land on the endpoint x just became, which must not trigger a bisection from a far bracket (the
          // converged step is clamped into the bracket once, after the loop)
          if (fabs(xn - x) <= 1e-12) {
            x = xn;
            conv = true;
            break;
          }
          if (!(xn > a && xn < b)) xn = 0.5 * (a + b);
          x = xn;
          if (b - a <= 1e-15) break;
        }
        root = conv ? dmin(dmax(a, x), b) : x;
      }
      if (has) {
        cnt[C_VROOTS]++;
        cnt[C_CAND_JOBS]++;
        // back-substitution in a (phase 1's normalised coefficients, parked in shared memory) + domain pre-check
        double A[9];
        A[0] = s_aj[0][threadIdx.x]; A[1] = s_aj[1][threadIdx.x]; A[2] = s_aj[2][threadIdx.x];
        A[3] = s_aj[3][threadIdx.x]; A[4] = s_aj[4][threadIdx.x]; A[6] = s_aj[5][threadIdx.x];
        A[5] = A[7] = A[8] = 0.0;
        double al[3];
        bslices_at<2, 3>(A, root, al);
        if (!(fabs(al[0]) >= 1e-12 || fabs(al[1]) >= 1e-12 || fabs(al[2]) >= 1e-12)) {  // max|a(., v*)| < 1e-12
          complex_job = true;  // a(., v*) == 0: the b fallback runs in the general path kernel
        } else {
          uint32_t nc = 0, nrej = 0;
          double ua[2];
          bool near_double;
          const int nu = quadratic_u_roots_precheck(al, ua, &near_double);
          for (int iu = 0; iu < nu; ++iu) {
            ++nc;
            if (precheck_reject(ua[iu], root))
              ++nrej;
            else
              to_path = true;
          }
          if (near_double) complex_job = true;  // a near-double u-root: the general path kernel probes it (R11)
          if (complex_job)
            to_path = false;
          if (!to_path && !complex_job) {
            cnt[C_CANDIDATES] += nc;
            cnt[C_REJ_DOMAIN] += nrej;
          }
        }
      }
    }
    emit_flag(active && flags != 0, flags, i, S);
    // two-ended dense list: deeper recursions (pair, meta, r) from the back, path entries (pair, root) from the front
    // deep list: deeper recursions, and the rare monotone jobs whose back-substitution needs the b fallback or
    // a c14 probe (the deep kernel re-isolates their single root; the general path kernel finishes them)
    const bool deep = job && (!mono || complex_job);
    uint32_t ex2;
    const unsigned long long b2 = warp_alloc(J.count + 1, deep ? 1u : 0u, &ex2);
    if (deep && b2 + ex2 < J.capacity) {
      const unsigned long long p = J.capacity - 1 - (b2 + ex2);
      J.pair[p] = (uint32_t)i;
      J.meta[p] = meta;
      if (NR % 2 == 0) {  // R: 80 B per job, 16-byte aligned
        double2* r2 = reinterpret_cast<double2*>(J.r + p * NR);
#pragma unroll
        for (int t = 0; t < NR / 2; ++t) r2[t] = make_double2(r[2 * t], r[2 * t + 1]);
      } else {
#pragma unroll
        for (int t = 0; t < NR; ++t) J.r[p * NR + t] = r[t];
      }
    }
    // path entries (pair, root) from the front
#if defined(SPOLY_P1_WARP_BUFFER)
    // per-warp staging in shared memory, flushed 32 at a time with one atomic: no block barrier (the warps'
    // Newton loops end at different times), one global atomic per ~100 pairs
    {
      const unsigned mb = __ballot_sync(0xffffffffu, to_path);
      if (to_path) {
        const int pos = wbuf_n + __popc(mb & ((1u << lane) - 1u));
        s_wpair[warp][pos] = (uint32_t)i;
        s_wroot[warp][pos] = root;
      }
      wbuf_n += __popc(mb);
      __syncwarp();
      if (wbuf_n >= 32) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(J.count, 32ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b + lane < J.capacity) {
          J.pair[b + lane] = s_wpair[warp][lane];
          J.root[b + lane] = s_wroot[warp][lane];
        }
        __syncwarp();
        if (lane < wbuf_n - 32) {
          s_wpair[warp][lane] = s_wpair[warp][32 + lane];
          s_wroot[warp][lane] = s_wroot[warp][32 + lane];
        }
        wbuf_n -= 32;
        __syncwarp();
      }
    }
#else
    {
      // block-aggregated: one atomic per 128 pairs (same-address atomics serialise in L2)
      const unsigned mb = __ballot_sync(0xffffffffu, to_path);
      if (lane == 0) s_off[warp] = __popc(mb);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t c = s_off[w];
          s_off[w] = acc;
          acc += c;
        }
        s_base = acc ? atomicAdd(J.count, (unsigned long long)acc) : 0ull;
      }
      __syncthreads();
      const uint32_t ex1 = s_off[warp] + __popc(mb & ((1u << lane) - 1u));
      const unsigned long long b1 = s_base;
      if (to_path && b1 + ex1 < J.capacity) {
        J.pair[b1 + ex1] = (uint32_t)i;
        J.root[b1 + ex1] = root;
      }
    }
#endif
  }
#if defined(SPOLY_P1_WARP_BUFFER)
  if (wbuf_n > 0) {  // final partial flush
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(J.count, (unsigned long long)wbuf_n);
    b = __shfl_sync(0xffffffffu, b, 0);
    if (lane < wbuf_n && b + lane < J.capacity) {
      J.pair[b + lane] = s_wpair[warp][lane];
      J.root[b + lane] = s_wroot[warp][lane];
    }
  }
#endif
  flush_counters(S, cnt);
}

// reading R2: <= 3 Newton steps on (a, b) from (us, vv), keeping a step only if |F| decreases and the candidate
// stays within 1e-3 of (u0, v0) (local refinement, never a search); returns the final partial derivatives
template <bool TC>
__device__ __forceinline__ void refine_ab(const double* A, const double* B, double u0, double v0, double& us,
                                          double& vv, double& fau, double& fav, double& fbu, double& fbv) {
  constexpr int DB = Sys1<TC>::DB;
  double fa, fb;
  beval<2, 3>(A, us, vv, &fa, &fau, &fav);
  beval<DB, DB + 1>(B, us, vv, &fb, &fbu, &fbv);
  for (int it = 0; it < 3; ++it) {
    const double det = fau * fbv - fav * fbu;
    if (det == 0.0) break;
    const double idet = 1.0 / det;
    const double du = -(fbv * fa - fav * fb) * idet, dv = -(-fbu * fa + fau * fb) * idet;
    // a step below 1e-15 cannot change the double-precision candidate: converged
    if (fmax(fabs(du), fabs(dv)) <= 1e-15 * fmax(1.0, fmax(fabs(us), fabs(vv)))) break;
    if (!(fmax(fabs(us + du - u0), fabs(vv + dv - v0)) <= 1e-3)) break;
    double na, nau, nav, nb, nbu, nbv;
    beval<2, 3>(A, us + du, vv + dv, &na, &nau, &nav);
    beval<DB, DB + 1>(B, us + du, vv + dv, &nb, &nbu, &nbv);
    if (!(na * na + nb * nb < fa * fa + fb * fb)) break;
    us += du;
    vv += dv;
    fa = na; fau = nau; fav = nav;
    fb = nb; fbu = nbu; fbv = nbv;
  }
}

// c14 probe (reading R11): does the near-tangency condition at (u0, v0) sit at an (almost) admissible chain?  The
// candidate is refined like a root, then must lie within kProbeDomain of the triangle with Eq. 3 residual below
// theta_final.  Ghost double roots (the square form's P = Q = 0 points) fail it and raise no flag.
constexpr double kProbeDomain = 1e-3;
template <bool TC>
__device__ __forceinline__ bool probe_admissible(d3 x0, d3 x2, const d3 P_in[3], const d3 N_in[3],
                                                 const SolveParams& prm, const Sys1<TC>& Sys, double u0, double v0) {
  double us = u0, vv = v0, fau, fav, fbu, fbv;
  refine_ab<TC>(Sys.A, Sys.B, u0, v0, us, vv, fau, fav, fbu, fbv);
  const double ur = Sys.relabel ? vv : us, vr_ = Sys.relabel ? us : vv;
  if (!(ur >= -kProbeDomain && vr_ >= -kProbeDomain && ur + vr_ <= 1.0 + kProbeDomain)) return false;
  const d3 x1 = P_in[0] + ur * (P_in[1] - P_in[0]) + vr_ * (P_in[2] - P_in[0]);
  const d3 nx = N_in[0] + ur * (N_in[1] - N_in[0]) + vr_ * (N_in[2] - N_in[0]);
  return vertex_residual(x0, x1, x2, nx, Sys.eta0, Sys.eta1) < prm.theta_final;
}

// candidates u of the back-substitution at v (a(., v); b(., v) when a(., v) == 0, c11), at most 4
template <bool TC>
__device__ __forceinline__ int back_substitute(const Sys1<TC>& Sys, double vs, double* ua, double* udouble,
                                               uint32_t* flags, uint32_t* cnt) {
  constexpr int DB = Sys1<TC>::DB;
  double al[3];
  bslices_at<2, 3>(Sys.A, vs, al);
  *udouble = __longlong_as_double(0x7ff8000000000000ll);
  const double amax = dmax(fabs(al[0]), dmax(fabs(al[1]), fabs(al[2])));
  if (amax >= 1e-12) return quadratic_u_roots(al, ua, udouble);
  // fallback (c11): a(., v*) == 0 -> roots of b(., v*) on [-0.1, 1.1]
  double bl[DB + 1];
  bslices_at<DB, DB + 1>(Sys.B, vs, bl);
  double bmax = 0.0;
  int bd = 0;
#pragma unroll
  for (int i = 0; i <= DB; ++i) {
    bmax = dmax(bmax, fabs(bl[i]));
    if (bl[i] != 0.0) bd = i;
  }
  if (!(bmax >= 1e-12)) {
    *flags |= SPOLY_FLAG_DEGENERATE;
    return 0;
  }
  RootSet<DB + 1> Rb;
  isolate_roots<DB + 1>(bl, bd, -0.1, 1.1, 1e-7, Rb);
  int nu = 0;
  for (int i = 0; i < Rb.n; ++i)
    if (nu == 0 || Rb.x[i] - ua[nu - 1] >= 1e-7) {
      if (nu < 4) {
        ua[nu++] = Rb.x[i];
      } else {  // slot capacity (4 u-roots per v-root): flagged, never silent
        *flags |= SPOLY_FLAG_TRUNCATED;
        cnt[C_TRUNCATED]++;
      }
    }
  return nu;
}

// ---------------------------------------------------------------------------------------------
template <bool TC>
__device__ void path_phase(d3 x0, d3 x2, double intensity, const d3 P_in[3], const d3 N_in[3],
                           const SolveParams& prm, const Sys1<TC>& Sys, const double* vr, int nv, const double* vp,
                           int np, PairOut& out, uint32_t* cnt) {
  const d3 e1o = P_in[1] - P_in[0], e2o = P_in[2] - P_in[0];
  const d3 g_geo = cross(e1o, e2o);
  bool tangent = false;  // a probed near-tangency condition sits at an admissible chain (NEAR_TANGENT)
  for (int iv = 0; iv < nv; ++iv) {
    const double vs = vr[iv];
    double ua[4], ud;
    const int nu = back_substitute<TC>(Sys, vs, ua, &ud, &out.flags, cnt);
    if (!tangent && !isnan(ud)) tangent = probe_admissible<TC>(x0, x2, P_in, N_in, prm, Sys, ud, vs);
    for (int iu = 0; iu < nu; ++iu) {
      cnt[C_CANDIDATES]++;
      double us = ua[iu], vv = vs;
      // reject before refining (identical results, half the path-phase work on C2)
      if (precheck_reject(us, vv)) {
        cnt[C_REJ_DOMAIN]++;
        continue;
      }
      cnt[C_REFINED]++;
      double fau, fav, fbu, fbv;
      refine_ab<TC>(Sys.A, Sys.B, ua[iu], vs, us, vv, fau, fav, fbu, fbv);
      const double ur = Sys.relabel ? vv : us, vr_ = Sys.relabel ? us : vv;  // original labeling
      const d3 x1 = P_in[0] + ur * e1o + vr_ * e2o;
      const d3 nx = N_in[0] + ur * (N_in[1] - N_in[0]) + vr_ * (N_in[2] - N_in[0]);
      const double ed = fmin(fmin(ur, vr_), 1.0 - ur - vr_);
      const bool inside = ur >= -prm.eps_domain && vr_ >= -prm.eps_domain && ur + vr_ <= 1.0 + prm.eps_domain;
      const double rho = vertex_residual(x0, x1, x2, nx, Sys.eta0, Sys.eta1);
      if (!inside) {
        if (ed >= -prm.eps_flag && rho < prm.theta_final && side_ok(TC, x0, x1, x2, nx, g_geo))
          out.flags |= SPOLY_FLAG_BOUNDARY;
        cnt[C_REJ_DOMAIN]++;
        continue;
      }
      if (!(rho < prm.theta_final)) {
        cnt[C_REJ_CONSTRAINT]++;
        continue;
      }
      if (!side_ok(TC, x0, x1, x2, nx, g_geo)) {
        cnt[C_REJ_SIDE]++;
        continue;
      }
      if (rho >= 1e-7) out.flags |= SPOLY_FLAG_RESIDUAL;
      if (ed <= prm.eps_flag) out.flags |= SPOLY_FLAG_BOUNDARY;
      if (fabs(fau * fbv - fav * fbu) < 1e-6 * hypot(fau, fav) * hypot(fbu, fbv)) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
      bool dup = false;  // dedup against accepted chains (1e-7)
      for (int s = 0; s < out.nsol; ++s)
        if (fabs(out.u[s] - ur) < 1e-7 && fabs(out.v[s] - vr_) < 1e-7) dup = true;
      if (dup) {
        cnt[C_REJ_SIDE]++;
        continue;
      }
      if (out.nsol < kMaxSolPerPair) {
        // light-side trace: incoming medium eta_1 (light side), outgoing eta_0
        const double J = jacobian_k1(TC, x0, x2, x1, e1o, e2o, N_in[1] - N_in[0], N_in[2] - N_in[0], nx, Sys.eta1,
                                     Sys.eta0);
        const int s = out.nsol++;
        out.u[s] = ur;
        out.v[s] = vr_;
        out.contrib[s] = J > 0 ? intensity / J : 0.0;
        out.resid[s] = (float)rho;
        out.slot[s] = (uint32_t)(iv * 4 + iu);
        cnt[C_ADMISSIBLE]++;
      } else {  // per-pair capacity: flagged, never silent
        out.flags |= SPOLY_FLAG_TRUNCATED;
        cnt[C_TRUNCATED]++;
      }
    }
  }
  // c14 conditions of the root isolation (deep jobs): close v-roots, tiny critical values (reading R11)
  for (int ip = 0; ip < np && !tangent; ++ip) {
    double ua[4], ud;
    uint32_t fdummy = 0;
    const int nu = back_substitute<TC>(Sys, vp[ip], ua, &ud, &fdummy, cnt);
    for (int iu = 0; iu < nu && !tangent; ++iu) tangent = probe_admissible<TC>(x0, x2, P_in, N_in, prm, Sys, ua[iu], vp[ip]);
  }
  if (tangent) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
}

// ---- phase 2a': jobs with a deeper derivative recursion (~1%), thread per job
template <bool TC>
__global__ void __launch_bounds__(128) k1_roots_deep(SolSink S, JobSink J, uint64_t jcap, SolveParams prm) {
  constexpr int NR = Sys1<TC>::NR;
  uint32_t cnt[C_NUM];
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const uint64_t ndeep = J.count[1];
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = gw * 32; base < ndeep; base += nw * 32) {
    const uint64_t d = base + lane;
    const bool active = d < ndeep;
    const uint64_t jj = active ? jcap - 1 - d : 0;
    uint32_t flags = 0, pair = 0;
    int nv = 0;
    double vr[NR];
    if (active) {
      pair = __ldg(J.pair + jj);
      const uint32_t meta = __ldg(J.meta + jj);
      double r[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) r[i] = __ldg(J.r + jj * NR + i);
      RootSet<NR, true> R;
      isolate_roots<NR, true>(r, (int)(meta >> 8), 0.0, 1.0, prm.eps_flag, R, (int)(meta & 0xFF));
      cnt[C_EVAL_DEEP] += R.terms;
      for (int i = 0; i < R.n; ++i)
        if (nv == 0 || R.x[i] - vr[nv - 1] >= 1e-7) vr[nv++] = R.x[i];
      cnt[C_VROOTS] += nv;
      // [nv | np << 8, roots..., probes...]: the c14 near-tangency conditions go to the path kernel, which probes
      // them (reading R11); probes that do not fit flag the tuple conservatively
      const int np = min(R.nprobe, NR - 1 - nv);
      if (np < R.nprobe) flags |= SPOLY_FLAG_NEAR_TANGENT;
      J.r[jj * NR] = (double)(nv | (np << 8));
      for (int i = 0; i < nv; ++i) J.r[jj * NR + 1 + i] = vr[i];
      for (int i = 0; i < np; ++i) J.r[jj * NR + 1 + nv + i] = R.probe[i];
    }
    emit_flag(active && flags != 0, flags, pair, S);
  }
  flush_counters(S, cnt);
}

// ---- phase 2b: back-substitution, refinement, validation, contribution, emission; thread per job of the
// pre-pass list, then the deep jobs (jobs without roots exit at once)
template <bool TC>
__global__ void SPOLY_PATH_BOUNDS k1_path(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                               const TriRec* __restrict__ tris, const double* __restrict__ ep,
                                               const double* __restrict__ inten, SolveParams prm, SolSink S,
                                               JobSink J) {
  constexpr int NR = Sys1<TC>::NR;
  uint32_t cnt[C_NUM];
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const uint64_t nl = 0, n = J.count[1];  // deep entries only (the path entries run in k1_path_fast)
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = gw * 32; base < n; base += nw * 32) {
    const uint64_t i = base + lane;
    const uint64_t jj = i < nl ? i : J.capacity - 1 - (i - nl);
    // front: (pair, root) of phase 1's surviving monotone jobs; back: deep jobs, [nv | np << 8, roots..., probes...]
    const double r0 = i < nl ? J.root[jj] : 0.0;
    const int hdr = i < nl ? 1 : (i < n ? (int)J.r[jj * NR] : 0);
    const int nv = hdr & 0xFF, np = hdr >> 8;
    const bool active = nv > 0 || np > 0;
    PairOut o;
    o.nsol = 0;
    o.flags = 0;
    uint32_t pair = 0;
    if (active) {
      pair = __ldg(J.pair + jj);
      double vr[NR], vp[NR];
      if (i < nl) {
        vr[0] = r0;
      } else {
        for (int k = 0; k < nv; ++k) vr[k] = J.r[jj * NR + 1 + k];
        for (int k = 0; k < np; ++k) vp[k] = J.r[jj * NR + 1 + nv + k];
      }
      d3 P[3], N[3], x0, x2;
      uint32_t q;
      load_pair(pq, pt, tris, ep, pair, P, N, x0, x2, q);
      Sys1<TC> Sys;
      build_system<TC>(x0, x2, P, N, prm, Sys);  // bit-identical to phase 1 (known non-degenerate)
      cnt[C_REBUILDS]++;
      const double I = inten ? __ldg(inten + q) : 1.0;
      path_phase<TC>(x0, x2, I, P, N, prm, Sys, vr, nv, vp, np, o, cnt);
    }
    emit_flag(active && o.flags != 0, o.flags, pair, S);
    uint32_t ex;
    const unsigned long long b = warp_alloc(S.count, active ? (uint32_t)o.nsol : 0u, &ex);
    for (int s = 0; s < o.nsol; ++s) {
      const unsigned long long p = b + ex + s;
      if (p < S.capacity) {
        S.key[p] = ((unsigned long long)pair << 6) | o.slot[s];
        S.bary[2 * p] = o.u[s];
        S.bary[2 * p + 1] = o.v[s];
        S.contrib[p] = o.contrib[s];
        S.resid[p] = o.resid[s];
      }
    }
  }
  flush_counters(S, cnt);
}

// ---- phase 2c: the common case, thread per path entry (pair, root) of phase 1: the quadratic back-substitution
// (<= 2 candidates, no b fallback, no c14 probe: phase 1 routed those jobs to the deep list), (a, b) refinement
// (reading R2), Eq. 3 validation, sides, flags, analytic contribution (c15), <= 2 chains emitted with
// warp-aggregated appends.  Same arithmetic and slots as path_phase(), with the lean state of one root.
#ifndef SPOLY_FAST_MINB
#define SPOLY_FAST_MINB 4  // <= 128 registers (A/B: 222 unbounded -> 1.59, 128 -> 1.54 ms on C2)
#endif
#define SPOLY_FAST_BOUNDS __launch_bounds__(128, SPOLY_FAST_MINB)
#ifdef SPOLY_PROF_FAST  // section clocks of k1_path_fast (lane 0 of each warp; diagnostic only)
__device__ unsigned long long g_fprof[8];
#define FPROF_INIT long long fprof_t = clock64();
#define FPROF(k)                                                                          \
  do {                                                                                    \
    const long long fprof_n = clock64();                                                  \
    if (lane == 0) atomicAdd(&g_fprof[k], (unsigned long long)(fprof_n - fprof_t));        \
    fprof_t = fprof_n;                                                                    \
  } while (0)
#else
#define FPROF_INIT
#define FPROF(k)
#endif
template <bool TC>
__global__ void SPOLY_FAST_BOUNDS k1_path_fast(const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                                    const TriRec* __restrict__ tris, const double* __restrict__ ep,
                                                    const double* __restrict__ inten, SolveParams prm, SolSink S,
                                                    JobSink J) {
  uint32_t cnt[C_NUM];
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const uint64_t n = J.count[0];
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  FPROF_INIT
  for (uint64_t base = gw * 32; base < n; base += nw * 32) {
    const uint64_t i = base + lane;
    const bool active = i < n;
    uint32_t flags = 0, pair = 0;
    int nsol = 0;
    double su[2], sv[2], sc[2];
    float sr[2];
    uint32_t ss[2];
    if (active) {
      pair = __ldg(J.pair + i);
      const double vs = __ldg(J.root + i);
      d3 P[3], N[3], x0, x2;
      uint32_t q;
      load_pair(pq, pt, tris, ep, pair, P, N, x0, x2, q);
      Sys1<TC> Sys;
      build_system<TC>(x0, x2, P, N, prm, Sys);  // bit-identical to phase 1 (known non-degenerate)
      FPROF(0);
      cnt[C_REBUILDS]++;
      const double I = inten ? __ldg(inten + q) : 1.0;
      const d3 e1o = P[1] - P[0], e2o = P[2] - P[0];
      const d3 g_geo = cross(e1o, e2o);
      double al[3], ua[2], ud;
      bslices_at<2, 3>(Sys.A, vs, al);
      const int nu = quadratic_u_roots(al, ua, &ud);
      for (int iu = 0; iu < nu; ++iu) {
        cnt[C_CANDIDATES]++;
        double us = ua[iu], vv = vs;
        if (precheck_reject(us, vv)) {
          cnt[C_REJ_DOMAIN]++;
          continue;
        }
        cnt[C_REFINED]++;
        FPROF(1);
        double fau, fav, fbu, fbv;
        refine_ab<TC>(Sys.A, Sys.B, ua[iu], vs, us, vv, fau, fav, fbu, fbv);
        FPROF(2);
        const double ur = Sys.relabel ? vv : us, vr_ = Sys.relabel ? us : vv;  // original labeling
        const d3 x1 = P[0] + ur * e1o + vr_ * e2o;
        const d3 nx = N[0] + ur * (N[1] - N[0]) + vr_ * (N[2] - N[0]);
        const double ed = fmin(fmin(ur, vr_), 1.0 - ur - vr_);
        const bool inside = ur >= -prm.eps_domain && vr_ >= -prm.eps_domain && ur + vr_ <= 1.0 + prm.eps_domain;
        const double rho = vertex_residual(x0, x1, x2, nx, Sys.eta0, Sys.eta1);
        if (!inside) {
          if (ed >= -prm.eps_flag && rho < prm.theta_final && side_ok(TC, x0, x1, x2, nx, g_geo))
            flags |= SPOLY_FLAG_BOUNDARY;
          cnt[C_REJ_DOMAIN]++;
          continue;
        }
        if (!(rho < prm.theta_final)) {
          cnt[C_REJ_CONSTRAINT]++;
          continue;
        }
        if (!side_ok(TC, x0, x1, x2, nx, g_geo)) {
          cnt[C_REJ_SIDE]++;
          continue;
        }
        if (rho >= 1e-7) flags |= SPOLY_FLAG_RESIDUAL;
        if (ed <= prm.eps_flag) flags |= SPOLY_FLAG_BOUNDARY;
        if (fabs(fau * fbv - fav * fbu) < 1e-6 * hypot(fau, fav) * hypot(fbu, fbv)) flags |= SPOLY_FLAG_NEAR_TANGENT;
        if (nsol == 1 && fabs(su[0] - ur) < 1e-7 && fabs(sv[0] - vr_) < 1e-7) {  // dedup (1e-7)
          cnt[C_REJ_SIDE]++;
          continue;
        }
        FPROF(3);
        const double J1 = jacobian_k1(TC, x0, x2, x1, e1o, e2o, N[1] - N[0], N[2] - N[0], nx, Sys.eta1, Sys.eta0);
        FPROF(4);
        su[nsol] = ur;
        sv[nsol] = vr_;
        sc[nsol] = J1 > 0 ? I / J1 : 0.0;
        sr[nsol] = (float)rho;
        ss[nsol] = (uint32_t)iu;  // slot iv * 4 + iu with iv = 0
        nsol++;
        cnt[C_ADMISSIBLE]++;
      }
    }
    FPROF(5);
    emit_flag(active && flags != 0, flags, pair, S);
    uint32_t ex;
    const unsigned long long b = warp_alloc(S.count, (uint32_t)nsol, &ex);
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const unsigned long long p = b + ex + s2;
      if (s2 < nsol && p < S.capacity) {
        S.key[p] = ((unsigned long long)pair << 6) | ss[s2];
        S.bary[2 * p] = su[s2];
        S.bary[2 * p + 1] = sv[s2];
        S.contrib[p] = sc[s2];
        S.resid[p] = sr[s2];
      }
    }
    FPROF(6);
  }
  flush_counters(S, cnt);
}

void launch_solve_k1(int phase, int refract, const uint32_t* pq, const uint32_t* pt, uint64_t npairs,
                     const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                     const SolSink& S, const JobSink& J, int nsm, cudaStream_t st) {
  if (npairs == 0) return;
  const int threads = 128;
#ifndef SPOLY_P1_GRID
#define SPOLY_P1_GRID 64  // blocks per SM (grid-stride); A/B on C2: 4 -> 2.22, 16 -> 2.15, 64 -> 2.07, 256 -> 2.20 ms
#endif
  const uint64_t cap1 = (uint64_t)nsm * SPOLY_P1_GRID;
  const uint64_t want1 = (npairs + threads - 1) / threads;
  const int g1 = (int)(want1 < cap1 ? want1 : cap1);
  if (phase == 1) {
    if (refract)
      k1_phase1<true><<<g1, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, prm, S, J);
    else
      k1_phase1<false><<<g1, threads, 0, st>>>(pq, pt, npairs, M.tris, ep, prm, S, J);
  } else if (phase == 2) {  // deep jobs (derivative recursion below level 1, ~1% of the jobs)
    if (refract)
      k1_roots_deep<true><<<nsm * 2, threads, 0, st>>>(S, J, J.capacity, prm);
    else
      k1_roots_deep<false><<<nsm * 2, threads, 0, st>>>(S, J, J.capacity, prm);
  } else {  // path
#ifndef SPOLY_PATH_GRID
#define SPOLY_PATH_GRID 4  // blocks per SM (2 resident at 243 registers); A/B: 16 -> 4 took k1_path<R> 2.04 -> 2.03 ms, <T> 0.167 -> 0.155 ms
#endif
#ifndef SPOLY_FAST_GRID
#define SPOLY_FAST_GRID 8
#endif
    if (refract) {
      k1_path_fast<true><<<nsm * SPOLY_FAST_GRID, threads, 0, st>>>(pq, pt, M.tris, ep, inten, prm, S, J);
      k1_path<true><<<nsm * SPOLY_PATH_GRID, threads, 0, st>>>(pq, pt, M.tris, ep, inten, prm, S, J);
    } else {
      k1_path_fast<false><<<nsm * SPOLY_FAST_GRID, threads, 0, st>>>(pq, pt, M.tris, ep, inten, prm, S, J);
      k1_path<false><<<nsm * SPOLY_PATH_GRID, threads, 0, st>>>(pq, pt, M.tris, ep, inten, prm, S, J);
    }
#ifdef SPOLY_PROF_FAST
    unsigned long long h[8];
    cudaStreamSynchronize(st);
    if (cudaMemcpyFromSymbol(h, g_fprof, sizeof(h)) == cudaSuccess) {
      fprintf(stderr, "k1_path_fast section clocks (cumulative, lane 0):");
      for (int k = 0; k < 7; ++k) fprintf(stderr, " %d:%.3e", k, (double)h[k]);
      fprintf(stderr, "\n");
    }
#endif
  }
}

}  // namespace spoly
