// One-bounce fused solve kernels (chain "R" now; "T" shares the path phase).
#include "kernels.cuh"
#include "solve_k1.cuh"

namespace spoly {

// ---------------------------------------------------------------------------------------------
// Solve one (query, triangle) pair of a one-bounce reflection chain (Eq. 21).  All decisions follow
// the readings in DESIGN.md §3 (t choice, truncation, flags) so that the oracle takes the same ones.
__device__ void solve_pair_R(d3 x0, d3 x2, double intensity, const d3 P_in[3], const d3 N_in[3],
                             const SolveParams& prm, PairOut& out, uint32_t* cnt) {
  out.nsol = 0;
  out.flags = 0;
  cnt[C_PAIRS]++;
  // ---- decision (reading R1): incidence-plane normal l_c = (x2 - x0) x n(centroid)
  d3 nc = (1.0 / 3.0) * (N_in[0] + N_in[1] + N_in[2]);
  d3 lc = cross(x2 - x0, nc);
  const double ln = norm(lc);
  if (!(ln > 1e-12 * norm(x2 - x0) * norm(nc))) out.flags |= SPOLY_FLAG_DEGENERATE;
  d3 e1o = P_in[1] - P_in[0], e2o = P_in[2] - P_in[0];
  bool relabel = false;
  if (ln > 0) {
    double s1 = fabs(dot(e1o, lc)) / (norm(e1o) * ln), s2 = fabs(dot(e2o, lc)) / (norm(e2o) * ln);
    relabel = s1 < s2;
  }
  const d3 p0 = P_in[0], p1 = relabel ? P_in[2] : P_in[1], p2 = relabel ? P_in[1] : P_in[2];
  const d3 n0 = N_in[0], n1 = relabel ? N_in[2] : N_in[1], n2 = relabel ? N_in[1] : N_in[2];
  const d3 e1 = p1 - p0, e2 = p2 - p0, m1 = n1 - n0, m2 = n2 - n0;
  const d3 q = p0 - x0, w = x2 - x0;

  // ---- coefficient phase
  double A[9], B[25];
  build_a(q, w, e1, e2, n0, m1, m2, A);
  build_b_R(q, w, e1, e2, n0, m1, m2, B);
  const double ma = bmaxabs<2, 3>(A), mb = bmaxabs<4, 5>(B);
  if (!(ma > 0) || !(mb > 0)) {
    out.flags |= SPOLY_FLAG_DEGENERATE;
    cnt[C_FLAGGED]++;
    return;
  }
  bscale<2, 3>(A, 1.0 / ma);
  bscale<4, 5>(B, 1.0 / mb);
  const int da = bnum_udeg<2, 3>(A, prm.tau_trunc), db = bnum_udeg<4, 5>(B, prm.tau_trunc);
  btrunc_u<2, 3>(A, da);
  btrunc_u<4, 5>(B, db);
  const int n = max(da, db);
  if (n == 0) {
    out.flags |= SPOLY_FLAG_DEGENERATE;
    cnt[C_FLAGGED]++;
    return;
  }
  cnt[C_SYSTEMS]++;

  // ---- elimination phase: r(v) = det R(v), Laplace expansion (deg <= 9)
  double r[10];
  det_R(A, B, n, r);
  double mr = 0.0;
#pragma unroll
  for (int i = 0; i < 10; ++i) mr = fmax(mr, fabs(r[i]));
  if (!(mr > 0)) {
    out.flags |= SPOLY_FLAG_DEGENERATE;
    cnt[C_FLAGGED]++;
    return;
  }
  int deg = 0;
  const double inv = 1.0 / mr;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    r[i] *= inv;
    if (r[i] != 0.0) deg = i;
  }

  // ---- univariate roots on [0,1]
  RootSet<10> R;
  isolate_roots<10>(r, deg, 0.0, 1.0, prm.eps_flag, R);
  cnt[C_EVAL_TERMS] += R.terms;
  if (R.flags & 1) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
  if (R.min_crit_ratio <= 1e-10) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
  // dedup (1e-7) as the oracle
  double vr[10];
  int nv = 0;
  for (int i = 0; i < R.n; ++i)
    if (nv == 0 || R.x[i] - vr[nv - 1] >= 1e-7) vr[nv++] = R.x[i];
  cnt[C_VROOTS] += nv;

  const d3 g_geo = cross(e1o, e2o);
  // ---- path phase
  for (int iv = 0; iv < nv; ++iv) {
    const double vs = vr[iv];
    double al[3];
    bslices_at<2, 3>(A, vs, al);
    double ua[4];
    int nu = 0;
    double amax = fmax(fabs(al[0]), fmax(fabs(al[1]), fabs(al[2])));
    if (amax >= 1e-12) {
      // quadratic / linear in u (stable formula, disc clamp; reading R4)
      if (al[2] != 0.0) {
        const double a0 = al[0], a1 = al[1], a2 = al[2];
        double disc = a1 * a1 - 4.0 * a2 * a0, sc = a1 * a1 + 4.0 * fabs(a2 * a0);
        if (fabs(disc) <= 1e-8 * sc) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
        if (!(disc < -1e-12 * sc)) {
          if (disc < 0) disc = 0;
          double qq = -0.5 * (a1 + copysign(sqrt(disc), a1));
          if (qq == 0.0) {
            ua[nu++] = 0.0;
          } else {
            double r1 = qq / a2, r2 = a0 / qq;
            if (r1 > r2) {
              double t = r1;
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
    } else {
      // fallback (c11): a(., v*) == 0 -> roots of b(., v*) on [-0.1, 1.1]
      double bl[5];
      bslices_at<4, 5>(B, vs, bl);
      double bmax = 0.0;
      int bd = 0;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        bmax = fmax(bmax, fabs(bl[i]));
        if (bl[i] != 0.0) bd = i;
      }
      if (!(bmax >= 1e-12)) {
        out.flags |= SPOLY_FLAG_DEGENERATE;
        continue;
      }
      double bc[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) bc[i] = bl[i];
      RootSet<5> Rb;
      isolate_roots<5>(bc, bd, -0.1, 1.1, 1e-7, Rb);
      for (int i = 0; i < Rb.n && nu < 4; ++i)
        if (nu == 0 || Rb.x[i] - ua[nu - 1] >= 1e-7) ua[nu++] = Rb.x[i];
    }
    for (int iu = 0; iu < nu; ++iu) {
      cnt[C_CANDIDATES]++;
      double us = ua[iu], vv = vs;
      // reading R2: <= 3 Newton steps on (a, b), keep a step only if |F| decreases and the candidate
      // stays within 1e-3 of its back-substituted position (local refinement, never a search)
      double fa, fau, fav, fb, fbu, fbv;
      beval<2, 3>(A, us, vv, &fa, &fau, &fav);
      beval<4, 5>(B, us, vv, &fb, &fbu, &fbv);
      for (int it = 0; it < 3; ++it) {
        double det = fau * fbv - fav * fbu;
        if (det == 0.0) break;
        double du = -(fbv * fa - fav * fb) / det, dv = -(-fbu * fa + fau * fb) / det;
        if (!(fmax(fabs(us + du - ua[iu]), fabs(vv + dv - vs)) <= 1e-3)) break;
        double na, nau, nav, nb, nbu, nbv;
        beval<2, 3>(A, us + du, vv + dv, &na, &nau, &nav);
        beval<4, 5>(B, us + du, vv + dv, &nb, &nbu, &nbv);
        if (!(hypot(na, nb) < hypot(fa, fb))) break;
        us += du;
        vv += dv;
        fa = na; fau = nau; fav = nav;
        fb = nb; fbu = nbu; fbv = nbv;
      }
      const double ur = relabel ? vv : us, vr_ = relabel ? us : vv;  // original labeling
      const d3 x1 = P_in[0] + ur * e1o + vr_ * e2o;
      const d3 nx = N_in[0] + ur * (N_in[1] - N_in[0]) + vr_ * (N_in[2] - N_in[0]);
      const double ed = fmin(fmin(ur, vr_), 1.0 - ur - vr_);
      const bool inside = ur >= -prm.eps_domain && vr_ >= -prm.eps_domain && ur + vr_ <= 1.0 + prm.eps_domain;
      const double rho = vertex_residual(x0, x1, x2, nx, 1.0, 1.0);
      if (!inside) {
        if (ed >= -prm.eps_flag && rho < prm.theta_final && side_ok(false, x0, x1, x2, nx, g_geo))
          out.flags |= SPOLY_FLAG_BOUNDARY;
        cnt[C_REJ_DOMAIN]++;
        continue;
      }
      if (!(rho < prm.theta_final)) {
        cnt[C_REJ_CONSTRAINT]++;
        continue;
      }
      if (!side_ok(false, x0, x1, x2, nx, g_geo)) {
        cnt[C_REJ_SIDE]++;
        continue;
      }
      if (rho >= 1e-7) out.flags |= SPOLY_FLAG_RESIDUAL;
      if (ed <= prm.eps_flag) out.flags |= SPOLY_FLAG_BOUNDARY;
      if (fabs(fau * fbv - fav * fbu) < 1e-6 * hypot(fau, fav) * hypot(fbu, fbv)) out.flags |= SPOLY_FLAG_NEAR_TANGENT;
      // dedup against accepted chains (1e-7)
      bool dup = false;
      for (int s = 0; s < out.nsol; ++s)
        if (fabs(out.u[s] - ur) < 1e-7 && fabs(out.v[s] - vr_) < 1e-7) dup = true;
      if (dup) {
        cnt[C_REJ_SIDE]++;
        continue;
      }
      if (out.nsol < kMaxSolPerPair) {
        const double J = jacobian_k1(false, x0, x2, x1, e1o, e2o, N_in[1] - N_in[0], N_in[2] - N_in[0], nx, 1.0, 1.0);
        const int s = out.nsol++;
        out.u[s] = ur;
        out.v[s] = vr_;
        out.contrib[s] = J > 0 ? intensity / J : 0.0;
        out.resid[s] = (float)rho;
        out.slot[s] = (uint32_t)(iv * 4 + iu);
        cnt[C_ADMISSIBLE]++;
      }
    }
  }
  if (out.flags) cnt[C_FLAGGED]++;
}

// ---------------------------------------------------------------------------------------------
// warp-aggregated emission of the pair results (all 32 lanes must call)
__device__ __forceinline__ void emit_k1(const PairOut& o, bool active, uint32_t q, uint32_t orig, uint64_t pair_idx,
                                        const SolSink& S) {
  const int lane = threadIdx.x & 31;
  const uint32_t n = active ? (uint32_t)o.nsol : 0u;
  uint32_t incl = n;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total) {
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(S.count, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    unsigned long long pos = base + incl - n;
    for (uint32_t s = 0; s < n; ++s, ++pos) {
      if (pos < S.capacity) {
        S.key[pos] = ((unsigned long long)pair_idx << 6) | o.slot[s];
        S.query[pos] = q;
        S.tuple[pos] = orig;
        S.bary[2 * pos] = o.u[s];
        S.bary[2 * pos + 1] = o.v[s];
        S.contrib[pos] = o.contrib[s];
        S.resid[pos] = o.resid[s];
        S.flags[pos] = o.flags;
      }
    }
  }
  const bool fl = active && o.flags != 0;
  const unsigned bal = __ballot_sync(0xffffffffu, fl);
  if (bal) {
    unsigned long long fbase = 0;
    const int leader = __ffs(bal) - 1;
    if (lane == leader) fbase = atomicAdd(S.fcount, (unsigned long long)__popc(bal));
    fbase = __shfl_sync(0xffffffffu, fbase, leader);
    if (fl) {
      unsigned long long pos = fbase + __popc(bal & ((1u << lane) - 1u));
      if (pos < S.fcapacity) {
        S.fkey[pos] = pair_idx;
        S.fquery[pos] = q;
        S.ftuple[pos] = orig;
        S.fflags[pos] = o.flags;
      }
    }
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

// Flat work list: pair i = (pair_query[i], pair_tpos[i]) with tpos a Morton position; all lanes of a
// warp iterate the same number of times so the emission stays warp-synchronous.
__global__ void __launch_bounds__(128) k_solve_R_list(const uint32_t* __restrict__ pair_query,
                                                      const uint32_t* __restrict__ pair_tpos, uint64_t npairs,
                                                      uint64_t pair_base, const TriRec* __restrict__ tris,
                                                      const uint32_t* __restrict__ orig_id,
                                                      const double* __restrict__ ep, const double* __restrict__ inten,
                                                      SolveParams prm, SolSink S) {
  uint32_t cnt[C_NUM];
#pragma unroll
  for (int i = 0; i < C_NUM; ++i) cnt[i] = 0;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = gw * 32; base < npairs; base += nw * 32) {
    const uint64_t i = base + lane;
    const bool active = i < npairs;
    PairOut o;
    o.nsol = 0;
    o.flags = 0;
    uint32_t q = 0, orig = 0;
    if (active) {
      q = __ldg(pair_query + i);
      const uint32_t tp = __ldg(pair_tpos + i);
      orig = __ldg(orig_id + tp);
      d3 P[3], N[3];
      load_tri(tris, tp, P, N);
      const double* e = ep + 6ull * q;
      d3 x0 = mk3(__ldg(e), __ldg(e + 1), __ldg(e + 2)), x2 = mk3(__ldg(e + 3), __ldg(e + 4), __ldg(e + 5));
      const double I = inten ? __ldg(inten + q) : 1.0;
      solve_pair_R(x0, x2, I, P, N, prm, o, cnt);
    }
    emit_k1(o, active, q, orig, pair_base + i, S);
  }
  flush_counters(S, cnt);
}

void launch_solve_R_list(const uint32_t* pq, const uint32_t* pt, uint64_t npairs, uint64_t pair_base,
                         const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                         const SolSink& S, int nsm, cudaStream_t st) {
  if (npairs == 0) return;
  const int threads = 128;
  uint64_t want = (npairs + threads - 1) / threads;
  uint64_t cap = (uint64_t)nsm * 16;  // persistent-ish grid: 16 CTAs of 4 warps per SM
  int blocks = (int)(want < cap ? want : cap);
  k_solve_R_list<<<blocks, threads, 0, st>>>(pq, pt, npairs, pair_base, M.tris, M.orig_id, ep, inten, prm, S);
}

}  // namespace spoly
