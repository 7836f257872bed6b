// Culling pre-pass (replaces the Wang20 pruning of PAPER.md:680).
//
// Predicate (sound): any admissible x_1 on T has a generalised half vector
//   h = eta_prev w_prev + eta_next w_next  parallel to +-n(x_1)            (Eq. 3)
// where w_prev / w_next are the unit directions from x_1 to x_0 / x_2.  Each direction set is bounded
// by a cone (axis a, chord c = 2 sin(theta/2)); h then lies in the ball B(A, r), A = sum eta a,
// r = sum eta c, i.e. in the cone (A^, asin(r/|A|)) when |A| > r.  The tuple is culled when that cone
// misses both the normal cone and its negation by more than `margin`.  Cluster level: bounding
// sphere + cluster normal cone; triangle level: exact vertex-direction cones + the triangle's normal
// cone.  FP32 with a margin: at most more permissive than the FP64 oracle predicate.
//
// One warp per query (grid-stride).  pass 0 counts survivors per query; pass 1 rewrites the same
// decisions into the query-major work list at the scanned offsets (deterministic order: Morton
// position ascending).
#include "kernels.cuh"

namespace spoly {

struct DirCone {
  f3 a;
  float chord;
  bool ok;
};

__device__ __forceinline__ f3 nrmz(f3 v) {
  float l = rsqrtf(dotf(v, v));
  return l * v;
}

// cone of the directions from the three vertices to x
__device__ __forceinline__ DirCone tri_dir_cone(f3 x, f3 p0, f3 p1, f3 p2) {
  f3 w0 = nrmz(x - p0), w1 = nrmz(x - p1), w2 = nrmz(x - p2);
  f3 s = w0 + w1 + w2;
  f3 a = nrmz(s);
  DirCone c;
  c.a = a;
  f3 d0 = w0 - a, d1 = w1 - a, d2 = w2 - a;
  c.chord = sqrtf(fmaxf(dotf(d0, d0), fmaxf(dotf(d1, d1), dotf(d2, d2))));
  // all directions within 90 deg of the axis (chord < sqrt 2) -> the cone bounds their spherical hull
  c.ok = dotf(w0, a) > 1e-3f && dotf(w1, a) > 1e-3f && dotf(w2, a) > 1e-3f;
  return c;
}

// cone of the directions from a sphere (c, rho) to x
__device__ __forceinline__ DirCone sphere_dir_cone(f3 x, f3 c, float rho) {
  f3 d = x - c;
  float l2 = dotf(d, d);
  DirCone r;
  r.a = rsqrtf(l2) * d;
  float s2 = rho * rho / l2;  // sin^2 theta
  r.ok = s2 < 0.98f;
  float ct = sqrtf(fmaxf(1.f - s2, 0.f));
  r.chord = sqrtf(2.f * s2 / (1.f + ct));  // 2 sin(theta/2)
  return r;
}

// keep test against the normal cone (axis nax, half angle nth), both orientations
__device__ __forceinline__ bool cone_keep(const DirCone& p, const DirCone& q, float ep, float en, f3 nax, float nth,
                                          float margin) {
  if (!p.ok || !q.ok || nth >= 1.5707f) return true;
  f3 A = ep * p.a + en * q.a;
  float r = ep * p.chord + en * q.chord;
  float An = sqrtf(dotf(A, A));
  if (!(An > r * 1.0001f + 1e-6f)) return true;
  float alpha = asinf(fminf(r / An, 1.f));
  float beta = alpha + nth + margin;
  if (beta >= 1.5707f) return true;
  f3 cr = crossf(A, nax);
  float phi = atan2f(sqrtf(dotf(cr, cr)), dotf(A, nax));
  return phi <= beta || (3.14159265f - phi) <= beta;
}

__device__ __forceinline__ f3 ld3(float4 a) { return {a.x, a.y, a.z}; }

__global__ void __launch_bounds__(256) k_cull_k1(int pass, const double* __restrict__ ep, uint32_t nq,
                                                 const TriRec* __restrict__ tris, const float4* __restrict__ tricone,
                                                 const ClusterRec* __restrict__ cl, uint32_t ntris, uint32_t ncl,
                                                 CullParams cp, uint32_t* counts,
                                                 const unsigned long long* __restrict__ offsets,
                                                 uint32_t* pair_query, uint32_t* pair_tpos) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = gw; q < nq; q += nw) {
    const double* e = ep + 6ull * q;
    const f3 x0 = {(float)e[0], (float)e[1], (float)e[2]};
    const f3 x2 = {(float)e[3], (float)e[4], (float)e[5]};
    uint32_t count = 0;
    unsigned long long wpos = pass ? offsets[q] : 0ull;
    for (uint32_t cb = 0; cb < ncl; cb += 32) {
      const uint32_t c = cb + lane;
      bool keep = false;
      if (c < ncl) {
        const ClusterRec R = cl[c];
        const f3 cc = ld3(R.sphere);
        DirCone dp = sphere_dir_cone(x0, cc, R.sphere.w), dn = sphere_dir_cone(x2, cc, R.sphere.w);
        const f3 nax = ld3(R.cone);
        if (cp.refract)
          keep = cone_keep(dp, dn, cp.eta_front, cp.eta_back, nax, R.cone.w, cp.margin) ||
                 cone_keep(dp, dn, cp.eta_back, cp.eta_front, nax, R.cone.w, cp.margin);
        else
          keep = cone_keep(dp, dn, 1.f, 1.f, nax, R.cone.w, cp.margin);
      }
      unsigned cmask = __ballot_sync(0xffffffffu, keep);
      while (cmask) {
        const int b = __ffs(cmask) - 1;
        cmask &= cmask - 1;
        const uint32_t cid = cb + b;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t t = cid * kClusterSize + half * 32 + lane;
          bool k = false;
          if (t < ntris) {
            const float4* r = tris[t].r;
            float4 a = __ldg(r), bb = __ldg(r + 1), c2 = __ldg(r + 2);
            f3 p0 = {a.x, a.y, a.z}, p1 = {a.w, bb.x, bb.y}, p2 = {bb.z, bb.w, c2.x};
            float4 nc = __ldg(tricone + t);
            DirCone dp = tri_dir_cone(x0, p0, p1, p2), dn = tri_dir_cone(x2, p0, p1, p2);
            float e0 = 1.f, e1 = 1.f;
            if (cp.refract) {
              f3 g = crossf(p1 - p0, p2 - p0);
              bool front = dotf(x0 - p0, g) > 0.f;
              e0 = front ? cp.eta_front : cp.eta_back;
              e1 = front ? cp.eta_back : cp.eta_front;
              // a side decision within float noise of the plane: test both media
              float dd = dotf(x0 - p0, g), gl = sqrtf(dotf(g, g)), xl = sqrtf(dotf(x0 - p0, x0 - p0));
              if (fabsf(dd) <= 1e-4f * gl * xl)
                k = cone_keep(dp, dn, e1, e0, ld3(nc), nc.w, cp.margin);
            }
            k = k || cone_keep(dp, dn, e0, e1, ld3(nc), nc.w, cp.margin);
          }
          const unsigned m = __ballot_sync(0xffffffffu, k);
          if (pass && k) {
            const unsigned long long pos = wpos + __popc(m & ((1u << lane) - 1u));
            pair_query[pos] = q;
            pair_tpos[pos] = t;
          }
          wpos += __popc(m);
          count += __popc(m);
        }
      }
    }
    if (!pass && lane == 0) counts[q] = count;
  }
}

void launch_cull_k1(int pass, const double* ep, uint32_t nq, const DeviceMesh& M, const CullParams& cp,
                    uint32_t* counts, const unsigned long long* offsets, uint32_t* pair_query, uint32_t* pair_tpos,
                    int nsm, cudaStream_t st) {
  if (!nq) return;
  const int threads = 256;
  uint64_t want = ((uint64_t)nq * 32 + threads - 1) / threads;
  uint64_t cap = (uint64_t)nsm * 8;
  int blocks = (int)(want < cap ? want : cap);
  k_cull_k1<<<blocks, threads, 0, st>>>(pass, ep, nq, M.tris, M.tricone, M.clusters, M.ntris, M.nclusters, cp, counts,
                                        offsets, pair_query, pair_tpos);
}

// no cull: every (query, triangle) pair, query-major, Morton order
__global__ void k_all_pairs(uint32_t nq, uint32_t ntris, uint32_t* pq, uint32_t* pt) {
  const uint64_t n = (uint64_t)nq * ntris;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    pq[i] = (uint32_t)(i / ntris);
    pt[i] = (uint32_t)(i % ntris);
  }
}
void launch_all_pairs_k1(uint32_t nq, uint32_t ntris, uint32_t* pair_query, uint32_t* pair_tpos, cudaStream_t st) {
  k_all_pairs<<<1024, 256, 0, st>>>(nq, ntris, pair_query, pair_tpos);
}

// explicit CSR tuple list (original ids) -> work list (Morton positions); one warp per query
__global__ void k_expand_list(const uint32_t* __restrict__ off, const uint32_t* __restrict__ ids, uint32_t nq, int k,
                              const uint32_t* __restrict__ perm_of, uint32_t* pq, uint32_t* pt) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = gw; q < nq; q += nw) {
    for (uint32_t i = off[q] + lane; i < off[q + 1]; i += 32) {
      pq[i] = q;
      for (int j = 0; j < k; ++j) pt[(uint64_t)k * i + j] = perm_of[ids[(uint64_t)k * i + j]];
    }
  }
}
void launch_expand_list(const uint32_t* offsets, const uint32_t* tri_ids, uint32_t nq, int k, const uint32_t* perm_of,
                        uint32_t* pair_query, uint32_t* pair_tpos, int nsm, cudaStream_t st) {
  if (!nq) return;
  k_expand_list<<<nsm * 8, 256, 0, st>>>(offsets, tri_ids, nq, k, perm_of, pair_query, pair_tpos);
}

}  // namespace spoly
