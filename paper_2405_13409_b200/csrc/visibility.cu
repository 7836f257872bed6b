// Visibility test of the path phase (Sec. 5.3: "An admissible path will be rejected when the ray from
// any vertex x_i towards the next vertex x_{i+1} is blocked").
//
// Scene = the specular mesh (every triangle occludes) + an optional occluder-only mesh.  Each is indexed by an
// implicit 8-ary AABB hierarchy over its Morton-ordered triangles (level l node i covers triangles
// [i 8^l, (i + 1) 8^l)): boxes are exact float32 min/max of float32 vertices.  One thread per admissible chain
// walks the k + 1 segments x_i -> x_{i+1} through both hierarchies (FP64 slab tests, a small explicit stack) and
// tests the leaf triangles with Moller-Trumbore in FP64: a hit iff t in (1e-7, 1 - 1e-7) and the hit inside the
// closed triangle, the chain's own triangles at the segment's ends skipped -- the same decision as the oracle's
// brute force.  Blocked chains are dropped before the deterministic ordering (kept chains keep their keys).
#include <algorithm>
#include <cfloat>

#include "kernels.cuh"

namespace spoly {

constexpr double kVisEps = 1e-7;

// ---------------------------------------------------------------- hierarchy build
__global__ void k_occ_tris(const float* __restrict__ pos, const uint32_t* __restrict__ tri,
                           const uint32_t* __restrict__ order, uint32_t ntris, TriRec* recs) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntris) return;
  const uint32_t t = order[i];
  float p[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t v = tri[3ull * t + j];
#pragma unroll
    for (int c = 0; c < 3; ++c) p[3 * j + c] = pos[3ull * v + c];
  }
  TriRec R;
  R.r[0] = make_float4(p[0], p[1], p[2], p[3]);
  R.r[1] = make_float4(p[4], p[5], p[6], p[7]);
  R.r[2] = make_float4(p[8], 0.f, 0.f, 0.f);
  R.r[3] = make_float4(0.f, 0.f, 0.f, 0.f);
  R.r[4] = make_float4(0.f, 0.f, __uint_as_float(t), 0.f);
  recs[i] = R;
}

// level-1 boxes from the triangles (8 per node)
__global__ void k_aabb_leaf(const TriRec* __restrict__ recs, uint32_t ntris, float4* __restrict__ box, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  for (uint32_t t = 8 * i; t < min(ntris, 8 * i + 8); ++t) {
    const float4 a = recs[t].r[0], b = recs[t].r[1], c = recs[t].r[2];
    const float v[9] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x};
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        lo[d] = fminf(lo[d], v[3 * j + d]);
        hi[d] = fmaxf(hi[d], v[3 * j + d]);
      }
  }
  box[2 * i] = make_float4(lo[0], lo[1], lo[2], 0.f);
  box[2 * i + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
}

// level-l boxes from level l-1 (8 children per node)
__global__ void k_aabb_up(const float4* __restrict__ child, uint32_t nchild, float4* __restrict__ box, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 lo = make_float4(FLT_MAX, FLT_MAX, FLT_MAX, 0.f), hi = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, 0.f);
  for (uint32_t c = 8 * i; c < min(nchild, 8 * i + 8); ++c) {
    const float4 a = child[2 * c], b = child[2 * c + 1];
    lo.x = fminf(lo.x, a.x); lo.y = fminf(lo.y, a.y); lo.z = fminf(lo.z, a.z);
    hi.x = fmaxf(hi.x, b.x); hi.y = fmaxf(hi.y, b.y); hi.z = fmaxf(hi.z, b.z);
  }
  box[2 * i] = lo;
  box[2 * i + 1] = hi;
}

int aabb_levels(uint32_t ntris, uint32_t* n) {
  int L = 0;
  uint64_t m = ntris;
  n[0] = ntris;
  while (m > 8 && L < kMaxAabbLevels - 1) {
    m = (m + 7) / 8;
    n[++L] = (uint32_t)m;
  }
  return L;  // top level index (0: the triangles themselves)
}

void launch_build_aabbs(const TriRec* recs, AabbTree& T, cudaStream_t st) {
  for (int l = 1; l <= T.top; ++l) {
    const uint32_t n = T.n[l];
    if (l == 1)
      k_aabb_leaf<<<(n + 127) / 128, 128, 0, st>>>(recs, T.n[0], T.box[1], n);
    else
      k_aabb_up<<<(n + 127) / 128, 128, 0, st>>>(T.box[l - 1], T.n[l - 1], T.box[l], n);
  }
}

void launch_occ_tris(const float* pos, const uint32_t* tri, const uint32_t* order, uint32_t ntris, TriRec* recs,
                     cudaStream_t st) {
  if (ntris) k_occ_tris<<<(ntris + 255) / 256, 256, 0, st>>>(pos, tri, order, ntris, recs);
}

// ---------------------------------------------------------------- traversal
__device__ __forceinline__ bool seg_box(d3 a, d3 inv, double tmax_seg, float4 lo, float4 hi) {
  // slab test of the segment a + t d, t in [0, 1] (inv = 1/d per axis, +-inf for 0 components), box grown by a
  // relative 1e-6 + 1e-9 absolute (the float boxes are exact; the margin absorbs the FP64 slab arithmetic)
  double t0 = 0.0, t1 = tmax_seg;
  const double ax[3] = {a.x, a.y, a.z}, iv[3] = {inv.x, inv.y, inv.z};
  const double l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double pad = 1e-6 * (h[d] - l[d]) + 1e-9 * (1.0 + fabs(l[d]) + fabs(h[d]));
    double ta = (l[d] - pad - ax[d]) * iv[d], tb = (h[d] + pad - ax[d]) * iv[d];
    if (isnan(ta) || isnan(tb)) {  // zero direction component: inside the slab or not
      if (ax[d] < l[d] - pad || ax[d] > h[d] + pad) return false;
      continue;
    }
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    t0 = fmax(t0, ta);
    t1 = fmin(t1, tb);
    if (t0 > t1) return false;
  }
  return true;
}

__device__ __forceinline__ bool seg_tri(d3 a, d3 d, const TriRec* __restrict__ recs, uint32_t t) {
  const float4 r0 = __ldg(&recs[t].r[0]), r1 = __ldg(&recs[t].r[1]), r2 = __ldg(&recs[t].r[2]);
  const d3 p0 = mk3(r0.x, r0.y, r0.z), p1 = mk3(r0.w, r1.x, r1.y), p2 = mk3(r1.z, r1.w, r2.x);
  const d3 e1 = p1 - p0, e2 = p2 - p0;
  const d3 P = cross(d, e2);
  const double det = dot(e1, P);
  if (det == 0.0) return false;
  const d3 s = a - p0;
  const double u = dot(s, P) / det;
  const d3 Q = cross(s, e1);
  const double v = dot(d, Q) / det;
  const double tt = dot(e2, Q) / det;
  return tt > kVisEps && tt < 1.0 - kVisEps && u >= 0.0 && v >= 0.0 && u + v <= 1.0;
}

__device__ bool tree_blocked(const AabbTree& T, d3 a, d3 b, uint32_t skip1, uint32_t skip2) {
  if (!T.n[0]) return false;
  const d3 d = b - a;
  const d3 inv = mk3(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
  uint32_t stack[8 * kMaxAabbLevels + 8];
  int sp = 0;
  for (uint32_t i = 0; i < T.n[T.top]; ++i) stack[sp++] = ((uint32_t)T.top << 27) | i;
  while (sp > 0) {
    const uint32_t e = stack[--sp];
    const int l = (int)(e >> 27);
    const uint32_t i = e & ((1u << 27) - 1);
    if (l == 0) {
      if (i != skip1 && i != skip2 && seg_tri(a, d, T.tris, i)) return true;
      continue;
    }
    if (!seg_box(a, inv, 1.0, __ldg(&T.box[l][2 * i]), __ldg(&T.box[l][2 * i + 1]))) continue;
    const uint32_t c0 = 8 * i, c1 = min(T.n[l - 1], 8 * i + 8);
    for (uint32_t c = c0; c < c1; ++c) stack[sp++] = ((uint32_t)(l - 1) << 27) | c;
  }
  return false;
}

// one thread per raw solution: keep[s] = 1 when every segment of its chain is unblocked
__global__ void k_visibility(int k, uint64_t n, const unsigned long long* __restrict__ key, const double* __restrict__ bary,
                             const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                             const double* __restrict__ ep, AabbTree mesh, AabbTree occ, uint8_t* __restrict__ keep,
                             unsigned long long* __restrict__ counters) {
  uint32_t blocked_cnt = 0;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pair = key[s] >> 6;
    const uint32_t q = pq[pair];
    const double* e = ep + 6ull * q;
    d3 x[4];
    uint32_t tp[2] = {0xffffffffu, 0xffffffffu};
    x[0] = mk3(e[0], e[1], e[2]);
    for (int i = 0; i < k; ++i) {
      tp[i] = pt[(uint64_t)k * pair + i];
      d3 P[3], N[3];
      load_tri(mesh.tris, tp[i], P, N);
      const double u = bary[(uint64_t)2 * k * s + 2 * i], v = bary[(uint64_t)2 * k * s + 2 * i + 1];
      x[i + 1] = P[0] + u * (P[1] - P[0]) + v * (P[2] - P[0]);
    }
    x[k + 1] = mk3(e[3], e[4], e[5]);
    bool blk = false;
    for (int i = 0; i <= k && !blk; ++i) {
      const uint32_t s1 = i >= 1 ? tp[i - 1] : 0xffffffffu, s2 = i < k ? tp[i] : 0xffffffffu;
      blk = tree_blocked(mesh, x[i], x[i + 1], s1, s2) || tree_blocked(occ, x[i], x[i + 1], 0xffffffffu, 0xffffffffu);
    }
    keep[s] = blk ? 0 : 1;
    blocked_cnt += blk;
  }
  for (int off = 16; off > 0; off >>= 1) blocked_cnt += __shfl_xor_sync(0xffffffffu, blocked_cnt, off);
  if ((threadIdx.x & 31) == 0 && blocked_cnt) {
    atomicAdd(counters + C_REJ_VIS, (unsigned long long)blocked_cnt);
    atomicAdd(counters + C_ADMISSIBLE, (unsigned long long)0 - blocked_cnt);
  }
}

// compaction of the raw solution sink by the selected indices (order preserved)
__global__ void k_gather_raw(const uint32_t* __restrict__ sel, uint64_t n, int k, SolSink in, unsigned long long* okey,
                             double* obary, double* ocontrib, float* oresid) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = sel[j];
    okey[j] = in.key[s];
    for (int c = 0; c < 2 * k; ++c) obary[(uint64_t)2 * k * j + c] = in.bary[(uint64_t)2 * k * s + c];
    ocontrib[j] = in.contrib[s];
    oresid[j] = in.resid[s];
  }
}

void launch_visibility(int k, uint64_t n, const SolSink& S, const uint32_t* pq, const uint32_t* pt, const double* ep,
                       const AabbTree& mesh, const AabbTree& occ, uint8_t* keep, int nsm, cudaStream_t st) {
  if (!n) return;
  const uint64_t want = (n + 127) / 128, cap = (uint64_t)nsm * 16;
  k_visibility<<<(int)(want < cap ? want : cap), 128, 0, st>>>(k, n, S.key, S.bary, pq, pt, ep, mesh, occ, keep,
                                                               S.counters);
}

void launch_gather_raw(const uint32_t* sel, uint64_t n, int k, const SolSink& in, unsigned long long* okey,
                       double* obary, double* ocontrib, float* oresid, cudaStream_t st) {
  if (!n) return;
  k_gather_raw<<<(int)std::min<uint64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(sel, n, k, in, okey, obary,
                                                                                     ocontrib, oresid);
}

}  // namespace spoly
