// Culling pre-pass (replaces the Wang20 pruning of PAPER.md:680).
//
// Predicate (sound): any admissible x_1 on a node (triangle, or cluster of triangles) has a generalised
// half vector h = eta_prev w_prev + eta_next w_next parallel to +-n(x_1)  (Eq. 3), with w_prev / w_next
// the unit directions from x_1 to x_0 / x_2.  Each direction set is bounded through the node's bounding
// sphere (c, rho): axis (x - c)^, chord <= s (1 + s^2), s = rho / |x - c|.  Then h lies in the ball
// B(A, r), A = sum eta axis, r = sum eta chord, i.e. in the cone (A^, alpha), sin alpha = r/|A|.  The node
// is culled when |A x N| > |A| sin(alpha + beta) with beta the node's normal-cone half angle plus the
// FP32 margin (folded in at upload), i.e. when the h-cone misses both +N and -N cones.  FP32 with a
// margin: at most more permissive than the FP64 oracle predicate.
//
// Hierarchy: 64-triangle clusters -> 8-triangle sub-clusters -> triangles (all in Morton order), first
// per tile of 32 Morton-sorted queries (tile endpoint spheres), then per query on the tile's survivors;
// the work list is query-major and Morton-ordered (deterministic).
#include <algorithm>

#include "kernels.cuh"

namespace spoly {

__device__ __forceinline__ f3 ld3(float4 a) { return {a.x, a.y, a.z}; }

// direction bound from a sphere to x: writes axis and chord, returns false when no bound (s^2 > 1/4)
__device__ __forceinline__ bool sphere_dir(f3 x, float4 s, f3& a, float& chord) {
  f3 d = {x.x - s.x, x.y - s.y, x.z - s.z};
  const float l2 = dotf(d, d);
  const float inv = rsqrtf(l2);
  const float sn = s.w * inv;
  const float s2 = sn * sn;
  a = inv * d;
  chord = sn * (1.f + s2);  // >= 2 sin(asin(sn)/2) for s2 <= 1/4
  return s2 <= 0.25f;
}

// keep test of one node given the two direction bounds and the IOR pair
__device__ __forceinline__ bool node_keep(f3 ap, float cp, f3 an, float cn, float ep, float en, float4 nc) {
  const f3 A = ep * ap + en * an;
  const float r = ep * cp + en * cn;
  const float A2 = dotf(A, A);
  if (!(A2 > r * r * 1.0001f + 1e-12f)) return true;
  const float sb = nc.w, cb = sqrtf(fmaxf(1.f - sb * sb, 0.f));
  const float q = sqrtf(A2 - r * r);             // |A| cos(alpha)
  if (!(q * cb - r * sb > 0.f)) return true;      // alpha + beta >= 90 deg: no bound
  const f3 X = crossf(A, ld3(nc));
  const float rhs = r * cb + q * sb;              // |A| sin(alpha + beta)
  return !(dotf(X, X) > rhs * rhs);
}

template <bool REFRACT>
__device__ __forceinline__ bool test_cluster(f3 x0, f3 x2, const ClusterRec& C, float ef, float eb) {
  f3 ap, an;
  float cp, cn;
  if (!sphere_dir(x0, C.sphere, ap, cp) || !sphere_dir(x2, C.sphere, an, cn)) return true;
  if (!REFRACT) return node_keep(ap, cp, an, cn, 1.f, 1.f, C.cone);
  return node_keep(ap, cp, an, cn, ef, eb, C.cone) || node_keep(ap, cp, an, cn, eb, ef, C.cone);
}

// Coplanarity sign test (exact condition, FP32 with margin): a = ((x1 - x0) x (x2 - x0)) . n (Eq. 6) is the
// product of two barycentric-linear functions, so its triangle-Bernstein control points are
// A_ii (corners) and (A_ij + A_ji)/2 (edges) with A_ij = ((p_i - x0) x w) . n_j, w = x2 - x0.  A strict
// common sign beyond 1e-3 sum|A| (FP32 errors are ~1e-6 relative) proves a != 0 on the triangle: no chain.
__device__ __forceinline__ bool coplanar_keep_r(const float4 a, const float4 b, const float4 c, const float4 d,
                                                const float4 e, f3 x0, f3 x2) {
  const f3 w = x2 - x0;
  const f3 c0 = crossf(f3{a.x, a.y, a.z} - x0, w), c1 = crossf(f3{a.w, b.x, b.y} - x0, w),
           c2 = crossf(f3{b.z, b.w, c.x} - x0, w);
  const f3 n0 = {c.y, c.z, c.w}, n1 = {d.x, d.y, d.z}, n2 = {d.w, e.x, e.y};
  const float a00 = dotf(c0, n0), a11 = dotf(c1, n1), a22 = dotf(c2, n2);
  const float e01 = 0.5f * (dotf(c0, n1) + dotf(c1, n0)), e02 = 0.5f * (dotf(c0, n2) + dotf(c2, n0)),
              e12 = 0.5f * (dotf(c1, n2) + dotf(c2, n1));
  const float m = 1e-3f * (fabsf(a00) + fabsf(a11) + fabsf(a22) + 2.f * (fabsf(e01) + fabsf(e02) + fabsf(e12)));
  const bool pos = a00 > m && a11 > m && a22 > m && e01 > m && e02 > m && e12 > m;
  const bool neg = a00 < -m && a11 < -m && a22 < -m && e01 < -m && e02 < -m && e12 < -m;
  return !(pos || neg);
}
__device__ __forceinline__ bool coplanar_keep(const TriRec* __restrict__ tris, uint32_t t, f3 x0, f3 x2) {
  const float4* r = tris[t].r;
  return coplanar_keep_r(__ldg(r), __ldg(r + 1), __ldg(r + 2), __ldg(r + 3), __ldg(r + 4), x0, x2);
}

// Product-form sign test (exact condition, FP32 with margin; reading R21): every admissible
// reflection zeroes b = (d0.n)(d1.t) + (d0.t)(d1.n) (Eq. 12) for ANY tangent field t perpendicular to n, here
// t = n x e1.  With barycentric lambda, d0 = sum l_i (p_i - x0), d1 = sum l_i (x2 - p_i), n = sum l_j n_j and
// t = sum l_j (n_j x e1) are linear, so each factor is a quadratic form whose triangle-Bernstein coefficients
// are its symmetrised matrix entries, and b's 15 degree-4 Bernstein coefficients follow from the product
// rule of Bernstein polynomials.  A strict common sign beyond 1e-4 of the term-magnitude bound
// M = max|d0| max|n| max|d1| max|t| + max|d0| max|t| max|d1| max|n| (FP32 errors are ~1e-6 M) proves b != 0
// on the closed triangle: no reflection chain, the pair is dropped.
__device__ __forceinline__ bool bprod_keep_r(const float4 a, const float4 b, const float4 c4, const float4 d,
                                             const float4 e, f3 x0, f3 x2) {
  const f3 p[3] = {{a.x, a.y, a.z}, {a.w, b.x, b.y}, {b.z, b.w, c4.x}};
  const f3 n[3] = {{c4.y, c4.z, c4.w}, {d.x, d.y, d.z}, {d.w, e.x, e.y}};
  const f3 e1 = p[1] - p[0];
  f3 D[3], E[3], T[3];
  float mD = 0.f, mE = 0.f, mN = 0.f, mT = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    D[i] = p[i] - x0;
    E[i] = x2 - p[i];
    T[i] = crossf(n[i], e1);
    mD = fmaxf(mD, dotf(D[i], D[i]));
    mE = fmaxf(mE, dotf(E[i], E[i]));
    mN = fmaxf(mN, dotf(n[i], n[i]));
    mT = fmaxf(mT, dotf(T[i], T[i]));
  }
  // symmetrised quadratic forms, Bernstein order (00, 11, 22, 01, 02, 12): P = d0.n, Q = d1.t, R = d0.t, U = d1.n
  float P[6], Q[6], R[6], U[6];
  constexpr int I0[6] = {0, 1, 2, 0, 0, 1}, I1[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int i = I0[k], j = I1[k];
    P[k] = 0.5f * (dotf(D[i], n[j]) + dotf(D[j], n[i]));
    Q[k] = 0.5f * (dotf(E[i], T[j]) + dotf(E[j], T[i]));
    R[k] = 0.5f * (dotf(D[i], T[j]) + dotf(D[j], T[i]));
    U[k] = 0.5f * (dotf(E[i], n[j]) + dotf(E[j], n[i]));
  }
  float c[15];
  c[0] = (P[2] * Q[2] + R[2] * U[2]);
  c[1] = 0.5f * (P[2] * Q[5] + P[5] * Q[2] + R[2] * U[5] + R[5] * U[2]);
  c[2] = 0.16666666666666666f * (P[1] * Q[2] + P[2] * Q[1] + R[1] * U[2] + R[2] * U[1]) + 0.6666666666666666f * (P[5] * Q[5] + R[5] * U[5]);
  c[3] = 0.5f * (P[1] * Q[5] + P[5] * Q[1] + R[1] * U[5] + R[5] * U[1]);
  c[4] = (P[1] * Q[1] + R[1] * U[1]);
  c[5] = 0.5f * (P[2] * Q[4] + P[4] * Q[2] + R[2] * U[4] + R[4] * U[2]);
  c[6] = 0.16666666666666666f * (P[2] * Q[3] + P[3] * Q[2] + R[2] * U[3] + R[3] * U[2]) + 0.3333333333333333f * (P[4] * Q[5] + P[5] * Q[4] + R[4] * U[5] + R[5] * U[4]);
  c[7] = 0.16666666666666666f * (P[1] * Q[4] + P[4] * Q[1] + R[1] * U[4] + R[4] * U[1]) + 0.3333333333333333f * (P[3] * Q[5] + P[5] * Q[3] + R[3] * U[5] + R[5] * U[3]);
  c[8] = 0.5f * (P[1] * Q[3] + P[3] * Q[1] + R[1] * U[3] + R[3] * U[1]);
  c[9] = 0.16666666666666666f * (P[0] * Q[2] + P[2] * Q[0] + R[0] * U[2] + R[2] * U[0]) + 0.6666666666666666f * (P[4] * Q[4] + R[4] * U[4]);
  c[10] = 0.16666666666666666f * (P[0] * Q[5] + P[5] * Q[0] + R[0] * U[5] + R[5] * U[0]) + 0.3333333333333333f * (P[3] * Q[4] + P[4] * Q[3] + R[3] * U[4] + R[4] * U[3]);
  c[11] = 0.16666666666666666f * (P[0] * Q[1] + P[1] * Q[0] + R[0] * U[1] + R[1] * U[0]) + 0.6666666666666666f * (P[3] * Q[3] + R[3] * U[3]);
  c[12] = 0.5f * (P[0] * Q[4] + P[4] * Q[0] + R[0] * U[4] + R[4] * U[0]);
  c[13] = 0.5f * (P[0] * Q[3] + P[3] * Q[0] + R[0] * U[3] + R[3] * U[0]);
  c[14] = (P[0] * Q[0] + R[0] * U[0]);
  const float M = sqrtf(mD * mN * mE * mT) * 2.f;
  const float m = 1e-4f * M;
  bool pos = true, neg = true;
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    pos = pos && c[k] > m;
    neg = neg && c[k] < -m;
  }
  return !(pos || neg);
}
__device__ __forceinline__ bool bprod_keep(const TriRec* __restrict__ tris, uint32_t t, f3 x0, f3 x2) {
  const float4* r = tris[t].r;
  return bprod_keep_r(__ldg(r), __ldg(r + 1), __ldg(r + 2), __ldg(r + 3), __ldg(r + 4), x0, x2);
}

template <bool REFRACT>
__device__ __forceinline__ bool test_tri(f3 x0, f3 x2, const TriCull& T, float ef, float eb) {
  f3 ap, an;
  float cp, cn;
  if (!sphere_dir(x0, T.sphere, ap, cp) || !sphere_dir(x2, T.sphere, an, cn)) return true;
  if (!REFRACT) return node_keep(ap, cp, an, cn, 1.f, 1.f, T.cone);
  // eta_0 from the side of x_0 w.r.t. the triangle plane (c7); within float noise of the plane: both
  const float sd = dotf(ld3(T.plane), x0) - T.plane.w;
  const float gl = sqrtf(dotf(ld3(T.plane), ld3(T.plane)));
  const bool front = sd > 0.f;
  bool k = front ? node_keep(ap, cp, an, cn, ef, eb, T.cone) : node_keep(ap, cp, an, cn, eb, ef, T.cone);
  if (!k && fabsf(sd) <= 1e-4f * gl * (fabsf(x0.x) + fabsf(x0.y) + fabsf(x0.z) + 1.f))
    k = front ? node_keep(ap, cp, an, cn, eb, ef, T.cone) : node_keep(ap, cp, an, cn, ef, eb, T.cone);
  return k;
}

// ------------------------------------------------------------------ query-coherent tiles
// Queries are sorted by a Morton code of their endpoints; each tile of 32 consecutive sorted queries is
// culled once against the tile's endpoint bounding spheres (the direction sets from a node to a sphere of
// endpoints are bounded by axis (c_x - c)^, sin(theta) = (rho + rho_x)/|c_x - c|), then each query is
// tested exactly against its tile's surviving triangles only.

__global__ void k_endpoint_bounds(const double* __restrict__ ep, uint32_t nq, float* bounds /* 12: min6, max6 */) {
  __shared__ float smin[6][256], smax[6][256];
  float lo[6], hi[6];
  for (int c = 0; c < 6; ++c) {
    lo[c] = INFINITY;
    hi[c] = -INFINITY;
  }
  // a strided sample of <= 16k queries: the bounds only scale the Morton keys (any bounds give a valid
  // order; keys are clamped), so they need not be exact
  const uint32_t stride = nq > 16384 ? nq / 16384 : 1;
  for (uint32_t q = threadIdx.x * stride; q < nq; q += blockDim.x * stride)
    for (int c = 0; c < 6; ++c) {
      const float v = (float)ep[6ull * q + c];
      lo[c] = fminf(lo[c], v);
      hi[c] = fmaxf(hi[c], v);
    }
  for (int c = 0; c < 6; ++c) {
    smin[c][threadIdx.x] = lo[c];
    smax[c][threadIdx.x] = hi[c];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int c = 0; c < 6; ++c) {
        smin[c][threadIdx.x] = fminf(smin[c][threadIdx.x], smin[c][threadIdx.x + s]);
        smax[c][threadIdx.x] = fmaxf(smax[c][threadIdx.x], smax[c][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) {
    bounds[threadIdx.x] = smin[threadIdx.x][0];
    bounds[6 + threadIdx.x] = smax[threadIdx.x][0];
  }
}

// 30-bit key: 5 bits per endpoint coordinate, interleaved (x0.x x0.y x0.z x2.x x2.y x2.z)
__global__ void k_query_keys(const double* __restrict__ ep, uint32_t nq, const float* __restrict__ bounds,
                             uint32_t* keys, uint32_t* idx) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint32_t b[6];
  for (int c = 0; c < 6; ++c) {
    const float lo = bounds[c], hi = bounds[6 + c];
    const float s = hi > lo ? ((float)ep[6ull * q + c] - lo) / (hi - lo) : 0.f;
    b[c] = (uint32_t)fminf(31.f, fmaxf(0.f, s * 32.f));
  }
  uint32_t key = 0;
  for (int bit = 4; bit >= 0; --bit)
    for (int c = 0; c < 6; ++c) key = (key << 1) | ((b[c] >> bit) & 1u);
  keys[q] = key;
  idx[q] = q;
}

void launch_query_order(const double* ep, uint32_t nq, float* bounds, uint32_t* keys, uint32_t* idx,
                        cudaStream_t st) {
  if (!nq) return;
  k_endpoint_bounds<<<1, 256, 0, st>>>(ep, nq, bounds);
  k_query_keys<<<(nq + 255) / 256, 256, 0, st>>>(ep, nq, bounds, keys, idx);
}

// direction bound from a node sphere to a sphere of endpoints (c_x, rho_x)
__device__ __forceinline__ bool sphere_dir2(f3 x, float rx, float4 s, f3& a, float& chord) {
  f3 d = {x.x - s.x, x.y - s.y, x.z - s.z};
  const float l2 = dotf(d, d);
  const float inv = rsqrtf(l2);
  const float sn = (s.w + rx) * inv;
  const float s2 = sn * sn;
  a = inv * d;
  chord = sn * (1.f + s2);
  return s2 <= 0.25f;
}

template <bool REFRACT>
__device__ __forceinline__ bool tile_node_keep(f3 x0, float r0, f3 x2, float r2, float4 sphere, float4 cone, float ef,
                                               float eb) {
  f3 ap, an;
  float cp, cn;
  if (!sphere_dir2(x0, r0, sphere, ap, cp) || !sphere_dir2(x2, r2, sphere, an, cn)) return true;
  if (!REFRACT) return node_keep(ap, cp, an, cn, 1.f, 1.f, cone);
  return node_keep(ap, cp, an, cn, ef, eb, cone) || node_keep(ap, cp, an, cn, eb, ef, cone);
}

// one warp per tile: hierarchical (64-cluster, 8-sub-cluster, triangle) cull against the tile bounds;
// survivors (Morton positions, ascending) -> tile_list[t * cap ...], true count -> tile_count[t]
template <bool REFRACT>
__global__ void __launch_bounds__(256) k_tile_cull(const double* __restrict__ ep, uint32_t nq,
                                                   const uint32_t* __restrict__ order,
                                                   const ClusterRec* __restrict__ l1,
                                                   const ClusterRec* __restrict__ l2, const TriCull* __restrict__ tc,
                                                   uint32_t ntris, uint32_t nl1, float ef, float eb, uint32_t cap,
                                                   uint32_t* __restrict__ tile_list, uint32_t* __restrict__ tile_count,
                                                   unsigned int* max_count) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t ntiles = (nq + 31) / 32;
  const uint32_t nl2 = (ntris + 7) >> 3;
  for (uint32_t t = gw; t < ntiles; t += nw) {
    // tile endpoint spheres (FP32, inflated); lanes past nq duplicate the tile's first query
    const uint32_t i = t * 32 + lane;
    const uint32_t q = i < nq ? order[i] : order[t * 32];
    const double* e = ep + 6ull * q;
    const f3 a0 = {(float)e[0], (float)e[1], (float)e[2]}, a2 = {(float)e[3], (float)e[4], (float)e[5]};
    f3 s0 = a0, s2 = a2;
    for (int off = 16; off; off >>= 1) {
      s0.x += __shfl_xor_sync(0xffffffffu, s0.x, off);
      s0.y += __shfl_xor_sync(0xffffffffu, s0.y, off);
      s0.z += __shfl_xor_sync(0xffffffffu, s0.z, off);
      s2.x += __shfl_xor_sync(0xffffffffu, s2.x, off);
      s2.y += __shfl_xor_sync(0xffffffffu, s2.y, off);
      s2.z += __shfl_xor_sync(0xffffffffu, s2.z, off);
    }
    const f3 c0 = (1.f / 32.f) * s0, c2 = (1.f / 32.f) * s2;
    float r0 = sqrtf(dotf(a0 - c0, a0 - c0)), r2 = sqrtf(dotf(a2 - c2, a2 - c2));
    for (int off = 16; off; off >>= 1) {
      r0 = fmaxf(r0, __shfl_xor_sync(0xffffffffu, r0, off));
      r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, off));
    }
    r0 = r0 * 1.0001f + 1e-6f * (fabsf(c0.x) + fabsf(c0.y) + fabsf(c0.z) + 1.f);
    r2 = r2 * 1.0001f + 1e-6f * (fabsf(c2.x) + fabsf(c2.y) + fabsf(c2.z) + 1.f);
    uint32_t count = 0;
    uint32_t* out = tile_list + (uint64_t)t * cap;
    for (uint32_t base = 0; base < nl1; base += 32) {
      const uint32_t c = base + lane;
      const bool k1 = c < nl1 && tile_node_keep<REFRACT>(c0, r0, c2, r2, l1[c].sphere, l1[c].cone, ef, eb);
      uint32_t m1 = __ballot_sync(0xffffffffu, k1);
      while (m1) {
        uint32_t sel[4];
        int nsel = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (m1) {
            sel[k] = base + __ffs(m1) - 1;
            m1 &= m1 - 1;
            nsel = k + 1;
          } else {
            sel[k] = 0;
          }
        }
        const int which = lane >> 3, sub = lane & 7;
        const uint32_t sc = sel[which] * 8 + sub;
        const bool k2 = which < nsel && sc < nl2 &&
                        tile_node_keep<REFRACT>(c0, r0, c2, r2, l2[sc].sphere, l2[sc].cone, ef, eb);
        uint32_t m2 = __ballot_sync(0xffffffffu, k2);
        // triangles of the surviving sub-clusters in ascending Morton order: 4 sub-clusters per step
        while (m2) {
          int pick[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (m2) {
              pick[k] = __ffs(m2) - 1;
              m2 &= m2 - 1;
            } else {
              pick[k] = -1;
            }
          }
          const int j = lane >> 3, tt = lane & 7;
          bool k3 = false;
          uint32_t tri = 0;
          if (pick[j] >= 0) {
            tri = sel[pick[j] >> 3] * 64 + (pick[j] & 7) * 8 + tt;
            if (tri < ntris) {
              const TriCull T = tc[tri];
              k3 = tile_node_keep<REFRACT>(c0, r0, c2, r2, T.sphere, T.cone, ef, eb);
            }
          }
          const unsigned m3 = __ballot_sync(0xffffffffu, k3);
          if (k3) {
            const uint32_t pos = count + __popc(m3 & ((1u << lane) - 1u));
            if (pos < cap) out[pos] = tri;
          }
          count += __popc(m3);
        }
      }
    }
    if (lane == 0) {
      tile_count[t] = count;
      atomicMax(max_count, count);
    }
  }
}

void launch_tile_cull(const double* ep, uint32_t nq, const uint32_t* order, const DeviceMesh& M, int refract,
                      uint32_t cap, uint32_t* tile_list, uint32_t* tile_count, unsigned int* max_count, int nsm,
                      cudaStream_t st) {
  const uint32_t ntiles = (nq + 31) / 32;
  if (!ntiles) return;
  const int threads = 256;
  uint64_t want = ((uint64_t)ntiles * 32 + threads - 1) / threads;
  uint64_t capb = (uint64_t)nsm * 8;
  const int blocks = (int)(want < capb ? want : capb);
  if (refract)
    k_tile_cull<true><<<blocks, threads, 0, st>>>(ep, nq, order, M.clusters, M.sub, M.tcull, M.ntris, M.nclusters,
                                                   M.eta_front, M.eta_back, cap, tile_list, tile_count, max_count);
  else
    k_tile_cull<false><<<blocks, threads, 0, st>>>(ep, nq, order, M.clusters, M.sub, M.tcull, M.ntris, M.nclusters,
                                                    M.eta_front, M.eta_back, cap, tile_list, tile_count, max_count);
}

// per query (one warp) on its tile's surviving triangles: cone test + Eq. 6 sign test; the keep masks
// (one 32-bit ballot per 32 tile entries) and the per-query count are stored, and k_query_expand writes
// the query-major list from them at the scanned offsets (the tests run once).
template <bool REFRACT>
__global__ void __launch_bounds__(256) k_query_cull(const double* __restrict__ ep, uint32_t nq,
                                                    const uint32_t* __restrict__ order, const TriCull* __restrict__ tc,
                                                    const TriRec* __restrict__ tris,
                                                    float ef, float eb, uint32_t cap,
                                                    const uint32_t* __restrict__ tile_list,
                                                    const uint32_t* __restrict__ tile_count, uint32_t* counts,
                                                    uint32_t* __restrict__ masks) {
  __shared__ uint32_t squeue[8][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t words = (cap + 31) / 32;
  for (uint32_t i = gw; i < nq; i += nw) {
    const uint32_t q = order[i], t = i / 32;
    const double* e = ep + 6ull * q;
    const f3 x0 = {(float)e[0], (float)e[1], (float)e[2]};
    const f3 x2 = {(float)e[3], (float)e[4], (float)e[5]};
    const uint32_t n = tile_count[t];
    const uint32_t* list = tile_list + (uint64_t)t * cap;
    uint32_t* mrow = masks + (uint64_t)q * words;
    uint32_t count = 0;
    int qn = 0;  // R: positions j passing the cone + coplanarity tests, queued for the product-form test
    for (uint32_t b = 0; b < n; b += 32) {
      const uint32_t j = b + lane;
      bool k = false;
      if (j < n) {
        const uint32_t tri = list[j];
        k = test_tri<REFRACT>(x0, x2, tc[tri], ef, eb) && coplanar_keep(tris, tri, x0, x2);
      }
      const unsigned m = __ballot_sync(0xffffffffu, k);
      if (lane == 0) mrow[b / 32] = m;
      count += __popc(m);
      if (!REFRACT) {
        // product-form sign test (reading R21) on full warps of queued survivors: a failing pair clears its
        // mask bit (same warp, ordered by __syncwarp)
        if (k) squeue[wib][qn + __popc(m & ((1u << lane) - 1u))] = j;
        qn += __popc(m);
        const bool last = b + 32 >= n;
        while (qn >= 32 || (last && qn > 0)) {
          __syncwarp();
          const int take = qn < 32 ? qn : 32;
          bool fail = false;
          uint32_t jj = 0;
          if (lane < take) {
            jj = squeue[wib][qn - take + lane];
            fail = !bprod_keep(tris, list[jj], x0, x2);
          }
          __syncwarp();
          if (fail) atomicAnd(mrow + jj / 32, ~(1u << (jj & 31)));
          count -= __popc(__ballot_sync(0xffffffffu, fail));
          qn -= take;
        }
      }
    }
    if (lane == 0) counts[q] = count;
  }
}

// Tile-major form of the same per-query cull (default; SPOLY_QC_QUERY_MAJOR builds the query-major one above): one
// warp per tile of 32 Morton-sorted queries, lane = candidate triangle of the tile's list, its cull node and record
// loaded once into registers and tested against every query of the tile (the query-major form loaded them once
// per query).  Same predicate per (query, triangle), same mask layout and counts.
template <bool REFRACT>
__global__ void __launch_bounds__(256) k_tile_query_cull(const double* __restrict__ ep, uint32_t nq,
                                                         const uint32_t* __restrict__ order,
                                                         const TriCull* __restrict__ tc,
                                                         const TriRec* __restrict__ tris, float ef, float eb,
                                                         uint32_t cap, const uint32_t* __restrict__ tile_list,
                                                         const uint32_t* __restrict__ tile_count, uint32_t* counts,
                                                         uint32_t* __restrict__ masks) {
  __shared__ float sx[8][32][6];
  __shared__ uint32_t sq[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t words = (cap + 31) / 32;
  const uint32_t ntiles = (nq + 31) / 32;
  constexpr uint32_t S = 8;  // warps per tile: warp (t, sub) takes the tile's candidate blocks sub, sub + S, ...
  for (uint32_t vw = gw; vw < ntiles * S; vw += nw) {
    const uint32_t t = vw / S, sub = vw % S;
    const uint32_t n = tile_count[t];
    if (sub * 32 >= n) continue;  // warp-uniform
    const int nqt = (int)min(32u, nq - t * 32);
    __syncwarp();
    if (lane < nqt) {
      const uint32_t q = order[t * 32 + lane];
      const double* e = ep + 6ull * q;
#pragma unroll
      for (int c = 0; c < 6; ++c) sx[wib][lane][c] = (float)e[c];
      sq[wib][lane] = q;
    }
    __syncwarp();
    const uint32_t* list = tile_list + (uint64_t)t * cap;
    uint32_t cnt = 0;  // lane qi's query count (this warp's blocks)
    for (uint32_t b = sub * 32; b < n; b += 32 * S) {
      const uint32_t j = b + lane;
      const bool have = j < n;
      const uint32_t tri = have ? list[j] : list[0];
      const TriCull C = tc[tri];
      const float4* r = tris[tri].r;
      const float4 r0 = __ldg(r), r1 = __ldg(r + 1), r2 = __ldg(r + 2), r3 = __ldg(r + 3), r4 = __ldg(r + 4);
      for (int qi = 0; qi < nqt; ++qi) {
        const f3 x0 = {sx[wib][qi][0], sx[wib][qi][1], sx[wib][qi][2]};
        const f3 x2 = {sx[wib][qi][3], sx[wib][qi][4], sx[wib][qi][5]};
        bool k = have && test_tri<REFRACT>(x0, x2, C, ef, eb) && coplanar_keep_r(r0, r1, r2, r3, r4, x0, x2);
        if (!REFRACT && k) k = bprod_keep_r(r0, r1, r2, r3, r4, x0, x2);  // reading R21
        const unsigned m = __ballot_sync(0xffffffffu, k);
        if (lane == 0) masks[(uint64_t)sq[wib][qi] * words + b / 32] = m;
        if (lane == qi) cnt += __popc(m);
      }
    }
    if (lane < nqt && cnt) atomicAdd(counts + sq[wib][lane], cnt);
  }
}

__global__ void __launch_bounds__(256) k_query_expand(uint32_t nq, const uint32_t* __restrict__ order, uint32_t cap,
                                                      const uint32_t* __restrict__ tile_list,
                                                      const uint32_t* __restrict__ tile_count,
                                                      const uint32_t* __restrict__ masks,
                                                      const unsigned long long* __restrict__ offsets,
                                                      uint32_t* __restrict__ pq, uint32_t* __restrict__ pt) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t words = (cap + 31) / 32;
  for (uint32_t i = gw; i < nq; i += nw) {
    const uint32_t q = order[i], t = i / 32;
    const uint32_t n = tile_count[t];
    const uint32_t* list = tile_list + (uint64_t)t * cap;
    const uint32_t* mrow = masks + (uint64_t)q * words;
    unsigned long long wpos = offsets[q];
    for (uint32_t b = 0; b < n; b += 32) {
      const unsigned m = mrow[b / 32];
      if ((m >> lane) & 1u) {
        const unsigned long long pos = wpos + __popc(m & ((1u << lane) - 1u));
        pq[pos] = q;
        pt[pos] = list[b + lane];
      }
      wpos += __popc(m);
    }
  }
}

void launch_query_cull(int pass, const double* ep, uint32_t nq, const uint32_t* order, const DeviceMesh& M,
                       int refract, uint32_t cap, const uint32_t* tile_list, const uint32_t* tile_count,
                       uint32_t* counts, uint32_t* masks, const unsigned long long* offsets, uint32_t* pq,
                       uint32_t* pt, int nsm, cudaStream_t st) {
  if (!nq) return;
  const int threads = 256;
  uint64_t want = ((uint64_t)nq * 32 + threads - 1) / threads;
#ifndef SPOLY_QC_GRID
#define SPOLY_QC_GRID 64  // blocks per SM; A/B: 16 -> 64 took the C2 cull 1.98 -> 1.90 ms, C3 1.35 -> 1.27 ms
#endif
  uint64_t capb = (uint64_t)nsm * SPOLY_QC_GRID;
  const int blocks = (int)(want < capb ? want : capb);
  if (pass == 1) {
    k_query_expand<<<blocks, threads, 0, st>>>(nq, order, cap, tile_list, tile_count, masks, offsets, pq, pt);
    return;
  }
#ifndef SPOLY_QC_QUERY_MAJOR
  {
    const uint64_t wt = ((uint64_t)(nq + 31) / 32 * 8 * 32 + threads - 1) / threads, ct = (uint64_t)nsm * 32;
    const int bt = (int)(wt < ct ? wt : ct);
    cudaMemsetAsync(counts, 0, sizeof(uint32_t) * nq, st);
    if (refract)
      k_tile_query_cull<true><<<bt, threads, 0, st>>>(ep, nq, order, M.tcull, M.tris, M.eta_front, M.eta_back, cap,
                                                       tile_list, tile_count, counts, masks);
    else
      k_tile_query_cull<false><<<bt, threads, 0, st>>>(ep, nq, order, M.tcull, M.tris, M.eta_front, M.eta_back, cap,
                                                        tile_list, tile_count, counts, masks);
    return;
  }
#endif
  if (refract)
    k_query_cull<true><<<blocks, threads, 0, st>>>(ep, nq, order, M.tcull, M.tris, M.eta_front, M.eta_back, cap,
                                                    tile_list, tile_count, counts, masks);
  else
    k_query_cull<false><<<blocks, threads, 0, st>>>(ep, nq, order, M.tcull, M.tris, M.eta_front, M.eta_back, cap,
                                                     tile_list, tile_count, counts, masks);
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

// no cull, k = 2: every ordered pair of distinct triangles per query (tiny meshes / tests)
__global__ void k_all_pairs2(uint32_t nq, uint32_t ntris, uint32_t* pq, uint32_t* pt) {
  const uint64_t per = (uint64_t)ntris * (ntris - 1);
  const uint64_t n = (uint64_t)nq * per;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = i / per, r = i % per;
    const uint32_t a = (uint32_t)(r / (ntris - 1));
    uint32_t b = (uint32_t)(r % (ntris - 1));
    if (b >= a) ++b;
    pq[i] = (uint32_t)q;
    pt[2 * i] = a;
    pt[2 * i + 1] = b;
  }
}
void launch_all_pairs_k2(uint32_t nq, uint32_t ntris, uint32_t* pair_query, uint32_t* pair_tpos, cudaStream_t st) {
  if (ntris >= 2) k_all_pairs2<<<1024, 256, 0, st>>>(nq, ntris, pair_query, pair_tpos);
}

// explicit CSR tuple list (original ids) -> work list (Morton positions); one warp per query
__global__ void k_expand_list(const uint32_t* __restrict__ off, const uint32_t* __restrict__ ids, uint32_t nq, int k,
                              const uint32_t* __restrict__ perm_of, uint32_t ntris, uint64_t total, uint32_t* pq,
                              uint32_t* pt, unsigned int* err) {
  // caller-supplied ids are checked here (an out-of-range id would otherwise fault and poison the context):
  // a bad id or a non-monotone / out-of-range CSR row sets *err and writes position 0 in its place
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = gw; q < nq; q += nw) {
    const uint32_t b = off[q], e = off[q + 1];
    if (e < b || e > total) {
      if (lane == 0) atomicOr(err, 2u);
      continue;
    }
    for (uint32_t i = b + lane; i < e; i += 32) {
      pq[i] = q;
      for (int j = 0; j < k; ++j) {
        const uint32_t id = ids[(uint64_t)k * i + j];
        if (id >= ntris) atomicOr(err, 1u);
        pt[(uint64_t)k * i + j] = id < ntris ? perm_of[id] : 0u;
      }
    }
  }
}
void launch_expand_list(const uint32_t* offsets, const uint32_t* tri_ids, uint32_t nq, int k, const uint32_t* perm_of,
                        uint32_t ntris, uint64_t total, uint32_t* pair_query, uint32_t* pair_tpos, unsigned int* err,
                        int nsm, cudaStream_t st) {
  if (!nq) return;
  k_expand_list<<<nsm * 8, 256, 0, st>>>(offsets, tri_ids, nq, k, perm_of, ntris, total, pair_query, pair_tpos, err);
}

}  // namespace spoly

namespace spoly {

// ------------------------------------------------------------------ two-bounce pair cull
// Node pair (A, B): the directions from any point of A to any point of B lie in the cone with axis
// (cB - cA)^ and sin(theta) = (rhoA + rhoB) / |cB - cA| (Minkowski difference of the two spheres).
// Vertex 1 at A: h1 = eta0 w(x1->x0) + eta1 w(x1->x2) parallel to +-n(A); vertex 2 at B:
// h2 = eta1 w(x2->x1) + eta2 w(x2->x3) parallel to +-n(B).  The pair is kept if both hold for one of the
// IOR assignments consistent with the chain (reading R9 enumerated: RR (1,1,1); RT (f,f,b),(b,b,f);
// TR (f,b,b),(b,f,f); TT (f,b,f),(b,f,b)).
__device__ __forceinline__ bool pair_dir(float4 sa, float4 sb, f3& a, float& chord) {
  f3 d = {sb.x - sa.x, sb.y - sa.y, sb.z - sa.z};
  const float l2 = dotf(d, d);
  const float inv = rsqrtf(l2);
  const float sn = (sa.w + sb.w) * inv;
  const float s2 = sn * sn;
  a = inv * d;
  chord = sn * (1.f + s2);
  return s2 <= 0.25f && l2 > 0.f;
}

__device__ __forceinline__ bool pair_keep(f3 x0, f3 x3, float4 sA, float4 nA, float4 sB, float4 nB, int v1t, int v2t,
                                          float ef, float eb, int side = -1 /* x_0 front (0) / back (1) of T_1 */,
                                          float r0 = 0.f, float r3 = 0.f /* endpoint sphere radii (query tiles) */) {
  f3 a0, a3, aAB;
  float c0, c3, cAB;
  if (!sphere_dir2(x0, r0, sA, a0, c0) || !sphere_dir2(x3, r3, sB, a3, c3) || !pair_dir(sA, sB, aAB, cAB)) return true;
  const f3 aBA = {-aAB.x, -aAB.y, -aAB.z};
  float e[2][3];
  int ncombo = 0;
  if (!v1t && !v2t) {
    e[0][0] = e[0][1] = e[0][2] = 1.f;
    ncombo = 1;
  } else {
    // combo 0 starts in the front medium, combo 1 in the back medium
    for (int c = 0; c < 2; ++c) {
      const float s = c == 0 ? ef : eb, o = c == 0 ? eb : ef;
      e[c][0] = s;
      e[c][1] = v1t ? o : s;
      e[c][2] = v2t ? (e[c][1] == s ? o : s) : e[c][1];
    }
    ncombo = 2;
  }
#pragma unroll
  for (int c = 0; c < ncombo; ++c) {
    if (ncombo == 2 && side >= 0 && c != side) continue;
    if (node_keep(a0, c0, aAB, cAB, e[c][0], e[c][1], nA) && node_keep(aBA, cAB, a3, c3, e[c][1], e[c][2], nB))
      return true;
  }
  return false;
}

// side filter (readings R10, R14): the other triangle needs a vertex strictly on the required side of
// this triangle's plane (x_0's / x_3's side for a reflection, the opposite side for a refraction), by more
// than 1e-6 of the triangle scale; FP32 with the tolerance halved is at most more permissive.
__device__ __forceinline__ bool side_keep(const TriRec* __restrict__ tris, uint32_t tp, f3 xref, int refract,
                                          uint32_t to) {
  const float4* r = tris[tp].r;
  const float4 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2);
  const f3 p0 = {a.x, a.y, a.z}, p1 = {a.w, b.x, b.y}, p2 = {b.z, b.w, c.x};
  const f3 e1 = p1 - p0, e2 = p2 - p0;
  const f3 g = crossf(e1, e2);
  const float gl = sqrtf(dotf(g, g)), sc = sqrtf(fmaxf(dotf(e1, e1), dotf(e2, e2)));
  const float sref = dotf(xref - p0, g);
  if (sref == 0.f) return true;
  const float sg = (sref > 0.f) == (refract == 0) ? 1.f : -1.f;
  const float4* o = tris[to].r;
  const float4 oa = __ldg(o), ob = __ldg(o + 1), oc = __ldg(o + 2);
  const f3 q0 = {oa.x, oa.y, oa.z}, q1 = {oa.w, ob.x, ob.y}, q2 = {ob.z, ob.w, oc.x};
  const float tol = 0.5e-6f * gl * sc;
  return sg * dotf(q0 - p0, g) > tol || sg * dotf(q1 - p0, g) > tol || sg * dotf(q2 - p0, g) > tol;
}

// Level-synchronous dual-tree expansion over the implicit 8-ary Morton hierarchy (levels: triangles, 8, 64,
// 512, 4096, ... consecutive triangles).  The root frontier is every (query, node pair) of the split level
// (the lowest level with <= 16 nodes); each expansion gives one warp per frontier entry, which tests the
// entry's 64 child pairs (2 per lane) and keeps them in (entry, child) order.  Pass 0 counts per entry,
// pass 1 writes at the scanned offsets (deterministic, query-major).  Every entry costs the same 64 tests,
// so the work is balanced however unevenly the kept pairs are spread over queries (the same-surface
// "diagonal" blocks of a mirror keep far more pairs than the rest).
__device__ __forceinline__ void node_bounds(const CullLevels& L, int level, uint32_t i, float4& sphere, float4& cone) {
  if (level == 0) {
    sphere = L.tc[i].sphere;
    cone = L.tc[i].cone;
  } else {
    const ClusterRec C = L.lv[level][i];
    sphere = C.sphere;
    cone = C.cone;
  }
}

// Per-child record of one frontier entry, staged in shared memory: every one of the entry's 64 child
// pairs (a, b) combines child a of node A with child b of node B, so the per-node parts of pair_keep /
// side_keep (the direction bound to x_0 or x_3, and at the triangle level the plane and side data) are
// computed once per child (16 per entry) instead of once per pair (64).  The arithmetic is the same
// expressions in the same order as pair_keep / side_keep, so the kept set is unchanged.
struct ChildRec {
  float4 sph, cone;  // bounding sphere, normal cone
  float4 dir;        // axis (x_0 or x_3 -> node) and chord of sphere_dir
  float4 g;          // triangle level: geometric normal e1 x e2 (xyz), side tolerance (w)
  float4 p0, p1, p2; // triangle level: vertices; p0.w = side sign sg, p1.w / p2.w unused
  int flags;         // bit 0: valid child, 1: sphere_dir bound ok, 2: side filter keeps all (sref == 0),
                     // 3-4: eta side of x_0 w.r.t. the plane + 1 (0: both media)
};

__device__ __forceinline__ void make_child(ChildRec& R, int cl, const CullLevels& L, const TriRec* __restrict__ tris,
                                           uint32_t i, f3 xend, float rend, int refract, int want_side) {
  // rend > 0: the endpoint is a sphere (a tile of queries); the side decisions fall back to "both" / "keep all"
  // when the sphere reaches the plane
  R.flags = 0;
  if (i >= L.n[cl]) return;
  R.flags = 1;
  if (cl == 0) {
    const TriCull T = L.tc[i];
    R.sph = T.sphere;
    R.cone = T.cone;
    if (want_side) {
      // eta_0 from the side of x_0 w.r.t. T_1's plane (within float noise of the plane: both)
      const float sd = dotf(ld3(T.plane), xend) - T.plane.w;
      const float gl = sqrtf(dotf(ld3(T.plane), ld3(T.plane)));
      int side = -1;
      if (fabsf(sd) > 1e-4f * gl * (fabsf(xend.x) + fabsf(xend.y) + fabsf(xend.z) + 1.f) + rend * gl)
        side = sd > 0.f ? 0 : 1;
      R.flags |= (side + 1) << 3;
    }
    // side_keep's per-triangle part (plane, reference side, tolerance)
    const float4* r = tris[i].r;
    const float4 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2);
    const f3 p0 = {a.x, a.y, a.z}, p1 = {a.w, b.x, b.y}, p2 = {b.z, b.w, c.x};
    const f3 e1 = p1 - p0, e2 = p2 - p0;
    const f3 g = crossf(e1, e2);
    const float gl = sqrtf(dotf(g, g)), sc = sqrtf(fmaxf(dotf(e1, e1), dotf(e2, e2)));
    const float sref = dotf(xend - p0, g);
    if (sref == 0.f || fabsf(sref) <= rend * gl * 1.0001f) R.flags |= 4;
    const float sg = (sref > 0.f) == (refract == 0) ? 1.f : -1.f;
    R.g = make_float4(g.x, g.y, g.z, 0.5e-6f * gl * sc);
    R.p0 = make_float4(p0.x, p0.y, p0.z, sg);
    R.p1 = make_float4(p1.x, p1.y, p1.z, 0.f);
    R.p2 = make_float4(p2.x, p2.y, p2.z, 0.f);
  } else {
    const ClusterRec C = L.lv[cl][i];
    R.sph = C.sphere;
    R.cone = C.cone;
  }
  f3 d;
  float ch;
  if (sphere_dir2(xend, rend, R.sph, d, ch)) R.flags |= 2;
  R.dir = make_float4(d.x, d.y, d.z, ch);
}

// side_keep(tris, t, xref, refract, o) with t's part precomputed in record it and o's vertices in record io
// (records in the warp's SoA staging f[field][child], flags fl[child])
__device__ __forceinline__ bool side_keep_rec(const float4 (*f)[32], const int* fl, int it, int io) {
  if (fl[it] & 4) return true;
  const float4 G = f[3][it], P0 = f[4][it];
  const f3 g = ld3(G), p0 = ld3(P0);
  const float sg = P0.w, tol = G.w;
  return sg * dotf(ld3(f[4][io]) - p0, g) > tol || sg * dotf(ld3(f[5][io]) - p0, g) > tol ||
         sg * dotf(ld3(f[6][io]) - p0, g) > tol;
}

// pair_keep(x0, x3, sA, cA, sB, cB, ...) with the per-node direction bounds precomputed
__device__ __forceinline__ bool pair_keep_rec(const float4 (*f)[32], const int* fl, int ia, int ib, int v1t, int v2t,
                                              float ef, float eb, int side) {
  f3 aAB;
  float cAB;
  if (!(fl[ia] & 2) || !(fl[ib] & 2) || !pair_dir(f[0][ia], f[0][ib], aAB, cAB)) return true;
  const float4 DA = f[2][ia], DB = f[2][ib];
  const f3 a0 = ld3(DA), a3 = ld3(DB);
  const float c0 = DA.w, c3 = DB.w;
  const f3 aBA = {-aAB.x, -aAB.y, -aAB.z};
  float e[2][3];
  int ncombo = 0;
  if (!v1t && !v2t) {
    e[0][0] = e[0][1] = e[0][2] = 1.f;
    ncombo = 1;
  } else {
    for (int c = 0; c < 2; ++c) {
      const float s = c == 0 ? ef : eb, o = c == 0 ? eb : ef;
      e[c][0] = s;
      e[c][1] = v1t ? o : s;
      e[c][2] = v2t ? (e[c][1] == s ? o : s) : e[c][1];
    }
    ncombo = 2;
  }
#pragma unroll
  for (int c = 0; c < ncombo; ++c) {
    if (ncombo == 2 && side >= 0 && c != side) continue;
    if (node_keep(a0, c0, aAB, cAB, e[c][0], e[c][1], f[1][ia]) &&
        node_keep(aBA, cAB, a3, c3, e[c][1], e[c][2], f[1][ib]))
      return true;
  }
  return false;
}

// fq == nullptr: implicit root frontier (entry e -> query qbase + e / P, pair e % P of the split level), the
// root pair itself is tested first.  cl = level of the children (0: triangle pairs, written to pq / pt).
// Pass 0 tests the 64 child pairs of every entry (one warp per entry, 2 per lane; lanes 0-7 / 8-15 first
// stage the entry's 8 + 8 child records) and stores the 64-bit keep mask and its popcount; pass 1 writes
// the kept pairs from the masks at the scanned offsets in (entry, child) order (deterministic, query-major).
constexpr int kExpandThreads = 256;
__global__ void __launch_bounds__(kExpandThreads, 3) k_pair_expand(int pass, int cl, const double* __restrict__ ep,
                                                     uint32_t qbase, const uint32_t* __restrict__ fq, const uint32_t* __restrict__ fa,
                                                     const uint32_t* __restrict__ fb, uint64_t nf,
                                                     const TriRec* __restrict__ tris, CullLevels L, int v1t, int v2t,
                                                     float ef, float eb, uint32_t* __restrict__ counts,
                                                     unsigned long long* __restrict__ masks,
                                                     const unsigned long long* __restrict__ offsets,
                                                     uint32_t* __restrict__ oq, uint32_t* __restrict__ oa,
                                                     uint32_t* __restrict__ ob, const float4* __restrict__ tsph) {
  // tsph != NULL: frontier entries are (query TILE, node, node) and the endpoints are the tile's spheres
  // tsph[2 t] = (c0, r0), tsph[2 t + 1] = (c3, r3)
  // Two frontier entries per warp: half-warp h (lanes 16h..16h+15) stages its entry's 8 + 8 child records
  // and tests the entry's 64 child pairs, 4 per lane.  Structure-of-arrays staging, record i of half h at
  // slot 2i + h of smf[warp][field][.], so the records a warp-wide load touches sit in distinct banks.
  __shared__ float4 smf[kExpandThreads / 32][7][32];
  __shared__ int smk[kExpandThreads / 32][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, h = lane >> 4, hl = lane & 15;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t nt = L.n[L.top], P = nt * nt;
  for (uint64_t e0 = 2 * gw; e0 < nf; e0 += 2 * nw) {
    const uint64_t en = e0 + h;
    const bool valid = en < nf;
    uint32_t q = 0, A = 0, B = 0;
    if (valid) {
      if (fq) {
        q = fq[en];
        A = fa[en];
        B = fb[en];
      } else {
        q = qbase + (uint32_t)(en / P);
        A = (uint32_t)(en % P) / nt;
        B = (uint32_t)(en % P) % nt;
      }
    }
    if (pass) {
      const unsigned long long m = valid ? masks[en] : 0ull;
      if (m) {
        const unsigned long long base = offsets[en];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = t * 16 + hl;
          if ((m >> c) & 1ull) {
            const unsigned long long pos = base + __popcll(m & ((1ull << c) - 1ull));
            const uint32_t a = A * 8 + (c >> 3), b = B * 8 + (c & 7);
            oq[pos] = q;
            if (cl == 0) {
              oa[2 * pos] = a;
              oa[2 * pos + 1] = b;
            } else {
              oa[pos] = a;
              ob[pos] = b;
            }
          }
        }
      }
      continue;
    }
    f3 x0 = {0.f, 0.f, 0.f}, x3 = {0.f, 0.f, 0.f};
    float r0 = 0.f, r3 = 0.f;
    bool root_ok = valid;
    if (valid) {
      if (tsph) {
        const float4 s0 = tsph[2 * q], s3 = tsph[2 * q + 1];
        x0 = {s0.x, s0.y, s0.z};
        r0 = s0.w;
        x3 = {s3.x, s3.y, s3.z};
        r3 = s3.w;
      } else {
        const double* e = ep + 6ull * q;
        x0 = {(float)e[0], (float)e[1], (float)e[2]};
        x3 = {(float)e[3], (float)e[4], (float)e[5]};
      }
      if (!fq) {
        float4 sa, ca, sb, cb;
        node_bounds(L, cl + 1, A, sa, ca);
        node_bounds(L, cl + 1, B, sb, cb);
        root_ok = pair_keep(x0, x3, sa, ca, sb, cb, v1t, v2t, ef, eb, -1, r0, r3);
      }
    }
    __syncwarp();
    {
      const bool isB = hl >= 8;
      ChildRec R;
      R.flags = 0;
      if (root_ok)
        make_child(R, cl, L, tris, (isB ? B : A) * 8 + (hl & 7), isB ? x3 : x0, isB ? r3 : r0, isB ? v2t : v1t,
                   !isB && (v1t || v2t));
      const int sl = 2 * hl + h;
      smf[wib][0][sl] = R.sph;
      smf[wib][1][sl] = R.cone;
      smf[wib][2][sl] = R.dir;
      smf[wib][3][sl] = R.g;
      smf[wib][4][sl] = R.p0;
      smf[wib][5][sl] = R.p1;
      smf[wib][6][sl] = R.p2;
      smk[wib][sl] = R.flags;
    }
    __syncwarp();
    unsigned long long m = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int c = t * 16 + hl;
      const int ia = 2 * (c >> 3) + h, ib = 2 * (8 + (c & 7)) + h;
      const int fa_ = smk[wib][ia], fb_ = smk[wib][ib];
      bool k = false;
      if ((fa_ & 1) && (fb_ & 1)) {
        if (cl == 0) {
          if (A * 8 + (c >> 3) != B * 8 + (c & 7))
            k = pair_keep_rec(smf[wib], smk[wib], ia, ib, v1t, v2t, ef, eb, ((fa_ >> 3) & 3) - 1) &&
                side_keep_rec(smf[wib], smk[wib], ia, ib) && side_keep_rec(smf[wib], smk[wib], ib, ia);
        } else {
          k = pair_keep_rec(smf[wib], smk[wib], ia, ib, v1t, v2t, ef, eb, -1);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, k);
      m |= (unsigned long long)((bal >> (16 * h)) & 0xffffu) << (16 * t);
    }
    if (valid && hl == 0) {
      counts[en] = (uint32_t)__popcll(m);
      masks[en] = m;
    }
  }
}

static CullLevels cull_levels_of(const DeviceMesh& M) {
  CullLevels L;
  L.tc = M.tcull;
  L.lv[0] = nullptr;
  L.lv[1] = M.sub;
  L.lv[2] = M.clusters;
  L.n[0] = M.ntris;
  L.n[1] = (M.ntris + 7) / 8;
  L.n[2] = M.nclusters;
  int top = 2;
  for (int i = 0; i < M.nupper; ++i) {
    L.lv[3 + i] = M.upper[i];
    L.n[3 + i] = M.nupper_nodes[i];
    top = 3 + i;
  }
  while (top > 1 && L.n[top - 1] <= 16) --top;  // split level: the lowest (>= 1) with <= 16 nodes
  L.top = L.n[top] <= 16 ? top : -1;
  return L;
}

int cull_split_level(const DeviceMesh& M, uint32_t* pairs_per_query) {
  const CullLevels L = cull_levels_of(M);
  if (L.top < 0) return -1;
  *pairs_per_query = L.n[L.top] * L.n[L.top];
  return L.top;
}

void launch_pair_expand(int pass, int cl, const double* ep, uint32_t qbase, const uint32_t* fq, const uint32_t* fa,
                        const uint32_t* fb, uint64_t nf, const DeviceMesh& M, int v1t, int v2t, uint32_t* counts,
                        unsigned long long* masks, const unsigned long long* offsets, uint32_t* oq, uint32_t* oa, uint32_t* ob, int nsm,
                        cudaStream_t st, const float4* tsph) {
  if (!nf) return;
  const CullLevels L = cull_levels_of(M);
  const int threads = 256;
  const uint64_t want = (nf * 32 + threads - 1) / threads, cap = (uint64_t)nsm * 64;
  k_pair_expand<<<(int)(want < cap ? want : cap), threads, 0, st>>>(pass, cl, ep, qbase, fq, fa, fb, nf, M.tris, L, v1t, v2t,
                                                                    M.eta_front, M.eta_back, counts, masks, offsets, oq,
                                                                    oa, ob, tsph);
}

// ------------------------------------------------------------------ two-bounce query tiles
// Tiles of 32 consecutive Morton-sorted queries share one node-pair expansion against their endpoint spheres
// (the same predicate with the direction sets from a node to a sphere of endpoints, and "both / keep" side
// decisions when a sphere reaches a plane: a superset of every member query's pairs); each query then tests its
// tile's triangle pairs exactly (the triangle-level test of the per-query expansion).
__global__ void k_tile_spheres(const double* __restrict__ ep, uint32_t nq, const uint32_t* __restrict__ order,
                               uint32_t s0, uint32_t ntiles, uint32_t ts, float4* __restrict__ tsph) {
  // tiles of ts (<= 32) consecutive sorted queries; lanes past the tile or past nq repeat its first member
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = gw; t < ntiles; t += nw) {
    const uint32_t i = s0 + t * ts + (uint32_t)lane;
    const uint32_t q = order[((uint32_t)lane < ts && i < nq) ? i : s0 + t * ts];
    const double* e = ep + 6ull * q;
    const f3 a0 = {(float)e[0], (float)e[1], (float)e[2]}, a3 = {(float)e[3], (float)e[4], (float)e[5]};
    f3 s0v = a0, s3v = a3;
    for (int off = 16; off; off >>= 1) {
      s0v.x += __shfl_xor_sync(0xffffffffu, s0v.x, off);
      s0v.y += __shfl_xor_sync(0xffffffffu, s0v.y, off);
      s0v.z += __shfl_xor_sync(0xffffffffu, s0v.z, off);
      s3v.x += __shfl_xor_sync(0xffffffffu, s3v.x, off);
      s3v.y += __shfl_xor_sync(0xffffffffu, s3v.y, off);
      s3v.z += __shfl_xor_sync(0xffffffffu, s3v.z, off);
    }
    const f3 c0 = (1.f / 32.f) * s0v, c3 = (1.f / 32.f) * s3v;
    float r0 = sqrtf(dotf(a0 - c0, a0 - c0)), r3 = sqrtf(dotf(a3 - c3, a3 - c3));
    for (int off = 16; off; off >>= 1) {
      r0 = fmaxf(r0, __shfl_xor_sync(0xffffffffu, r0, off));
      r3 = fmaxf(r3, __shfl_xor_sync(0xffffffffu, r3, off));
    }
    // inflated for the float rounding of the members and the centre
    r0 = r0 * 1.0001f + 1e-6f * (fabsf(c0.x) + fabsf(c0.y) + fabsf(c0.z) + 1.f);
    r3 = r3 * 1.0001f + 1e-6f * (fabsf(c3.x) + fabsf(c3.y) + fabsf(c3.z) + 1.f);
    if (lane == 0) {
      tsph[2 * t] = make_float4(c0.x, c0.y, c0.z, r0);
      tsph[2 * t + 1] = make_float4(c3.x, c3.y, c3.z, r3);
    }
  }
}

// per query (warp) over its tile's triangle pairs [toff[t], toff[t + 1]): the exact triangle-level test of the
// per-query expansion (pair bound with the query's endpoints, eta side of x_0, both side filters).  Pass 0: keep
// masks (one word per 32 tile pairs) + per-query counts; pass 1: the query-major list at the scanned offsets.
__global__ void __launch_bounds__(256) k_query_pairs(int pass, const double* __restrict__ ep, uint32_t nq,
                                                     const uint32_t* __restrict__ order, uint32_t s0, uint32_t sn,
                                                     uint32_t ts, const unsigned long long* __restrict__ toff,
                                                     const uint32_t* __restrict__ tpair, const TriRec* __restrict__ tris,
                                                     const TriCull* __restrict__ tc, int v1t, int v2t, float ef,
                                                     float eb, const unsigned long long* __restrict__ moff,
                                                     uint32_t* __restrict__ masks, uint32_t* __restrict__ counts,
                                                     const unsigned long long* __restrict__ offsets,
                                                     uint32_t* __restrict__ oq, uint32_t* __restrict__ ot) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = gw; k < sn; k += nw) {
    const uint32_t i = s0 + k;
    if (i >= nq) continue;
    const uint32_t q = order[i], t = k / ts;
    const unsigned long long b0 = toff[t], b1 = toff[t + 1];
    uint32_t* mrow = masks + moff[t] + (unsigned long long)(k % ts) * ((b1 - b0 + 31) / 32);
    if (pass) {
      unsigned long long pos = offsets[k];
      for (unsigned long long b = b0; b < b1; b += 32) {
        const uint32_t m = mrow[(b - b0) / 32];
        const unsigned long long j = b + lane;
        if ((m >> lane) & 1u) {
          const unsigned long long p = pos + __popc(m & ((1u << lane) - 1u));
          oq[p] = q;
          ot[2 * p] = tpair[2 * j];
          ot[2 * p + 1] = tpair[2 * j + 1];
        }
        pos += __popc(m);
      }
      continue;
    }
    const double* e = ep + 6ull * q;
    const f3 x0 = {(float)e[0], (float)e[1], (float)e[2]}, x3 = {(float)e[3], (float)e[4], (float)e[5]};
    uint32_t count = 0;
    for (unsigned long long b = b0; b < b1; b += 32) {
      const unsigned long long j = b + lane;
      bool kp = false;
      if (j < b1) {
        const uint32_t A = tpair[2 * j], B = tpair[2 * j + 1];
        const TriCull TA = tc[A], TB = tc[B];
        int side = -1;
        if (v1t || v2t) {
          const float sd = dotf(ld3(TA.plane), x0) - TA.plane.w;
          const float gl = sqrtf(dotf(ld3(TA.plane), ld3(TA.plane)));
          if (fabsf(sd) > 1e-4f * gl * (fabsf(x0.x) + fabsf(x0.y) + fabsf(x0.z) + 1.f)) side = sd > 0.f ? 0 : 1;
        }
        kp = pair_keep(x0, x3, TA.sphere, TA.cone, TB.sphere, TB.cone, v1t, v2t, ef, eb, side) &&
             side_keep(tris, A, x0, v1t, B) && side_keep(tris, B, x3, v2t, A);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, kp);
      if (lane == 0) mrow[(b - b0) / 32] = m;
      count += __popc(m);
    }
    if (lane == 0) counts[k] = count;
  }
}

void launch_tile_spheres(const double* ep, uint32_t nq, const uint32_t* order, uint32_t s0, uint32_t ntiles,
                         uint32_t ts, float4* tsph, int nsm, cudaStream_t st) {
  if (!ntiles) return;
  const uint64_t want = ((uint64_t)ntiles * 32 + 255) / 256, cap = (uint64_t)nsm * 16;
  k_tile_spheres<<<(int)(want < cap ? want : cap), 256, 0, st>>>(ep, nq, order, s0, ntiles, ts, tsph);
}

void launch_query_pairs(int pass, const double* ep, uint32_t nq, const uint32_t* order, uint32_t s0, uint32_t sn,
                        uint32_t ts, const unsigned long long* toff, const uint32_t* tpair, const DeviceMesh& M,
                        int v1t, int v2t, const unsigned long long* moff, uint32_t* masks, uint32_t* counts,
                        const unsigned long long* offsets, uint32_t* oq, uint32_t* ot, int nsm, cudaStream_t st) {
  if (!sn) return;
  const uint64_t want = ((uint64_t)sn * 32 + 255) / 256, cap = (uint64_t)nsm * 32;
  k_query_pairs<<<(int)(want < cap ? want : cap), 256, 0, st>>>(pass, ep, nq, order, s0, sn, ts, toff, tpair, M.tris,
                                                                 M.tcull, v1t, v2t, M.eta_front, M.eta_back, moff,
                                                                 masks, counts, offsets, oq, ot);
}

// per-tile counts of a tile-major (tile, pair) list -> exclusive offsets computed by the caller's scan
__global__ void k_tile_hist(const uint32_t* __restrict__ tq, uint64_t n, unsigned long long* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + tq[i], 1ull);
}
void launch_tile_hist(const uint32_t* tq, uint64_t n, unsigned long long* cnt, int nsm, cudaStream_t st) {
  if (!n) return;
  const uint64_t want = (n + 255) / 256, cap = (uint64_t)nsm * 16;
  k_tile_hist<<<(int)(want < cap ? want : cap), 256, 0, st>>>(tq, n, cnt);
}

// ------------------------------------------------------------------ barycentric subdivision refinement (k=2)
// A kept triangle pair is re-tested on 4-way midpoint subdivisions of both triangles, `levels` deep (SURVEY
// A1 "Refinement"): positions and (linearly interpolated) normals of a sub-triangle are the interpolants at
// its corners, so its bounding sphere (centroid, max corner distance) and normal cone (axis = sum of the
// normalised corner normals, half angle = max corner angle; a positive combination of the corner
// directions stays inside a convex cone containing them) bound every point of it, and the pair-direction
// bound of the two sub-spheres holds as above.  The pair is kept iff some sub-pair passes at every level
// down to `levels` (depth-first, early exit on the first leaf).  FP64 with 1e-7 rad / 1e-9 relative
// slack, so it is at most more permissive than the exact predicate on the sub-pairs.
//
// A sub-triangle is (o_u, o_v, sigma) in units of 2^-kMaxLevels of the barycentric square with corners
// o, o + sigma (h, 0), o + sigma (0, h); children: three with the same sigma at o, o + sigma (h/2, 0),
// o + sigma (0, h/2) and the inverted middle one (-sigma) at o + sigma (h/2, h/2).
constexpr int kMaxLevels = 5;

struct SubB {
  d3 c, ax;
  double rho, sinb;
  bool ok;  // false: no bound (keep)
  d3 X[3];  // the cell's corners (exact direction cones)
};

__device__ __forceinline__ SubB sub_bound(const d3 P[3], const d3 N[3], int ou, int ov, int sg, int h) {
  constexpr double inv = 1.0 / (1 << kMaxLevels);
  const double u[3] = {ou * inv, (ou + sg * h) * inv, ou * inv};
  const double v[3] = {ov * inv, ov * inv, (ov + sg * h) * inv};
  d3 X[3], M[3];
  SubB B;
  B.ok = true;
  for (int j = 0; j < 3; ++j) {
    X[j] = P[0] + u[j] * (P[1] - P[0]) + v[j] * (P[2] - P[0]);
    const d3 n = N[0] + u[j] * (N[1] - N[0]) + v[j] * (N[2] - N[0]);
    const double l = norm(n);
    if (!(l > 1e-30)) B.ok = false;
    M[j] = (1.0 / l) * n;
  }
  B.X[0] = X[0];
  B.X[1] = X[1];
  B.X[2] = X[2];
  B.c = (1.0 / 3.0) * (X[0] + X[1] + X[2]);
  B.rho = fmax(norm(X[0] - B.c), fmax(norm(X[1] - B.c), norm(X[2] - B.c))) * (1.0 + 1e-9) + 1e-12;
  const d3 s = M[0] + M[1] + M[2];
  const double sl = norm(s);
  if (!(sl > 0)) {
    B.ok = false;
    return B;
  }
  B.ax = (1.0 / sl) * s;
  const double cmin = fmin(dot(M[0], B.ax), fmin(dot(M[1], B.ax), dot(M[2], B.ax)));
  if (!(cmin > 1e-6)) B.ok = false;
  B.sinb = fmin(1.0, sqrt(fmax(0.0, 1.0 - cmin * cmin)) + 1e-7);
  return B;
}

__device__ __forceinline__ bool sphere_dir_d(d3 x, d3 c, double rho, d3& a, double& chord) {
  const d3 d = x - c;
  const double l = norm(d);
  if (!(l > 0)) return false;
  const double sn = rho / l;
  a = (1.0 / l) * d;
  chord = sn * (1.0 + sn * sn);
  return sn * sn <= 0.25;
}

__device__ __forceinline__ bool node_keep_d(d3 ap, double cp, d3 an, double cn, double ep, double en, d3 nax,
                                            double sb) {
  const d3 A = ep * ap + en * an;
  const double r = ep * cp + en * cn;
  const double A2 = dot(A, A);
  if (!(A2 > r * r * (1.0 + 1e-9))) return true;
  const double cb = sqrt(fmax(1.0 - sb * sb, 0.0));
  const double q = sqrt(A2 - r * r);
  if (!(q * cb - r * sb > 0.0)) return true;
  const d3 X = cross(A, nax);
  const double rhs = r * cb + q * sb;
  return !(dot(X, X) > rhs * rhs * (1.0 + 1e-9));
}

__device__ __forceinline__ bool subpair_keep(d3 x0, d3 x3, const SubB& A, const SubB& B, const double e[2][3],
                                             int ncombo) {
  if (!A.ok || !B.ok) return true;
  d3 a0, a3, aAB;
  double c0, c3, cAB;
  if (!sphere_dir_d(x0, A.c, A.rho, a0, c0) || !sphere_dir_d(x3, B.c, B.rho, a3, c3) ||
      !sphere_dir_d(B.c, A.c, A.rho + B.rho, aAB, cAB))
    return true;
  const d3 aBA = -1.0 * aAB;
  for (int c = 0; c < ncombo; ++c)
    if (node_keep_d(a0, c0, aAB, cAB, e[c][0], e[c][1], A.ax, A.sinb) &&
        node_keep_d(aBA, cAB, a3, c3, e[c][1], e[c][2], B.ax, B.sinb))
      return true;
  return false;
}

// exact direction cone of a point set (the oracle's cone_of): axis = normalised sum of the unit
// directions, chord = max |w_j - axis| (+1e-9 relative slack).  Every direction to / between points of the convex
// hulls is a positive combination of these, so it lies in the cap {w : |w - axis| <= chord}.  false: no bound.
template <int M>
__device__ __forceinline__ bool exact_cone(const d3 (&d)[M], d3& axis, double& chord) {
  d3 w[M];
  d3 s = mk3(0, 0, 0);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double l2 = dot(d[j], d[j]);
    if (!(l2 > 0)) return false;
    w[j] = (1.0 / sqrt(l2)) * d[j];
    s = s + w[j];
  }
  const double sl = norm(s);
  if (!(sl > 0)) return false;
  axis = (1.0 / sl) * s;
  double c2 = 0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const d3 t = w[j] - axis;
    c2 = fmax(c2, dot(t, t));
  }
  chord = sqrt(c2) * (1.0 + 1e-9) + 1e-12;
  return true;
}

// sub-pair test with exact vertex cones (tighter than the sphere bounds of subpair_keep, same predicate)
__device__ __forceinline__ bool subpair_keep_exact(const SubB& A, const SubB& B, d3 a0, double c0, bool ok0, d3 a3,
                                                   double c3, bool ok3, const double e[2][3], int ncombo) {
  if (!A.ok || !B.ok || !ok0 || !ok3) return true;
  d3 d[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) d[3 * i + j] = B.X[j] - A.X[i];
  d3 aAB;
  double cAB;
  if (!exact_cone<9>(d, aAB, cAB)) return true;
  const d3 aBA = -1.0 * aAB;
  for (int c = 0; c < ncombo; ++c)
    if (node_keep_d(a0, c0, aAB, cAB, e[c][0], e[c][1], A.ax, A.sinb) &&
        node_keep_d(aBA, cAB, a3, c3, e[c][1], e[c][2], B.ax, B.sinb))
      return true;
  return false;
}

struct SubNode {
  int u1, v1, s1, u2, v2, s2;
};

__device__ __forceinline__ void child_of(int ou, int ov, int sg, int h, int c, int& cu, int& cv, int& cs) {
  const int hh = h >> 1;
  cu = ou + ((c == 1 || c == 3) ? sg * hh : 0);
  cv = ov + ((c == 2 || c == 3) ? sg * hh : 0);
  cs = c == 3 ? -sg : sg;
}

// 16-bit mask of the surviving child pairs of node n (size h)
__device__ uint32_t children_mask(const d3 P1[3], const d3 N1[3], const d3 P2[3], const d3 N2[3], d3 x0, d3 x3,
                                  const SubNode& n, int h, const double e[2][3], int ncombo) {
  SubB A[4], B[4];
  for (int c = 0; c < 4; ++c) {
    int cu, cv, cs;
    child_of(n.u1, n.v1, n.s1, h, c, cu, cv, cs);
    A[c] = sub_bound(P1, N1, cu, cv, cs, h >> 1);
    child_of(n.u2, n.v2, n.s2, h, c, cu, cv, cs);
    B[c] = sub_bound(P2, N2, cu, cv, cs, h >> 1);
  }
  uint32_t m = 0;
#ifndef SPOLY_REFINE_SPHERE
  // exact cones of the directions from each cell to its endpoint, once per cell
  d3 a0[4], a3[4];
  double c0[4], c3[4];
  bool ok0[4], ok3[4];
  for (int c = 0; c < 4; ++c) {
    d3 d0[3] = {x0 - A[c].X[0], x0 - A[c].X[1], x0 - A[c].X[2]};
    ok0[c] = exact_cone<3>(d0, a0[c], c0[c]);
    d3 d3_[3] = {x3 - B[c].X[0], x3 - B[c].X[1], x3 - B[c].X[2]};
    ok3[c] = exact_cone<3>(d3_, a3[c], c3[c]);
  }
  for (int i = 0; i < 16; ++i) {
    const int ia = i >> 2, ib = i & 3;
    if (subpair_keep_exact(A[ia], B[ib], a0[ia], c0[ia], ok0[ia], a3[ib], c3[ib], ok3[ib], e, ncombo)) m |= 1u << i;
  }
#else
  for (int i = 0; i < 16; ++i)
    if (subpair_keep(x0, x3, A[i >> 2], B[i & 3], e, ncombo)) m |= 1u << i;
#endif
  return m;
}

// ---- FP32 refinement (default; SPOLY_REFINE_FP64 restores the FP64 predicate above).  Same cells, same exact
// vertex cones, evaluated in FP32 with every bound inflated by its rounding error, so the kept set is a superset
// of the exact predicate's:
//  - cell corners X = p0 + u e1 + v e2 (u, v dyadic: exact) carry an absolute error <= 3 * 2^-24 (|p0|+|e1|+|e2|);
//    a direction d = X_b - X_a between two such points (or an endpoint rounded to FP32) is off by at most
//    eps_d <= 1.2e-6 (|X_a| + |X_b|) (the scales include the triangle's own), so its unit vector moves by at most
//    eps_d / |d| + 1e-6 (normalisation rounding); each cone chord is inflated by the largest such bound;
//  - normal cones: unit corner normals (error <= 1e-6), half-angle sine from |M_j x axis| + 4e-6 (no 1 - c^2
//    cancellation); no bound (keep) when a corner normal is within 89.9 deg of 90 from the axis;
//  - the final separation test keeps the pair unless it fails by a relative 1e-5.
struct SubBf {
  f3 X[3];
  float S[3];  // |X_j| + the triangle scale: the error scale of directions from X_j
  f3 ax;
  float sinb;
  bool ok;
};

__device__ __forceinline__ float fnorm(f3 a) { return sqrtf(dotf(a, a)); }

__device__ __forceinline__ SubBf sub_bound_f(const f3 P[3], const f3 N[3], float tscale, int ou, int ov, int sg,
                                             int h) {
  constexpr float inv = 1.f / (1 << kMaxLevels);
  const float u[3] = {ou * inv, (ou + sg * h) * inv, ou * inv};
  const float v[3] = {ov * inv, ov * inv, (ov + sg * h) * inv};
  const f3 e1 = P[1] - P[0], e2 = P[2] - P[0], m1 = N[1] - N[0], m2 = N[2] - N[0];
  SubBf B;
  B.ok = true;
  f3 M[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    B.X[j] = P[0] + u[j] * e1 + v[j] * e2;
    B.S[j] = fnorm(B.X[j]) + tscale;
    const f3 n = N[0] + u[j] * m1 + v[j] * m2;
    const float l2 = dotf(n, n);
    if (!(l2 > 1e-30f)) B.ok = false;
    M[j] = rsqrtf(l2) * n;
  }
  const f3 s = M[0] + M[1] + M[2];
  const float sl2 = dotf(s, s);
  if (!(sl2 > 1e-12f)) {
    B.ok = false;
    return B;
  }
  B.ax = rsqrtf(sl2) * s;
  float sb2 = 0.f;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    if (!(dotf(M[j], B.ax) > 2e-3f)) B.ok = false;
    const f3 x = crossf(M[j], B.ax);
    sb2 = fmaxf(sb2, dotf(x, x));
  }
  B.sinb = fminf(1.f, sqrtf(sb2) + 4e-6f);
  return B;
}

// exact direction cone of M directions d_j with error scales S_j (see above): axis, inflated chord
template <int M>
__device__ __forceinline__ bool exact_cone_f(const f3 (&d)[M], const float (&S)[M], f3& axis, float& chord) {
  f3 w[M];
  float er[M];
  f3 s = {0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const float l2 = dotf(d[j], d[j]);
    if (!(l2 > 1e-30f)) return false;
    const float il = rsqrtf(l2);
    w[j] = il * d[j];
    er[j] = 1.2e-6f * S[j] * il + 1e-6f;
    s = s + w[j];
  }
  const float sl2 = dotf(s, s);
  if (!(sl2 > 1e-12f)) return false;
  axis = rsqrtf(sl2) * s;
  // max_j (|w_j - axis| + er_j) <= sqrt(max_j |w_j - axis|^2) + max_j er_j: one square root
  float c2 = 0.f, em = 0.f;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const f3 t = w[j] - axis;
    c2 = fmaxf(c2, dotf(t, t));
    em = fmaxf(em, er[j]);
  }
  chord = (sqrtf(c2) + em) * (1.f + 1e-5f) + 2e-6f;
  return true;
}

// node_keep with a relative 1e-5 margin on the final separation test
__device__ __forceinline__ bool node_keep_r(f3 ap, float cp, f3 an, float cn, float ep, float en, f3 nax, float sb) {
  const f3 A = ep * ap + en * an;
  const float r = ep * cp + en * cn;
  const float A2 = dotf(A, A);
  if (!(A2 > r * r * 1.0001f + 1e-12f)) return true;
  const float cb = sqrtf(fmaxf(1.f - sb * sb, 0.f));
  const float q = sqrtf(A2 - r * r);
  if (!(q * cb - r * sb > 1e-6f * sqrtf(A2))) return true;
  const f3 X = crossf(A, nax);
  const float rhs = r * cb + q * sb;
  return !(dotf(X, X) > rhs * rhs * (1.f + 1e-5f) + 1e-12f * A2);
}

// 16-bit mask of the surviving child pairs of node n (size h), FP32
__device__ uint32_t children_mask_f(const f3 P1[3], const f3 N1[3], float s1, const f3 P2[3], const f3 N2[3], float s2,
                                    f3 x0, float n0, f3 x3, float n3, const SubNode& n, int h, const float e[2][3],
                                    int ncombo) {
  SubBf A[4], B[4];
  f3 a0[4], a3[4];
  float c0[4], c3[4];
  bool ok0[4], ok3[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int cu, cv, cs;
    child_of(n.u1, n.v1, n.s1, h, c, cu, cv, cs);
    A[c] = sub_bound_f(P1, N1, s1, cu, cv, cs, h >> 1);
    child_of(n.u2, n.v2, n.s2, h, c, cu, cv, cs);
    B[c] = sub_bound_f(P2, N2, s2, cu, cv, cs, h >> 1);
    const f3 d0[3] = {x0 - A[c].X[0], x0 - A[c].X[1], x0 - A[c].X[2]};
    const float S0[3] = {A[c].S[0] + n0, A[c].S[1] + n0, A[c].S[2] + n0};
    ok0[c] = exact_cone_f<3>(d0, S0, a0[c], c0[c]);
    const f3 d3_[3] = {x3 - B[c].X[0], x3 - B[c].X[1], x3 - B[c].X[2]};
    const float S3[3] = {B[c].S[0] + n3, B[c].S[1] + n3, B[c].S[2] + n3};
    ok3[c] = exact_cone_f<3>(d3_, S3, a3[c], c3[c]);
  }
  uint32_t m = 0;
#ifdef SPOLY_REFINE_ROLL
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int ia = 0; ia < 4; ++ia)
#pragma unroll 1
  for (int ib = 0; ib < 4; ++ib) {
    const int i = 4 * ia + ib;
    const SubBf& SA = A[ia];
    const SubBf& SB = B[ib];
    bool keep = true;
    if (SA.ok && SB.ok && ok0[ia] && ok3[ib]) {
      f3 d[9];
      float S[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          d[3 * a + b] = SB.X[b] - SA.X[a];
          S[3 * a + b] = SA.S[a] + SB.S[b];
        }
      f3 aAB;
      float cAB;
      if (exact_cone_f<9>(d, S, aAB, cAB)) {
        const f3 aBA = {-aAB.x, -aAB.y, -aAB.z};
        keep = false;
        for (int c = 0; c < ncombo && !keep; ++c)
          keep = node_keep_r(a0[ia], c0[ia], aAB, cAB, e[c][0], e[c][1], SA.ax, SA.sinb) &&
                 node_keep_r(aBA, cAB, a3[ib], c3[ib], e[c][1], e[c][2], SB.ax, SB.sinb);
      }
    }
    if (keep) m |= 1u << i;
  }
  return m;
}

__device__ __forceinline__ void load_tri_f(const TriRec* __restrict__ T, uint32_t i, f3 p[3], f3 n[3], float& scale) {
  const float4* r = T[i].r;
  const float4 a = __ldg(r), b = __ldg(r + 1), c = __ldg(r + 2), d = __ldg(r + 3), e = __ldg(r + 4);
  p[0] = {a.x, a.y, a.z};
  p[1] = {a.w, b.x, b.y};
  p[2] = {b.z, b.w, c.x};
  n[0] = {c.y, c.z, c.w};
  n[1] = {d.x, d.y, d.z};
  n[2] = {d.w, e.x, e.y};
  scale = fnorm(p[0]) + fnorm(p[1] - p[0]) + fnorm(p[2] - p[0]);
}

// eta combinations of a pair: eta_0 from the side of x_0 w.r.t. T_1's plane (reading R9; sub-triangles
// share the plane); within 1e-9 of the plane both media are tried
__device__ __forceinline__ int eta_combos(d3 x0, const d3 P1[3], int v1t, int v2t, float ef, float eb,
                                          double ec[2][3]) {
  if (!v1t && !v2t) {
    ec[0][0] = ec[0][1] = ec[0][2] = 1.0;
    return 1;
  }
  const d3 g1 = cross(P1[1] - P1[0], P1[2] - P1[0]);
  const double sd = dot(x0 - P1[0], g1), tol = 1e-9 * norm(g1) * (norm(x0 - P1[0]) + 1e-30);
  int ncombo = 0;
  for (int c = 0; c < 2; ++c) {
    if ((c == 0 && sd < -tol) || (c == 1 && sd > tol)) continue;
    const double s = c == 0 ? ef : eb, o = c == 0 ? eb : ef;
    ec[ncombo][0] = s;
    ec[ncombo][1] = v1t ? o : s;
    ec[ncombo][2] = v2t ? (ec[ncombo][1] == s ? o : s) : ec[ncombo][1];
    ++ncombo;
  }
  return ncombo;
}

// Breadth-first refinement: a frontier entry is (pair, sub-triangle of T_1, sub-triangle of T_2) at the
// current level, packed in 64 bits: pair (32) | T_1 node (11: u 5, v 5, sigma 1) | T_2 node (11), node
// coordinates in units of 2^-kMaxLevels.  One thread per entry tests its 16 child pairs; survivors are
// appended (order irrelevant: only the per-pair keep flag is produced), at the last level any survivor
// sets keep[pair] = 1.  An entry whose children overflow the frontier keeps its pair (conservative, sound).
__device__ __forceinline__ uint64_t enc_node(int u, int v, int s) { return (uint64_t)(u | (v << 5) | ((s > 0) << 10)); }
__device__ __forceinline__ void dec_node(uint64_t c, int& u, int& v, int& s) {
  u = (int)(c & 31);
  v = (int)((c >> 5) & 31);
  s = ((c >> 10) & 1) ? 1 : -1;
}

#ifndef SPOLY_REFINE_MINB
#define SPOLY_REFINE_MINB 1
#endif
__global__ void __launch_bounds__(128, SPOLY_REFINE_MINB) k_refine_level(int level, int last, const uint32_t* __restrict__ pq,
                                                      const uint32_t* __restrict__ pt, uint64_t npairs,
                                                      const TriRec* __restrict__ tris, const double* __restrict__ ep,
                                                      int v1t, int v2t, float ef, float eb,
                                                      const uint64_t* __restrict__ fin,
                                                      const unsigned long long* __restrict__ nin,
                                                      uint64_t* __restrict__ fout, unsigned long long* __restrict__ nout,
                                                      uint64_t cap, uint8_t* __restrict__ keep,
                                                      uint32_t* __restrict__ vrange) {
  const uint64_t n = fin ? min((uint64_t)*nin, cap) : npairs;  // appends beyond cap were not written
  const int H = 1 << kMaxLevels, h = H >> level;  // node size at this level
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    SubNode nd;
    uint32_t r;
    if (fin) {
      const uint64_t ent = fin[i];
      r = (uint32_t)(ent >> 22);
      dec_node((ent >> 11) & 2047, nd.u1, nd.v1, nd.s1);
      dec_node(ent & 2047, nd.u2, nd.v2, nd.s2);
      // already proven kept through another branch (without v-ranges: every surviving branch must be walked to
      // bound the surviving v-range)
      if (!vrange && keep[r]) continue;
    } else {
      r = (uint32_t)i;
      nd = {0, 0, 1, 0, 0, 1};
    }
    const double* e = ep + 6ull * pq[r];
    const d3 x0 = mk3(e[0], e[1], e[2]), x3 = mk3(e[3], e[4], e[5]);
#ifdef SPOLY_REFINE_FP64
    d3 P1[3], N1[3], P2[3], N2[3];
    load_tri(tris, pt[2 * r], P1, N1);
    load_tri(tris, pt[2 * r + 1], P2, N2);
    double ec[2][3];
    const int ncombo = eta_combos(x0, P1, v1t, v2t, ef, eb, ec);
    const uint32_t m = children_mask(P1, N1, P2, N2, x0, x3, nd, h, ec, ncombo);
#else
    uint32_t m;
    {
      d3 P1d[3], N1d[3];
      load_tri(tris, pt[2 * r], P1d, N1d);
      double ec[2][3];
      const int ncombo = eta_combos(x0, P1d, v1t, v2t, ef, eb, ec);  // FP64 side decision, as the FP64 path
      float ecf[2][3];
      for (int c = 0; c < 2; ++c)
        for (int j = 0; j < 3; ++j) ecf[c][j] = (float)ec[c][j];
      f3 P1[3], N1[3], P2[3], N2[3];
      float s1, s2;
      load_tri_f(tris, pt[2 * r], P1, N1, s1);
      load_tri_f(tris, pt[2 * r + 1], P2, N2, s2);
      const f3 x0f = {(float)x0.x, (float)x0.y, (float)x0.z}, x3f = {(float)x3.x, (float)x3.y, (float)x3.z};
      m = children_mask_f(P1, N1, s1, P2, N2, s2, x0f, fnorm(x0f), x3f, fnorm(x3f), nd, h, ecf, ncombo);
    }
#endif
    if (!m) continue;
    if (last) {
      keep[r] = 1;
      if (vrange) {
        // v-range (units of 2^-kMaxLevels) of the surviving T_1 cells: a chain of this pair can only have its x_1
        // there (the predicate is sound), so the determinant scan may skip the pieces outside it (reading R25)
        int lo = 1 << kMaxLevels, hi = 0;
        for (int c = 0; c < 4; ++c) {
          if (!((m >> (4 * c)) & 15u)) continue;
          int cu, cv, cs;
          child_of(nd.u1, nd.v1, nd.s1, h, c, cu, cv, cs);
          const int a = cs > 0 ? cv : cv - (h >> 1), b = cs > 0 ? cv + (h >> 1) : cv;
          lo = min(lo, a);
          hi = max(hi, b);
        }
        atomicMin(vrange + 2 * r, (uint32_t)lo);
        atomicMax(vrange + 2 * r + 1, (uint32_t)hi);
      }
      continue;
    }
    const unsigned long long pos = atomicAdd(nout, (unsigned long long)__popc(m));
    if (pos + __popc(m) > cap) {
      keep[r] = 1;
      if (vrange) {  // not refined further: the whole triangle
        atomicMin(vrange + 2 * r, 0u);
        atomicMax(vrange + 2 * r + 1, (uint32_t)(1 << kMaxLevels));
      }
      continue;
    }
    uint32_t mm = m;
    for (unsigned long long k = pos; mm; ++k) {
      const int c = __ffs(mm) - 1;
      mm &= mm - 1;
      SubNode ch;
      child_of(nd.u1, nd.v1, nd.s1, h, c >> 2, ch.u1, ch.v1, ch.s1);
      child_of(nd.u2, nd.v2, nd.s2, h, c & 3, ch.u2, ch.v2, ch.s2);
      fout[k] = ((uint64_t)r << 22) | (enc_node(ch.u1, ch.v1, ch.s1) << 11) | enc_node(ch.u2, ch.v2, ch.s2);
    }
  }
}

// Depth-first refinement, thread per pair (no frontier: the breadth-first frontier overflowed its cap at level 2 on
// C4 and kept whole pairs conservatively): a stack of (level, T_1 cell, T_2 cell); a pair is kept as soon as one
// cell pair survives `levels` deep (vrange == NULL), or every surviving leaf is visited and the v-range of its T_1
// cells recorded (vrange != NULL, reading R25).
__global__ void __launch_bounds__(128) k_refine_dfs(int levels, const uint32_t* __restrict__ pq,
                                                    const uint32_t* __restrict__ pt, uint64_t npairs,
                                                    const TriRec* __restrict__ tris, const double* __restrict__ ep,
                                                    int v1t, int v2t, float ef, float eb, uint8_t* __restrict__ keep,
                                                    uint32_t* __restrict__ vrange, unsigned long long* __restrict__ ntests) {
  constexpr int H = 1 << kMaxLevels;
  unsigned long long tests = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npairs; r += (uint64_t)gridDim.x * blockDim.x) {
    const double* e = ep + 6ull * pq[r];
    const d3 x0 = mk3(e[0], e[1], e[2]), x3 = mk3(e[3], e[4], e[5]);
    d3 P1[3], N1[3], P2[3], N2[3];
    load_tri(tris, pt[2 * r], P1, N1);
    load_tri(tris, pt[2 * r + 1], P2, N2);
    double ec[2][3];
    const int ncombo = eta_combos(x0, P1, v1t, v2t, ef, eb, ec);
    uint32_t stack[16 * kMaxLevels + 1];  // level (3) | T_1 cell (11) | T_2 cell (11)
    int sp = 0;
    stack[sp++] = (uint32_t)((enc_node(0, 0, 1) << 11) | enc_node(0, 0, 1));
    bool kept = false;
    int lo = H, hi = 0;
    while (sp > 0) {
      const uint32_t ent = stack[--sp];
      const int level = (int)(ent >> 22);
      SubNode nd;
      dec_node((ent >> 11) & 2047, nd.u1, nd.v1, nd.s1);
      dec_node(ent & 2047, nd.u2, nd.v2, nd.s2);
      const int h = H >> level;
      const uint32_t m = children_mask(P1, N1, P2, N2, x0, x3, nd, h, ec, ncombo);
      tests += 16;
      if (!m) continue;
      if (level + 1 == levels) {
        kept = true;
        if (!vrange) break;
        for (int c = 0; c < 4; ++c) {
          if (!((m >> (4 * c)) & 15u)) continue;
          int cu, cv, cs;
          child_of(nd.u1, nd.v1, nd.s1, h, c, cu, cv, cs);
          lo = min(lo, cs > 0 ? cv : cv - (h >> 1));
          hi = max(hi, cs > 0 ? cv + (h >> 1) : cv);
        }
        continue;
      }
      uint32_t mm = m;
      while (mm) {
        const int c = __ffs(mm) - 1;
        mm &= mm - 1;
        SubNode ch;
        child_of(nd.u1, nd.v1, nd.s1, h, c >> 2, ch.u1, ch.v1, ch.s1);
        child_of(nd.u2, nd.v2, nd.s2, h, c & 3, ch.u2, ch.v2, ch.s2);
        stack[sp++] = ((uint32_t)(level + 1) << 22) | (uint32_t)((enc_node(ch.u1, ch.v1, ch.s1) << 11) |
                                                                 enc_node(ch.u2, ch.v2, ch.s2));
      }
    }
    keep[r] = kept ? 1 : 0;
    if (vrange) {
      vrange[2 * r] = kept ? (uint32_t)lo : (uint32_t)H;
      vrange[2 * r + 1] = kept ? (uint32_t)hi : 0u;
    }
  }
  for (int off = 16; off > 0; off >>= 1) tests += __shfl_xor_sync(0xffffffffu, tests, off);
  if ((threadIdx.x & 31) == 0 && tests) atomicAdd(ntests, tests);
}

__global__ void k_vrange_init(uint32_t* vr, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    vr[2 * i] = 1u << kMaxLevels;
    vr[2 * i + 1] = 0u;
  }
}

void launch_refine_pairs(const uint32_t* pq, const uint32_t* pt, uint64_t n, const DeviceMesh& M, const double* ep,
                         int levels, int v1t, int v2t, uint8_t* keep, uint32_t* vrange, RefineScratch& W, int nsm,
                         cudaStream_t st) {
  if (!n) return;
  if (levels > kMaxLevels) levels = kMaxLevels;
#ifdef SPOLY_REFINE_DFS  // A/B: thread-per-pair depth-first (C4: same pairs, cull 0.56 -> 1.14 s: divergence)
  {
    cudaMemsetAsync(W.count, 0, sizeof(unsigned long long), st);
    const uint64_t want = (n + 127) / 128, cap = (uint64_t)nsm * 32;
    k_refine_dfs<<<(int)(want < cap ? want : cap), 128, 0, st>>>(levels, pq, pt, n, M.tris, ep, v1t, v2t,
                                                                  M.eta_front, M.eta_back, keep, vrange, W.count);
    W.launches = 1;
    return;
  }
#endif
  cudaMemsetAsync(keep, 0, n, st);
  if (vrange) k_vrange_init<<<(int)std::min<uint64_t>((n + 255) / 256, (uint64_t)nsm * 8), 256, 0, st>>>(vrange, n);
  cudaMemsetAsync(W.count, 0, 2 * levels * sizeof(unsigned long long), st);
  const uint64_t* fin = nullptr;
  const unsigned long long* nin = nullptr;
  for (int l = 0; l < levels; ++l) {
    const int last = l + 1 == levels;
    uint64_t* fout = W.front[l & 1];
    unsigned long long* nout = W.count + l;
    const uint64_t work = fin ? W.cap : n;  // device-side count bounds the loop
    const uint64_t want = (work + 127) / 128, cap = (uint64_t)nsm * 16;
    k_refine_level<<<(int)(want < cap ? want : cap), 128, 0, st>>>(l, last, pq, pt, n, M.tris, ep, v1t, v2t,
                                                                    M.eta_front, M.eta_back, fin, nin, fout, nout,
                                                                    W.cap, keep, vrange);
    fin = fout;
    nin = nout;
  }
  W.launches = levels;
}

}  // namespace spoly
