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
// Hierarchy: 64-triangle clusters -> 8-triangle sub-clusters -> triangles (all in Morton order).  One
// warp per query; survivors are OR-ed into a per-query bitmask row (one bit per Morton position), so
// the work list that `k_expand_bits` emits is query-major and Morton-ordered (deterministic) whatever
// order the tests ran in.
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

template <bool REFRACT>
__global__ void __launch_bounds__(256) k_cull_bits(const double* __restrict__ ep, uint32_t nq,
                                                   const ClusterRec* __restrict__ l1, const ClusterRec* __restrict__ l2,
                                                   const TriCull* __restrict__ tc, uint32_t ntris, uint32_t nl1,
                                                   float ef, float eb, uint32_t* __restrict__ bits, uint32_t words,
                                                   uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nl2 = (ntris + 7) >> 3;
  for (uint32_t q = gw; q < nq; q += nw) {
    const double* e = ep + 6ull * q;
    const f3 x0 = {(float)e[0], (float)e[1], (float)e[2]};
    const f3 x2 = {(float)e[3], (float)e[4], (float)e[5]};
    uint32_t* row = bits + (uint64_t)q * words;
    uint32_t count = 0;
    for (uint32_t base = 0; base < nl1; base += 32) {
      const uint32_t c = base + lane;
      const bool k1 = c < nl1 && test_cluster<REFRACT>(x0, x2, l1[c], ef, eb);
      uint32_t m1 = __ballot_sync(0xffffffffu, k1);
      while (m1) {
        // up to 4 surviving 64-clusters per round: 32 lanes test their 8 sub-clusters each
        uint32_t sel[4];
        int nsel = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (m1) {
            sel[i] = base + __ffs(m1) - 1;
            m1 &= m1 - 1;
            nsel = i + 1;
          } else {
            sel[i] = 0;
          }
        }
        const int which = lane >> 3, sub = lane & 7;
        const uint32_t sc = sel[which] * 8 + sub;
        const bool k2 = which < nsel && sc < nl2 && test_cluster<REFRACT>(x0, x2, l2[sc], ef, eb);
        uint32_t m2 = __ballot_sync(0xffffffffu, k2);
        uint32_t word = 0;  // lane i < 2*nsel owns bits [32*(i&1), 32*(i&1)+32) of cluster sel[i>>1]
        while (m2) {
          int pick[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (m2) {
              pick[i] = __ffs(m2) - 1;
              m2 &= m2 - 1;
            } else {
              pick[i] = -1;
            }
          }
          const int j = lane >> 3, t = lane & 7;
          bool k3 = false;
          if (pick[j] >= 0) {
            const uint32_t tri = sel[pick[j] >> 3] * 64 + (pick[j] & 7) * 8 + t;
            if (tri < ntris) k3 = test_tri<REFRACT>(x0, x2, tc[tri], ef, eb);
          }
          const uint32_t m3 = __ballot_sync(0xffffffffu, k3);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (pick[i] >= 0) {
              const int cl = pick[i] >> 3, sb = pick[i] & 7;
              const uint32_t b8 = (m3 >> (8 * i)) & 0xFFu;
              if (lane == 2 * cl + (sb >> 2)) word |= b8 << (8 * (sb & 3));
            }
          }
        }
        if (lane < 2 * nsel && word) {
          row[sel[lane >> 1] * 2 + (lane & 1)] = word;
          count += __popc(word);
        }
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) count += __shfl_xor_sync(0xffffffffu, count, off);
    if (lane == 0) counts[q] = count;
  }
}

void launch_cull_bits(const double* ep, uint32_t nq, const DeviceMesh& M, int refract, uint32_t* bits, uint32_t words,
                      uint32_t* counts, int nsm, cudaStream_t st) {
  if (!nq) return;
  const int threads = 256;
  uint64_t want = ((uint64_t)nq * 32 + threads - 1) / threads;
  uint64_t cap = (uint64_t)nsm * 8;
  int blocks = (int)(want < cap ? want : cap);
  if (refract)
    k_cull_bits<true><<<blocks, threads, 0, st>>>(ep, nq, M.clusters, M.sub, M.tcull, M.ntris, M.nclusters,
                                                   M.eta_front, M.eta_back, bits, words, counts);
  else
    k_cull_bits<false><<<blocks, threads, 0, st>>>(ep, nq, M.clusters, M.sub, M.tcull, M.ntris, M.nclusters,
                                                    M.eta_front, M.eta_back, bits, words, counts);
}

// bitmask rows -> query-major work list at the scanned offsets; one warp per query
__global__ void k_expand_bits(const uint32_t* __restrict__ bits, uint32_t words, uint32_t nq,
                              const unsigned long long* __restrict__ offsets, uint32_t* pq, uint32_t* pt) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = gw; q < nq; q += nw) {
    const uint32_t* row = bits + (uint64_t)q * words;
    unsigned long long pos = offsets[q];
    for (uint32_t w0 = 0; w0 < words; w0 += 32) {
      const uint32_t wi = w0 + lane;
      uint32_t word = wi < words ? row[wi] : 0u;
      const uint32_t c = __popc(word);
      uint32_t incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      unsigned long long p = pos + incl - c;
      while (word) {
        const int b = __ffs(word) - 1;
        word &= word - 1;
        pq[p] = q;
        pt[p] = wi * 32 + b;
        ++p;
      }
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

void launch_expand_bits(const uint32_t* bits, uint32_t words, uint32_t nq, const unsigned long long* offsets,
                        uint32_t* pq, uint32_t* pt, int nsm, cudaStream_t st) {
  if (!nq) return;
  k_expand_bits<<<nsm * 16, 256, 0, st>>>(bits, words, nq, offsets, pq, pt);
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
