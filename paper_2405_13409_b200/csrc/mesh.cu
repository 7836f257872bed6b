// Mesh upload kernels: de-indexed per-triangle FP32 records in Morton order,
// per-triangle cull nodes, and the two cluster levels (64 and 8 Morton-consecutive triangles).
#include <cfloat>

#include "kernels.cuh"

namespace spoly {

// sin(theta + margin), 1 when >= 90 deg
__device__ __forceinline__ float cone_sin(double theta, double margin) {
  double b = theta * (1.0 + 1e-6) + 1e-7 + margin;
  return b >= 1.5707963 ? 1.0f : (float)fmin(1.0, sin(b) * (1.0 + 1e-6) + 1e-7);
}

// per-triangle cull node: centroid sphere, cone of the normalised vertex normals, geometric plane
__device__ TriCull make_tcull(const float* p, const float* n, float margin) {
  d3 P[3] = {mk3(p[0], p[1], p[2]), mk3(p[3], p[4], p[5]), mk3(p[6], p[7], p[8])};
  d3 N[3] = {normalize(mk3(n[0], n[1], n[2])), normalize(mk3(n[3], n[4], n[5])), normalize(mk3(n[6], n[7], n[8]))};
  d3 c = (1.0 / 3.0) * (P[0] + P[1] + P[2]);
  double rho = fmax(norm(P[0] - c), fmax(norm(P[1] - c), norm(P[2] - c)));
  d3 ax = N[0] + N[1] + N[2];
  double al = norm(ax), th = 4.0;
  if (al > 0) {
    ax = (1.0 / al) * ax;
    th = 0;
    for (int j = 0; j < 3; ++j) th = fmax(th, atan2(norm(cross(N[j], ax)), dot(N[j], ax)));
  }
  d3 g = cross(P[1] - P[0], P[2] - P[0]);
  TriCull T;
  T.sphere = make_float4((float)c.x, (float)c.y, (float)c.z, (float)(rho * (1.0 + 1e-5) + 1e-6));
  T.cone = make_float4((float)ax.x, (float)ax.y, (float)ax.z, cone_sin(th, margin));
  T.plane = make_float4((float)g.x, (float)g.y, (float)g.z, (float)dot(g, P[0]));
  return T;
}

__global__ void k_build_tris(const float* __restrict__ pos, const float* __restrict__ nrm,
                             const uint32_t* __restrict__ tri, const uint32_t* __restrict__ order, uint32_t ntris,
                             float margin, TriRec* recs, TriCull* tc, uint32_t* orig_id, uint32_t* perm_of) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntris) return;
  const uint32_t t = order[i];
  float p[9], n[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t v = tri[3ull * t + j];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      p[3 * j + c] = pos[3ull * v + c];
      n[3 * j + c] = nrm[3ull * v + c];
    }
  }
  TriRec R;
  R.r[0] = make_float4(p[0], p[1], p[2], p[3]);
  R.r[1] = make_float4(p[4], p[5], p[6], p[7]);
  R.r[2] = make_float4(p[8], n[0], n[1], n[2]);
  R.r[3] = make_float4(n[3], n[4], n[5], n[6]);
  R.r[4] = make_float4(n[7], n[8], __uint_as_float(t), 0.f);
  recs[i] = R;
  orig_id[i] = t;
  perm_of[t] = i;
  tc[i] = make_tcull(p, n, margin);
}

void launch_build_tris(const float* pos, const float* nrm, const uint32_t* tri, const uint32_t* order, uint32_t ntris,
                       float margin, TriRec* recs, TriCull* tc, uint32_t* orig_id, uint32_t* perm_of,
                       cudaStream_t st) {
  if (!ntris) return;
  k_build_tris<<<(ntris + 255) / 256, 256, 0, st>>>(pos, nrm, tri, order, ntris, margin, recs, tc, orig_id, perm_of);
}

// Glossy vertices (reading R28): every triangle's three shading normals get the same microfacet
// offset p T + q B, with (T, B) the orthonormal frame of the triangle plane (T along e1, B = g^ x T),
// n_j' = fl32(n_j + p T + q B) computed in FP64 from the uploaded (base) record; the cull node is rebuilt from the
// perturbed normals.  slopes: [ntris][2] in ORIGINAL triangle order.
__global__ void k_perturb_tris(const TriRec* __restrict__ base, const double* __restrict__ slopes,
                               const uint32_t* __restrict__ orig_id, uint32_t ntris, float margin, TriRec* recs,
                               TriCull* tc) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntris) return;
  TriRec R = base[i];
  float f[20];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    f[4 * j] = R.r[j].x; f[4 * j + 1] = R.r[j].y; f[4 * j + 2] = R.r[j].z; f[4 * j + 3] = R.r[j].w;
  }
  const float* p = f;      // p[0..8]
  float* n = f + 9;        // n[0..8]
  const uint32_t t = orig_id[i];
  const double sp = slopes[2ull * t], sq = slopes[2ull * t + 1];
  const d3 P0 = mk3(p[0], p[1], p[2]), e1 = mk3(p[3], p[4], p[5]) - P0, e2 = mk3(p[6], p[7], p[8]) - P0;
  const d3 gh = normalize(cross(e1, e2)), T = normalize(e1), B = cross(gh, T);
  const d3 h = sp * T + sq * B;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    n[3 * j] = (float)((double)n[3 * j] + h.x);
    n[3 * j + 1] = (float)((double)n[3 * j + 1] + h.y);
    n[3 * j + 2] = (float)((double)n[3 * j + 2] + h.z);
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) R.r[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
  recs[i] = R;
  tc[i] = make_tcull(p, n, margin);
}

void launch_perturb_tris(const TriRec* base, const double* slopes, const uint32_t* orig_id, uint32_t ntris,
                         float margin, TriRec* recs, TriCull* tc, cudaStream_t st) {
  if (!ntris) return;
  k_perturb_tris<<<(ntris + 255) / 256, 256, 0, st>>>(base, slopes, orig_id, ntris, margin, recs, tc);
}

// cull nodes of the current records (after restoring the uploaded normals)
__global__ void k_rebuild_tcull(const TriRec* __restrict__ recs, uint32_t ntris, float margin, TriCull* tc) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntris) return;
  const TriRec R = recs[i];
  float f[20];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    f[4 * j] = R.r[j].x; f[4 * j + 1] = R.r[j].y; f[4 * j + 2] = R.r[j].z; f[4 * j + 3] = R.r[j].w;
  }
  tc[i] = make_tcull(f, f + 9, margin);
}

void launch_rebuild_tcull(const TriRec* recs, uint32_t ntris, float margin, TriCull* tc, cudaStream_t st) {
  if (ntris) k_rebuild_tcull<<<(ntris + 255) / 256, 256, 0, st>>>(recs, ntris, margin, tc);
}

// Renderer splat (SPEC S:661-669 cmd_render): acc[q] += scale * per_query[q]
__global__ void k_splat(const double* __restrict__ per_query, uint32_t nq, double scale, double* acc) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
    acc[q] += scale * per_query[q];
}

// 8-bit sRGB-gamma code of the linear radiance (gray): c = round(255 * min(1, exposure * L)^(1/2.2))
__global__ void k_tonemap(const double* __restrict__ L, uint32_t nq, double exposure, uint8_t* rgb) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const double v = fmin(1.0, fmax(0.0, exposure * L[q]));
    const uint8_t c = (uint8_t)rint(255.0 * pow(v, 1.0 / 2.2));
    rgb[3ull * q] = c;
    rgb[3ull * q + 1] = c;
    rgb[3ull * q + 2] = c;
  }
}

void launch_splat(const double* per_query, uint32_t nq, double scale, double* acc, cudaStream_t st) {
  if (nq) k_splat<<<(nq + 255) / 256 < 4096 ? (nq + 255) / 256 : 4096, 256, 0, st>>>(per_query, nq, scale, acc);
}

void launch_tonemap(const double* L, uint32_t nq, double exposure, uint8_t* rgb, cudaStream_t st) {
  if (nq) k_tonemap<<<(nq + 255) / 256 < 4096 ? (nq + 255) / 256 : 4096, 256, 0, st>>>(L, nq, exposure, rgb);
}

// one warp per cluster of G consecutive Morton triangles: bounding sphere of all vertices around their
// mean, normal cone of all (normalised) vertex normals
template <int G>
__global__ void k_build_clusters(const TriRec* __restrict__ recs, uint32_t ntris, float margin, ClusterRec* cl,
                                 uint32_t ncl) {
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncl) return;
  const uint32_t t0 = c * G;
  double s[3] = {0, 0, 0}, ax[3] = {0, 0, 0};
  int cnt = 0;
  for (int j = lane; j < G; j += 32) {
    uint32_t t = t0 + j;
    if (t >= ntris) continue;
    d3 P[3], N[3];
    load_tri(recs, t, P, N);
    for (int v = 0; v < 3; ++v) {
      s[0] += P[v].x; s[1] += P[v].y; s[2] += P[v].z;
      d3 nh = normalize(N[v]);
      ax[0] += nh.x; ax[1] += nh.y; ax[2] += nh.z;
      cnt++;
    }
  }
  for (int off = 16; off; off >>= 1) {
    for (int k = 0; k < 3; ++k) {
      s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
      ax[k] += __shfl_xor_sync(0xffffffffu, ax[k], off);
    }
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  const d3 cen = mk3(s[0] / cnt, s[1] / cnt, s[2] / cnt);
  d3 axis = mk3(ax[0], ax[1], ax[2]);
  const double an = norm(axis);
  const bool ok = an > 0;
  if (ok) axis = (1.0 / an) * axis;
  double rad = 0, th = ok ? 0.0 : 4.0;
  for (int j = lane; j < G; j += 32) {
    uint32_t t = t0 + j;
    if (t >= ntris) continue;
    d3 P[3], N[3];
    load_tri(recs, t, P, N);
    for (int v = 0; v < 3; ++v) {
      rad = fmax(rad, norm(P[v] - cen));
      if (ok) {
        d3 nh = normalize(N[v]);
        th = fmax(th, atan2(norm(cross(nh, axis)), dot(nh, axis)));
      }
    }
  }
  for (int off = 16; off; off >>= 1) {
    rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, off));
    th = fmax(th, __shfl_xor_sync(0xffffffffu, th, off));
  }
  if (lane == 0) {
    ClusterRec R;
    R.sphere = make_float4((float)cen.x, (float)cen.y, (float)cen.z, (float)(rad * (1.0 + 1e-5) + 1e-6));
    R.cone = make_float4((float)axis.x, (float)axis.y, (float)axis.z, cone_sin(th, margin));
    cl[c] = R;
  }
}

// upper levels (512 .. 262,144 triangles per cluster): one 256-thread block per cluster with block reductions (a warp
// per cluster scanned 32,768 triangles with 7 warps in flight: 2.4 ms per upload / glossy offset sample at C3)
__global__ void __launch_bounds__(256) k_build_clusters_blk(const TriRec* __restrict__ recs, uint32_t ntris, uint32_t G,
                                                            float margin, ClusterRec* cl) {
  __shared__ double red[4][8];
  __shared__ int redc[8];
  const uint32_t c = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint64_t t0 = (uint64_t)c * G, t1 = min((uint64_t)ntris, t0 + G);
  double s[3] = {0, 0, 0}, ax[3] = {0, 0, 0};
  int cnt = 0;
  for (uint64_t i = t0 + t; i < t1; i += blockDim.x) {
    d3 P[3], N[3];
    load_tri(recs, (uint32_t)i, P, N);
    for (int v = 0; v < 3; ++v) {
      s[0] += P[v].x; s[1] += P[v].y; s[2] += P[v].z;
      const d3 nh = normalize(N[v]);
      ax[0] += nh.x; ax[1] += nh.y; ax[2] += nh.z;
      cnt++;
    }
  }
  for (int off = 16; off; off >>= 1) {
    for (int k = 0; k < 3; ++k) {
      s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
      ax[k] += __shfl_xor_sync(0xffffffffu, ax[k], off);
    }
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  __shared__ double ssum[8][6];
  if (lane == 0) {
    for (int k = 0; k < 3; ++k) {
      ssum[wid][k] = s[k];
      ssum[wid][3 + k] = ax[k];
    }
    redc[wid] = cnt;
  }
  __syncthreads();
  double S[6] = {0, 0, 0, 0, 0, 0};
  int C = 0;
  for (int w = 0; w < 8; ++w) {
    for (int k = 0; k < 6; ++k) S[k] += ssum[w][k];
    C += redc[w];
  }
  const d3 cen = mk3(S[0] / C, S[1] / C, S[2] / C);
  d3 axis = mk3(S[3], S[4], S[5]);
  const double an = norm(axis);
  const bool ok = an > 0;
  if (ok) axis = (1.0 / an) * axis;
  double rad = 0, th = ok ? 0.0 : 4.0;
  for (uint64_t i = t0 + t; i < t1; i += blockDim.x) {
    d3 P[3], N[3];
    load_tri(recs, (uint32_t)i, P, N);
    for (int v = 0; v < 3; ++v) {
      rad = fmax(rad, norm(P[v] - cen));
      if (ok) {
        const d3 nh = normalize(N[v]);
        th = fmax(th, atan2(norm(cross(nh, axis)), dot(nh, axis)));
      }
    }
  }
  for (int off = 16; off; off >>= 1) {
    rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, off));
    th = fmax(th, __shfl_xor_sync(0xffffffffu, th, off));
  }
  if (lane == 0) {
    red[0][wid] = rad;
    red[1][wid] = th;
  }
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < 8; ++w) {
      rad = fmax(rad, red[0][w]);
      th = fmax(th, red[1][w]);
    }
    rad = fmax(rad, red[0][0]);
    th = fmax(th, red[1][0]);
    ClusterRec R;
    R.sphere = make_float4((float)cen.x, (float)cen.y, (float)cen.z, (float)(rad * (1.0 + 1e-5) + 1e-6));
    R.cone = make_float4((float)axis.x, (float)axis.y, (float)axis.z, cone_sin(th, margin));
    cl[c] = R;
  }
}

void launch_build_upper(const TriRec* recs, uint32_t ntris, float margin, int level /* 3.. */, ClusterRec* out,
                        uint32_t n, cudaStream_t st) {
  const int threads = 128, blocks = (int)((n * 32ull + threads - 1) / threads);
  if (!n) return;
#ifndef SPOLY_UPPER_WARP
  if (level >= 4) {
    const uint32_t G = 64u << (3 * (level - 2));  // 4096, 32768, 262144
    k_build_clusters_blk<<<n, 256, 0, st>>>(recs, ntris, G, margin, out);
    return;
  }
#endif
  switch (level) {
    case 3: k_build_clusters<512><<<blocks, threads, 0, st>>>(recs, ntris, margin, out, n); break;
    case 4: k_build_clusters<4096><<<blocks, threads, 0, st>>>(recs, ntris, margin, out, n); break;
    case 5: k_build_clusters<32768><<<blocks, threads, 0, st>>>(recs, ntris, margin, out, n); break;
    default: k_build_clusters<262144><<<blocks, threads, 0, st>>>(recs, ntris, margin, out, n); break;
  }
}

void launch_build_clusters(const TriRec* recs, uint32_t ntris, float margin, ClusterRec* l1, ClusterRec* l2,
                           cudaStream_t st) {
  const uint32_t n1 = (ntris + kClusterSize - 1) / kClusterSize, n2 = (ntris + kSubSize - 1) / kSubSize;
  const int threads = 128;
  if (n1) k_build_clusters<kClusterSize><<<(n1 * 32 + threads - 1) / threads, threads, 0, st>>>(recs, ntris, margin, l1, n1);
  if (n2) k_build_clusters<kSubSize><<<(n2 * 32 + threads - 1) / threads, threads, 0, st>>>(recs, ntris, margin, l2, n2);
}

}  // namespace spoly
