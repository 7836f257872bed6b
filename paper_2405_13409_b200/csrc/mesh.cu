// Mesh upload kernels: de-indexed per-triangle FP32 records in Morton order,
// per-triangle normal cones and per-cluster (64 consecutive Morton triangles) cull bounds.
#include <cfloat>

#include "kernels.cuh"

namespace spoly {

__global__ void k_build_tris(const float* __restrict__ pos, const float* __restrict__ nrm,
                             const uint32_t* __restrict__ tri, const uint32_t* __restrict__ order, uint32_t ntris,
                             TriRec* recs, float4* tricone, uint32_t* orig_id, uint32_t* perm_of) {
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
  // normal cone of the three (normalised) vertex normals; the interpolated normal lies in their
  // positive hull, hence in this cone when its half angle is < 90 deg.
  double a[3] = {0, 0, 0}, u[3][3];
  for (int j = 0; j < 3; ++j) {
    double l = sqrt((double)n[3 * j] * n[3 * j] + (double)n[3 * j + 1] * n[3 * j + 1] + (double)n[3 * j + 2] * n[3 * j + 2]);
    for (int c = 0; c < 3; ++c) {
      u[j][c] = n[3 * j + c] / l;
      a[c] += u[j][c];
    }
  }
  double al = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
  float theta = 3.2f;
  if (al > 0) {
    for (int c = 0; c < 3; ++c) a[c] /= al;
    double th = 0;
    for (int j = 0; j < 3; ++j) {
      double cx = u[j][1] * a[2] - u[j][2] * a[1], cy = u[j][2] * a[0] - u[j][0] * a[2],
             cz = u[j][0] * a[1] - u[j][1] * a[0];
      double d = u[j][0] * a[0] + u[j][1] * a[1] + u[j][2] * a[2];
      th = fmax(th, atan2(sqrt(cx * cx + cy * cy + cz * cz), d));
    }
    theta = (float)th * (1.0f + 1e-6f) + 1e-7f;
  }
  tricone[i] = make_float4((float)a[0], (float)a[1], (float)a[2], theta);
}

void launch_build_tris(const float* pos, const float* nrm, const uint32_t* tri, const uint32_t* order, uint32_t ntris,
                       TriRec* recs, float4* tricone, uint32_t* orig_id, uint32_t* perm_of, cudaStream_t st) {
  if (!ntris) return;
  k_build_tris<<<(ntris + 255) / 256, 256, 0, st>>>(pos, nrm, tri, order, ntris, recs, tricone, orig_id, perm_of);
}

// one warp per cluster of kClusterSize consecutive Morton triangles
__global__ void k_build_clusters(const TriRec* __restrict__ recs, const float4* __restrict__ tricone, uint32_t ntris,
                                 ClusterRec* cl, uint32_t ncl) {
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncl) return;
  const uint32_t t0 = c * kClusterSize;
  // centroid of vertex positions
  double s[3] = {0, 0, 0};
  int cnt = 0;
  for (int j = lane; j < kClusterSize; j += 32) {
    uint32_t t = t0 + j;
    if (t >= ntris) continue;
    d3 P[3], N[3];
    load_tri(recs, t, P, N);
    for (int v = 0; v < 3; ++v) {
      s[0] += P[v].x;
      s[1] += P[v].y;
      s[2] += P[v].z;
      cnt++;
    }
  }
  for (int off = 16; off; off >>= 1) {
    for (int k = 0; k < 3; ++k) s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  const d3 cen = mk3(s[0] / cnt, s[1] / cnt, s[2] / cnt);
  // radius and normal-cone axis
  double rad = 0, ax[3] = {0, 0, 0};
  for (int j = lane; j < kClusterSize; j += 32) {
    uint32_t t = t0 + j;
    if (t >= ntris) continue;
    d3 P[3], N[3];
    load_tri(recs, t, P, N);
    for (int v = 0; v < 3; ++v) {
      rad = fmax(rad, norm(P[v] - cen));
      d3 nh = normalize(N[v]);
      ax[0] += nh.x;
      ax[1] += nh.y;
      ax[2] += nh.z;
    }
  }
  for (int off = 16; off; off >>= 1) {
    rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, off));
    for (int k = 0; k < 3; ++k) ax[k] += __shfl_xor_sync(0xffffffffu, ax[k], off);
  }
  d3 axis = mk3(ax[0], ax[1], ax[2]);
  const double an = norm(axis);
  double th = 0;
  if (an > 0) {
    axis = (1.0 / an) * axis;
    for (int j = lane; j < kClusterSize; j += 32) {
      uint32_t t = t0 + j;
      if (t >= ntris) continue;
      d3 P[3], N[3];
      load_tri(recs, t, P, N);
      for (int v = 0; v < 3; ++v) {
        d3 nh = normalize(N[v]);
        th = fmax(th, atan2(norm(cross(nh, axis)), dot(nh, axis)));
      }
    }
  } else {
    th = 4.0;
  }
  for (int off = 16; off; off >>= 1) th = fmax(th, __shfl_xor_sync(0xffffffffu, th, off));
  if (lane == 0) {
    ClusterRec R;
    R.sphere = make_float4((float)cen.x, (float)cen.y, (float)cen.z, (float)(rad * (1.0 + 1e-5) + 1e-6));
    R.cone = make_float4((float)axis.x, (float)axis.y, (float)axis.z, (float)(th * (1.0 + 1e-6) + 1e-7));
    cl[c] = R;
  }
}

void launch_build_clusters(const TriRec* recs, const float4* tricone, uint32_t ntris, ClusterRec* cl, cudaStream_t st) {
  const uint32_t ncl = (ntris + kClusterSize - 1) / kClusterSize;
  if (!ncl) return;
  const int threads = 128;
  k_build_clusters<<<(ncl * 32 + threads - 1) / threads, threads, 0, st>>>(recs, tricone, ntris, cl, ncl);
}

}  // namespace spoly
