// Shared device-side definitions of the CUDA path (libspoly.so).  Nothing here is shared with the
// oracle: the oracle is a separate plain-C++ program used only by the tests.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spoly.h"

namespace spoly {

// ----------------------------------------------------------------------------- FP64 3-vectors
struct d3 {
  double x, y, z;
};
__host__ __device__ __forceinline__ d3 mk3(double x, double y, double z) { return {x, y, z}; }
__host__ __device__ __forceinline__ d3 operator+(d3 a, d3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ d3 operator-(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ d3 operator*(double s, d3 a) { return {s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ double dot(d3 a, d3 b) { return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z)); }
__host__ __device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ double norm(d3 a) { return sqrt(dot(a, a)); }
__host__ __device__ __forceinline__ d3 normalize(d3 a) { return rsqrt(dot(a, a)) * a; }

// max / min by one compare + select (DSETP + 2 FSEL) instead of fmax / fmin's NaN-quieting sequence (~6
// instructions on sm_100a).  Equal to fmax(a, b) / fmin(a, b) whenever a is not NaN (a NaN b returns a, as fmax).
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// ----------------------------------------------------------------------------- FP32 3-vectors
struct f3 {
  float x, y, z;
};
__device__ __forceinline__ f3 operator+(f3 a, f3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ f3 operator-(f3 a, f3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ f3 operator*(float s, f3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ float dotf(f3 a, f3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ f3 crossf(f3 a, f3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// ----------------------------------------------------------------------------- mesh records
// Per-triangle solve record: the float32 input vertices and vertex normals of P_i, N_i
// (PAPER.md:186), de-indexed, 5 x float4 = 80 B, triangles stored in Morton (cluster) order.
//   r0 = (p0.x p0.y p0.z p1.x)  r1 = (p1.y p1.z p2.x p2.y)  r2 = (p2.z n0.x n0.y n0.z)
//   r3 = (n1.x n1.y n1.z n2.x)  r4 = (n2.y n2.z orig_id(bits) 0)
struct TriRec {
  float4 r[5];
};
// Cull nodes (FP32).  Bounding sphere (c, rho) and normal cone (axis, sin(beta)) where beta is the cone
// half angle of the (normalised) vertex normals plus the cull margin; sin(beta) = 1 means "no bound".
struct ClusterRec {
  float4 sphere;  // c.xyz, rho
  float4 cone;    // axis.xyz, sin(beta)
};
struct TriCull {
  float4 sphere;  // centroid, rho
  float4 cone;    // axis.xyz, sin(beta)
  float4 plane;   // geometric normal g = e1 x e2 (unnormalised), g . p0
};
constexpr int kClusterSize = 64;  // level-1 cull cluster (Morton-consecutive triangles)
constexpr int kSubSize = 8;       // level-2 sub-cluster

struct DeviceMesh {
  uint32_t ntris = 0;
  uint32_t nclusters = 0;
  float eta_front = 1, eta_back = 1;
  TriRec* tris = nullptr;         // [ntris], Morton order
  TriCull* tcull = nullptr;       // [ntris]
  uint32_t* orig_id = nullptr;    // [ntris] Morton position -> original id
  uint32_t* perm_of = nullptr;    // [ntris] original id -> Morton position
  ClusterRec* clusters = nullptr; // [ceil(ntris/64)]
  ClusterRec* sub = nullptr;      // [ceil(ntris/8)]
  int nupper = 0;                 // levels above the 64-clusters: 512, 4096, ... triangles (until <= 8 nodes)
  ClusterRec* upper[4] = {nullptr, nullptr, nullptr, nullptr};
  uint32_t nupper_nodes[4] = {0, 0, 0, 0};
};

// implicit 8-ary AABB hierarchy over Morton-ordered triangles for the visibility test (visibility.cu): level 0 =
// the triangles, level l node i covers triangles [i 8^l, (i + 1) 8^l); box[l][2 i] / box[l][2 i + 1] = lo / hi
constexpr int kMaxAabbLevels = 9;
struct AabbTree {
  const TriRec* tris = nullptr;
  float4* box[kMaxAabbLevels] = {};
  uint32_t n[kMaxAabbLevels] = {};
  int top = 0;
};

// the implicit 8-ary Morton hierarchy as seen by the pair cull: level 0 = triangles, 1 = 8, 2 = 64, ...
struct CullLevels {
  const TriCull* tc;
  const ClusterRec* lv[7];
  uint32_t n[7];
  int top;
};

__device__ __forceinline__ void load_tri(const TriRec* __restrict__ T, uint32_t i, d3 p[3], d3 n[3]) {
  const float4* r = T[i].r;
  float4 a = __ldg(r + 0), b = __ldg(r + 1), c = __ldg(r + 2), d = __ldg(r + 3), e = __ldg(r + 4);
  p[0] = mk3(a.x, a.y, a.z);
  p[1] = mk3(a.w, b.x, b.y);
  p[2] = mk3(b.z, b.w, c.x);
  n[0] = mk3(c.y, c.z, c.w);
  n[1] = mk3(d.x, d.y, d.z);
  n[2] = mk3(d.w, e.x, e.y);
}

// ----------------------------------------------------------------------------- solve parameters
struct SolveParams {
  double bisect_tol, theta_admit, theta_final, eps_domain, eps_flag, tau_trunc;
  int pieces, scan_bisect_iters, polish_iters;
  double eta_front, eta_back;
};

// solution sink (ctx-owned, appended with warp-aggregated atomics).  Records carry only the sort key
// (pair index << 6 | root slot); query and triangle ids are recovered from the work list at gather time.
struct SolSink {
  unsigned long long* count;  // [0] solutions, [1] flag records
  uint64_t capacity;
  unsigned long long* key;
  double* bary;  // 2k per solution
  double* contrib;
  float* resid;
  uint64_t fcapacity;
  unsigned long long* fkey;  // pair index (a pair may emit several flag records; OR-reduced later)
  uint32_t* fflags;
  unsigned long long* counters;  // [C_NUM]
};
constexpr int kJobStride = 13;  // max doubles per job (r(v) up to degree 12; R uses 10)
// two-ended dense list between the one-bounce kernels: [0, count[0]) path entries (pair, root) of the monotone
// jobs phase 1 solved and could not finish; (capacity - 1 - d) for d < count[1]: deep jobs (pair, meta, r)
struct JobSink {
  unsigned long long* count;
  uint64_t capacity;
  uint32_t* pair;
  uint32_t* meta;  // deep jobs: kfree | deg << 8
  double* r;       // deep jobs: NR coefficients of r; the deep kernel overwrites them with [nv | np << 8, roots, probes]
  double* root;    // path entries: the v-root
};

enum { C_PAIRS = 0, C_SYSTEMS, C_VROOTS, C_CANDIDATES, C_REJ_DOMAIN, C_REJ_CONSTRAINT, C_REJ_SIDE, C_REJ_KAPPA,
       C_FLAGGED, C_ADMISSIBLE, C_EVAL_TERMS, C_REBUILDS, C_KFLOP, C_ELIMS, C_REFINED, C_CAND_JOBS, C_TRUNCATED, C_BIG_SCAN,
       C_EVAL_DEEP, C_REJ_VIS, C_NUM };

}  // namespace spoly
