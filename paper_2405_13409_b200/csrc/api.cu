// C-ABI of libspoly.so (include/spoly.h): context, mesh upload, solve orchestration on one stream.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace spoly;

namespace {

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(n, 1);
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Grows b to hold `need` elements, keeping its first `used` elements (stream-ordered copy).
template <class T>
static cudaError_t grow_keep(DBuf<T>& b, size_t used, size_t need, cudaStream_t st) {
  if (need <= b.cap && b.p) return cudaSuccess;
  const size_t want = std::max<size_t>({need, b.cap + b.cap / 2, 1});
  T* np = nullptr;
  cudaError_t e = cudaMalloc(&np, want * sizeof(T));
  if (e != cudaSuccess) return e;
  if (used) {
    e = cudaMemcpyAsync(np, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      cudaFree(np);
      return e;
    }
  }
  if (b.p) cudaFree(b.p);
  b.p = np;
  b.cap = want;
  return cudaSuccess;
}

}  // namespace

struct spoly_ctx {
  int device = 0;
  int nsm = 148;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  spoly_config cfg;
  std::string err;
  // mesh
  bool has_mesh = false;
  DeviceMesh M;
  DBuf<TriRec> d_tris, d_occ;
  DBuf<TriRec> d_tris_base;  // uploaded records while glossy normal offsets are applied (reading R28)
  bool has_base = false;
  DBuf<double> d_slopes, d_acc;
  DBuf<float4> d_box[kMaxAabbLevels], d_obox[kMaxAabbLevels];  // visibility hierarchies (mesh, occluders)
  AabbTree mesh_tree, occ_tree;
  DBuf<uint8_t> d_vkeep;
  DBuf<uint32_t> d_vsel, d_viota;
  DBuf<unsigned long long> d_vkey, d_vn;
  DBuf<double> d_vbary, d_vcontrib;
  DBuf<float> d_vresid;
  DBuf<TriCull> d_tcull;
  DBuf<uint32_t> d_orig, d_perm;
  DBuf<ClusterRec> d_cl, d_sub, d_up[4];
  DBuf<uint32_t> d_tlist, d_tcount, d_qkeys, d_qorder;
  DBuf<float> d_qbounds;
  uint32_t tile_cap = 4096, tile_used_cap = 4096;
  // work list
  DBuf<uint64_t> d_counts;
  DBuf<unsigned long long> d_offsets, d_emask;
  DBuf<uint32_t> d_pq, d_pt, d_pt_orig, d_pq2, d_pt2, d_pqa, d_pta;
  DBuf<uint32_t> d_vr, d_vr2, d_vra;  // k=2: per-pair v-range of the surviving cull cells (reading R25)
  DBuf<float4> d_tsph;                 // k=2 query tiles: endpoint spheres
  DBuf<uint32_t> d_tq, d_tp;           // k=2 query tiles: (tile, T_1, T_2) lists
  DBuf<unsigned long long> d_toff, d_moff;
  bool have_vr = false;
  uint32_t k2_chunk = 0;  // queries per two-bounce cull chunk (learned; reset by mesh upload)
  DBuf<unsigned char> d_keep;
  DBuf<unsigned int> d_lerr;  // explicit tuple list validation word
  DBuf<uint32_t> d_qmask;
  DBuf<uint64_t> d_front;
  DBuf<unsigned long long> d_fcount;
  DBuf<uint32_t> d_fr[2][3];
  DBuf<double> d_rec;
  DBuf<uint32_t> d_plist, d_clist;
  DBuf<unsigned long long> d_nsel;
  uint64_t npairs = 0, npairs_culled = 0, cull_tests = 0;
  int last_k = 1;
  // raw sink + job list
  DBuf<unsigned long long> d_count, d_counters, d_key, d_key2, d_fkey, d_fkey2, d_upair, d_nruns;
  DBuf<unsigned long long> d_pmask;  // counting order: one slot bit per (pair, slot)
  DBuf<unsigned long long> d_qrange;  // per-query [begin, end) in the sorted solution list
  DBuf<uint32_t> d_pcnt;             // counting order: per-pair counts, then their exclusive scan
  DBuf<uint32_t> d_fflags, d_fflags2, d_uflags, d_perm_in, d_perm_out, d_jpair, d_jmeta;
  DBuf<double> d_bary, d_contrib, d_jr, d_jroot;
  DBuf<float> d_resid;
  // sorted output
  DBuf<uint32_t> o_query, o_tuple, o_flags, o_fquery, o_ftuple, o_fflags;
  DBuf<double> o_bary, o_contrib, o_per_query;
  DBuf<float> o_resid;
  DBuf<unsigned char> d_temp;
  DBuf<uint32_t> d_k32;
  // host staging
  DBuf<double> d_ep, d_int;
  double* h_pinned = nullptr;
  size_t h_pinned_cap = 0;
  cudaEvent_t ev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  uint32_t launches = 0;
};

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);              \
      return e_ == cudaErrorMemoryAllocation ? SPOLY_ERR_OOM : SPOLY_ERR_CUDA;    \
    }                                                                             \
  } while (0)

static spoly_status fail(spoly_ctx* ctx, spoly_status s, const char* msg) {
  if (ctx) ctx->err = msg;
  return s;
}

extern "C" {

spoly_status spoly_default_config(spoly_config* c) {
  if (!c) return SPOLY_ERR_INVALID_ARG;
  c->pieces = 100;
  c->scan_bisect_iters = 10;
  c->bisect_tol = 1e-9;
  c->polish_iters = 5;
  c->theta_admit = 3e-2;
  c->theta_final = 1e-6;
  c->eps_domain = 1e-9;
  c->eps_flag = 1e-6;
  c->tau_trunc = 1e-12;
  c->cull = 1;
  c->deterministic = 1;
  c->cull_margin = 1e-4f;
  c->max_solutions = 1ull << 22;
  c->max_pairs = 1ull << 27;
  c->cull_levels = 3;
  c->visibility = 0;
  c->scan_restrict = 1;
  c->k2_tiles = 1;
  return SPOLY_OK;
}

spoly_status spoly_create(int dev, const spoly_config* cfg, void* stream, spoly_ctx** out) {
  if (!out) return SPOLY_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev < 0 || dev >= ndev) return SPOLY_ERR_CUDA;
  spoly_ctx* ctx = new spoly_ctx;
  ctx->device = dev;
  if (cfg)
    ctx->cfg = *cfg;
  else
    spoly_default_config(&ctx->cfg);
  if (cudaSetDevice(dev) != cudaSuccess) {
    delete ctx;
    return SPOLY_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, dev);
  if (stream) {
    ctx->st = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return SPOLY_ERR_CUDA;
    }
    ctx->own_stream = true;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  *out = ctx;
  return SPOLY_OK;
}

void spoly_destroy(spoly_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->st);
  ctx->d_tris.release(); ctx->d_occ.release(); ctx->d_tcull.release();
  ctx->d_tris_base.release(); ctx->d_slopes.release(); ctx->d_acc.release();
  for (auto& b : ctx->d_box) b.release();
  for (auto& b : ctx->d_obox) b.release();
  ctx->d_vkeep.release(); ctx->d_vsel.release(); ctx->d_viota.release(); ctx->d_vkey.release(); ctx->d_vn.release();
  ctx->d_vbary.release(); ctx->d_vcontrib.release(); ctx->d_vresid.release(); ctx->d_orig.release(); ctx->d_perm.release(); ctx->d_cl.release();
  ctx->d_sub.release(); for (auto& u : ctx->d_up) u.release(); ctx->d_tlist.release(); ctx->d_tcount.release(); ctx->d_qkeys.release();
  ctx->d_qorder.release(); ctx->d_qbounds.release();
  ctx->d_counts.release(); ctx->d_offsets.release(); ctx->d_emask.release(); ctx->d_pq.release(); ctx->d_pt.release(); ctx->d_pqa.release(); ctx->d_pta.release(); ctx->d_pt_orig.release();
  ctx->d_pq2.release(); ctx->d_pt2.release(); ctx->d_vr.release(); ctx->d_vr2.release(); ctx->d_vra.release();
  ctx->d_tsph.release(); ctx->d_tq.release(); ctx->d_tp.release(); ctx->d_toff.release(); ctx->d_moff.release();
  ctx->d_keep.release(); ctx->d_lerr.release(); ctx->d_nsel.release();
  ctx->d_rec.release(); ctx->d_plist.release(); ctx->d_clist.release(); ctx->d_qmask.release(); ctx->d_front.release(); ctx->d_fcount.release();
  for (auto& f : ctx->d_fr)
    for (auto& b : f) b.release();
  ctx->d_count.release(); ctx->d_counters.release(); ctx->d_key.release(); ctx->d_key2.release();
  ctx->d_fkey.release(); ctx->d_fkey2.release(); ctx->d_upair.release(); ctx->d_nruns.release();
  ctx->d_fflags.release(); ctx->d_fflags2.release(); ctx->d_uflags.release(); ctx->d_perm_in.release();
  ctx->d_perm_out.release(); ctx->d_jpair.release(); ctx->d_jmeta.release(); ctx->d_jr.release(); ctx->d_jroot.release();
  ctx->d_bary.release(); ctx->d_contrib.release(); ctx->d_resid.release();
  ctx->d_pmask.release(); ctx->d_pcnt.release(); ctx->d_qrange.release();
  ctx->o_query.release(); ctx->o_tuple.release(); ctx->o_flags.release(); ctx->o_fquery.release();
  ctx->o_ftuple.release(); ctx->o_fflags.release(); ctx->o_bary.release(); ctx->o_contrib.release();
  ctx->o_per_query.release(); ctx->o_resid.release(); ctx->d_temp.release(); ctx->d_k32.release(); ctx->d_ep.release(); ctx->d_int.release();
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->st);
  delete ctx;
}

const char* spoly_last_error(const spoly_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

// triangle order along the 30-bit Morton code of the centroids in the mesh's bounding box (host, scene setup);
// returns false on a degenerate triangle (|e1 x e2| <= 1e-12 diag^2)
static bool morton_order(const float* pos, uint32_t nverts, const uint32_t* tri, uint32_t ntris, std::vector<uint32_t>& order,
                         bool check_degenerate) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint32_t v = 0; v < nverts; ++v)
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], (double)pos[3ull * v + c]);
      hi[c] = std::max(hi[c], (double)pos[3ull * v + c]);
    }
  const double diag2 = (hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                       (hi[2] - lo[2]) * (hi[2] - lo[2]);
  std::vector<uint64_t> key(ntris);
  for (uint32_t t = 0; t < ntris; ++t) {
    double P[3][3];
    for (int j = 0; j < 3; ++j)
      for (int c = 0; c < 3; ++c) P[j][c] = pos[3ull * tri[3ull * t + j] + c];
    double e1[3], e2[3];
    for (int c = 0; c < 3; ++c) {
      e1[c] = P[1][c] - P[0][c];
      e2[c] = P[2][c] - P[0][c];
    }
    double g[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    if (check_degenerate && !(std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]) > 1e-12 * diag2)) return false;
    uint32_t code = 0;
    uint32_t ix[3];
    for (int c = 0; c < 3; ++c) {
      double m = (P[0][c] + P[1][c] + P[2][c]) / 3.0;
      double sc = hi[c] > lo[c] ? (m - lo[c]) / (hi[c] - lo[c]) : 0.0;
      ix[c] = (uint32_t)std::min(1023.0, std::max(0.0, sc * 1024.0));
    }
    for (int b = 9; b >= 0; --b)
      for (int c = 0; c < 3; ++c) code = (code << 1) | ((ix[c] >> b) & 1u);
    key[t] = ((uint64_t)code << 32) | t;
  }
  std::sort(key.begin(), key.end());
  order.resize(ntris);
  for (uint32_t i = 0; i < ntris; ++i) order[i] = (uint32_t)(key[i] & 0xffffffffu);
  return true;
}

// AABB hierarchy (visibility) over the triangle records recs: levels in bufs, tree in T
static spoly_status build_tree(spoly_ctx* ctx, const TriRec* recs, uint32_t ntris, DBuf<float4>* bufs, AabbTree& T) {
  T = AabbTree();
  T.tris = recs;
  T.top = aabb_levels(ntris, T.n);
  for (int l = 1; l <= T.top; ++l) {
    CK(bufs[l].ensure(2ull * T.n[l]));
    T.box[l] = bufs[l].p;
  }
  launch_build_aabbs(recs, T, ctx->st);
  CK(cudaGetLastError());
  return SPOLY_OK;
}

spoly_status spoly_upload_occluders(spoly_ctx* ctx, const float* pos, uint32_t nverts, const uint32_t* tri,
                                    uint32_t ntris) {
  if (!ctx) return SPOLY_ERR_INVALID_ARG;
  CK(cudaSetDevice(ctx->device));
  if (ntris == 0) {
    ctx->occ_tree = AabbTree();
    return SPOLY_OK;
  }
  if (!pos || !tri || nverts == 0) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null occluder mesh");
  for (uint64_t i = 0; i < 3ull * ntris; ++i)
    if (tri[i] >= nverts) return fail(ctx, SPOLY_ERR_BAD_MESH, "occluder index out of range");
  for (uint64_t i = 0; i < 3ull * nverts; ++i)
    if (!std::isfinite(pos[i])) return fail(ctx, SPOLY_ERR_BAD_MESH, "non-finite occluder vertex");
  std::vector<uint32_t> order;
  morton_order(pos, nverts, tri, ntris, order, false);
  float* dpos = nullptr;
  uint32_t *dtri = nullptr, *dorder = nullptr;
  CK(cudaMalloc(&dpos, sizeof(float) * 3ull * nverts));
  CK(cudaMalloc(&dtri, sizeof(uint32_t) * 3ull * ntris));
  CK(cudaMalloc(&dorder, sizeof(uint32_t) * ntris));
  CK(cudaMemcpyAsync(dpos, pos, sizeof(float) * 3ull * nverts, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dtri, tri, sizeof(uint32_t) * 3ull * ntris, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dorder, order.data(), sizeof(uint32_t) * ntris, cudaMemcpyHostToDevice, ctx->st));
  CK(ctx->d_occ.ensure(ntris));
  launch_occ_tris(dpos, dtri, dorder, ntris, ctx->d_occ.p, ctx->st);
  spoly_status s = build_tree(ctx, ctx->d_occ.p, ntris, ctx->d_obox, ctx->occ_tree);
  CK(cudaStreamSynchronize(ctx->st));
  cudaFree(dpos);
  cudaFree(dtri);
  cudaFree(dorder);
  return s;
}

// cluster bounds of the current triangle records: levels 1-2 and the upper levels of the implicit 8-ary hierarchy
// (two-bounce pair cull) until <= 8 nodes
static spoly_status build_bounds(spoly_ctx* ctx, uint32_t ntris) {
  const uint32_t ncl = (ntris + kClusterSize - 1) / kClusterSize;
  launch_build_clusters(ctx->d_tris.p, ntris, ctx->cfg.cull_margin, ctx->d_cl.p, ctx->d_sub.p, ctx->st);
  ctx->M.nupper = 0;
  uint64_t n = ncl, size = kClusterSize;
  for (int i = 0; i < 4 && n > 8; ++i) {
    size *= 8;
    n = (ntris + size - 1) / size;
    CK(ctx->d_up[i].ensure(n));
    launch_build_upper(ctx->d_tris.p, ntris, ctx->cfg.cull_margin, 3 + i, ctx->d_up[i].p, (uint32_t)n, ctx->st);
    ctx->M.upper[i] = ctx->d_up[i].p;
    ctx->M.nupper_nodes[i] = (uint32_t)n;
    ctx->M.nupper = i + 1;
  }
  return SPOLY_OK;
}

spoly_status spoly_upload_mesh(spoly_ctx* ctx, const float* pos, const float* nrm, uint32_t nverts, const uint32_t* tri,
                               uint32_t ntris, float eta_front, float eta_back, uint32_t* mesh_id) {
  if (!ctx || !pos || !nrm || !tri || ntris == 0 || nverts == 0) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null mesh");
  if (!(eta_front > 0) || !(eta_back > 0)) return fail(ctx, SPOLY_ERR_INVALID_ARG, "eta must be > 0");
  CK(cudaSetDevice(ctx->device));
  // host-side validation + Morton order of the centroids (one-time scene setup)
  for (uint64_t i = 0; i < 3ull * ntris; ++i)
    if (tri[i] >= nverts) return fail(ctx, SPOLY_ERR_BAD_MESH, "triangle index out of range");
  for (uint64_t i = 0; i < 3ull * nverts; ++i)
    if (!std::isfinite(pos[i]) || !std::isfinite(nrm[i])) return fail(ctx, SPOLY_ERR_BAD_MESH, "non-finite vertex");
  std::vector<uint32_t> order;
  if (!morton_order(pos, nverts, tri, ntris, order, true)) return fail(ctx, SPOLY_ERR_BAD_MESH, "degenerate triangle");

  float *dpos = nullptr, *dnrm = nullptr;
  uint32_t *dtri = nullptr, *dorder = nullptr;
  CK(cudaMalloc(&dpos, sizeof(float) * 3ull * nverts));
  CK(cudaMalloc(&dnrm, sizeof(float) * 3ull * nverts));
  CK(cudaMalloc(&dtri, sizeof(uint32_t) * 3ull * ntris));
  CK(cudaMalloc(&dorder, sizeof(uint32_t) * ntris));
  CK(cudaMemcpyAsync(dpos, pos, sizeof(float) * 3ull * nverts, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dnrm, nrm, sizeof(float) * 3ull * nverts, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dtri, tri, sizeof(uint32_t) * 3ull * ntris, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(dorder, order.data(), sizeof(uint32_t) * ntris, cudaMemcpyHostToDevice, ctx->st));
  const uint32_t ncl = (ntris + kClusterSize - 1) / kClusterSize, nsub = (ntris + kSubSize - 1) / kSubSize;
  CK(ctx->d_tris.ensure(ntris));
  CK(ctx->d_tcull.ensure(ntris));
  CK(ctx->d_orig.ensure(ntris));
  CK(ctx->d_perm.ensure(ntris));
  CK(ctx->d_cl.ensure(ncl));
  CK(ctx->d_sub.ensure(nsub));
  launch_build_tris(dpos, dnrm, dtri, dorder, ntris, ctx->cfg.cull_margin, ctx->d_tris.p, ctx->d_tcull.p,
                    ctx->d_orig.p, ctx->d_perm.p, ctx->st);
  {
    spoly_status bs = build_bounds(ctx, ntris);
    if (bs != SPOLY_OK) return bs;
  }
  {
    spoly_status bs = build_tree(ctx, ctx->d_tris.p, ntris, ctx->d_box, ctx->mesh_tree);
    if (bs != SPOLY_OK) return bs;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st));
  cudaFree(dpos);
  cudaFree(dnrm);
  cudaFree(dtri);
  cudaFree(dorder);
  ctx->M.ntris = ntris;
  ctx->M.nclusters = ncl;
  ctx->M.eta_front = eta_front;
  ctx->M.eta_back = eta_back;
  ctx->M.tris = ctx->d_tris.p;
  ctx->M.tcull = ctx->d_tcull.p;
  ctx->M.sub = ctx->d_sub.p;
  ctx->M.orig_id = ctx->d_orig.p;
  ctx->M.perm_of = ctx->d_perm.p;
  ctx->M.clusters = ctx->d_cl.p;
  ctx->has_mesh = true;
  ctx->has_base = false;
  ctx->k2_chunk = 0;
  if (mesh_id) *mesh_id = 0;
  return SPOLY_OK;
}

static SolSink raw_sink(spoly_ctx* ctx) {
  SolSink S;
  S.count = ctx->d_count.p;
  S.capacity = ctx->d_key.cap;
  S.key = ctx->d_key.p;
  S.bary = ctx->d_bary.p;
  S.contrib = ctx->d_contrib.p;
  S.resid = ctx->d_resid.p;
  S.fcapacity = ctx->d_fkey.cap;
  S.fkey = ctx->d_fkey.p;
  S.fflags = ctx->d_fflags.p;
  S.counters = ctx->d_counters.p;
  return S;
}

static spoly_status ensure_sink(spoly_ctx* ctx, uint64_t nsol, uint64_t nflag, int k) {
  CK(ctx->d_key.ensure(nsol));
  CK(ctx->d_bary.ensure(nsol * 2 * k));
  CK(ctx->d_contrib.ensure(nsol));
  CK(ctx->d_resid.ensure(nsol));
  CK(ctx->d_fkey.ensure(nflag));
  CK(ctx->d_fflags.ensure(nflag));
  // keep all arrays at equal capacity so S.capacity bounds every write
  ctx->d_key.cap = std::min({ctx->d_key.cap, ctx->d_contrib.cap, ctx->d_resid.cap, ctx->d_bary.cap / (2 * k)});
  ctx->d_fkey.cap = std::min(ctx->d_fkey.cap, ctx->d_fflags.cap);
  return SPOLY_OK;
}

struct BitOr {
  __host__ __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a | b; }
};

static int bits_for(uint64_t n) {
  int b = 1;
  while (b < 64 && (1ull << b) <= n) ++b;
  return b;
}

// Two-bounce pair cull of the query chunk [q0, q0 + qn): level-synchronous node-pair expansion from the
// split level down to triangle pairs (count pass, scan, write pass per level), then the barycentric
// subdivision refinement and an order-preserving compaction.  On return (*kq, *kt) point at the kept
// (query, T1, T2) list of *nkept entries (ctx-owned scratch, valid until the next chunk).  If a level's
// frontier would exceed `budget` entries nothing is written and *over is set to its size.
// Tiled variant (order != NULL): q0 / qn are SORTED positions, multiples of 32 (tiles of 32 Morton-sorted queries,
// the last one ragged); the expansion runs once per tile against the tile's endpoint spheres, then every query
// tests its tile's triangle pairs exactly (launch_query_pairs).  The coarse list is query-major in sorted order.
static spoly_status cull_k2_chunk(spoly_ctx* ctx, const char* chain, const double* endpoints, uint32_t q0,
                                  uint32_t qn, int top, uint32_t P, uint64_t budget, uint64_t* ncoarse,
                                  uint64_t* nkept, const uint32_t** kq, const uint32_t** kt, const uint32_t** kv,
                                  uint64_t* over, const uint32_t* order, uint32_t nq_total, uint32_t ts) {
  cudaStream_t st = ctx->st;
  const int v1t = chain[0] == 'T', v2t = chain[1] == 'T';
  const uint32_t *fq = nullptr, *fa = nullptr, *fb = nullptr;  // implicit root frontier of the chunk
  const uint32_t ntl = order ? (qn + ts - 1) / ts : 0;
  const float4* tsph = nullptr;
  if (order) {
    CK(ctx->d_tsph.ensure(2ull * ntl));
    launch_tile_spheres(endpoints, nq_total, order, q0, ntl, ts, ctx->d_tsph.p, ctx->nsm, st);
    tsph = ctx->d_tsph.p;
    ctx->launches++;
  }
  uint64_t nf = (uint64_t)(order ? ntl : qn) * P;
  int cur = 0;
  *over = 0;
  for (int cl = top - 1; cl >= 0; --cl) {
    CK(ctx->d_counts.ensure(nf / 2 + 1));
    CK(ctx->d_offsets.ensure(nf + 1));
    uint32_t* c32 = reinterpret_cast<uint32_t*>(ctx->d_counts.p);
    CK(ctx->d_emask.ensure(nf));
    launch_pair_expand(0, cl, endpoints, order ? 0 : q0, fq, fa, fb, nf, ctx->M, v1t, v2t, c32, ctx->d_emask.p,
                       nullptr, nullptr, nullptr, nullptr, ctx->nsm, st, tsph);
    ctx->cull_tests += nf * (64 + (fq ? 0 : 1));  // child node-pair tests (+ the root pair test)
    size_t tbytes = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tbytes, c32, ctx->d_offsets.p + 1, (int64_t)nf, st));
    CK(ctx->d_temp.ensure(tbytes));
    CK(cudaMemsetAsync(ctx->d_offsets.p, 0, sizeof(unsigned long long), st));
    CK(cub::DeviceScan::InclusiveSum(ctx->d_temp.p, tbytes, c32, ctx->d_offsets.p + 1, (int64_t)nf, st));
    unsigned long long tot = 0;
    CK(cudaMemcpyAsync(&tot, ctx->d_offsets.p + nf, sizeof(tot), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->launches += 2;
    if (tot > budget) {
      *over = tot;
      return SPOLY_OK;
    }
    if (cl == 0) {
      // per-query mode: the coarse list; tile mode: the tiles' triangle-pair lists (tile-major)
      CK((order ? ctx->d_tq : ctx->d_pq).ensure(tot));
      CK((order ? ctx->d_tp : ctx->d_pt).ensure(2 * tot));
      launch_pair_expand(1, cl, endpoints, order ? 0 : q0, fq, fa, fb, nf, ctx->M, v1t, v2t, nullptr, ctx->d_emask.p,
                         ctx->d_offsets.p, order ? ctx->d_tq.p : ctx->d_pq.p, order ? ctx->d_tp.p : ctx->d_pt.p,
                         nullptr, ctx->nsm, st, tsph);
    } else {
      const int nx = 1 - cur;
      for (int c = 0; c < 3; ++c) CK(ctx->d_fr[nx][c].ensure(tot));
      launch_pair_expand(1, cl, endpoints, order ? 0 : q0, fq, fa, fb, nf, ctx->M, v1t, v2t, nullptr, ctx->d_emask.p,
                         ctx->d_offsets.p, ctx->d_fr[nx][0].p, ctx->d_fr[nx][1].p, ctx->d_fr[nx][2].p, ctx->nsm, st,
                         tsph);
      fq = ctx->d_fr[nx][0].p;
      fa = ctx->d_fr[nx][1].p;
      fb = ctx->d_fr[nx][2].p;
      cur = nx;
    }
    nf = tot;
  }
  if (order) {
    // tile offsets of the tile-major pair list, the per-query mask layout, then the exact per-query pass
    const uint64_t ntp = nf;
    CK(ctx->d_toff.ensure(ntl + 1));
    CK(cudaMemsetAsync(ctx->d_toff.p, 0, (ntl + 1) * sizeof(unsigned long long), st));
    launch_tile_hist(ctx->d_tq.p, ntp, ctx->d_toff.p + 1, ctx->nsm, st);
    std::vector<unsigned long long> hoff(ntl + 1), hmoff(ntl + 1);
    CK(cudaMemcpyAsync(hoff.data(), ctx->d_toff.p, (ntl + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    hmoff[0] = 0;
    for (uint32_t t = 0; t < ntl; ++t) {
      const unsigned long long c = hoff[t + 1];
      hoff[t + 1] = hoff[t] + c;
      hmoff[t + 1] = hmoff[t] + (unsigned long long)ts * ((c + 31) / 32);
    }
    CK(ctx->d_moff.ensure(ntl + 1));
    CK(cudaMemcpyAsync(ctx->d_toff.p, hoff.data(), (ntl + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->d_moff.p, hmoff.data(), (ntl + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    CK(ctx->d_qmask.ensure(std::max<unsigned long long>(hmoff[ntl], 1)));
    CK(ctx->d_counts.ensure(qn / 2 + 1));
    CK(ctx->d_offsets.ensure(qn + 1));
    uint32_t* c32 = reinterpret_cast<uint32_t*>(ctx->d_counts.p);
    launch_query_pairs(0, endpoints, nq_total, order, q0, qn, ts, ctx->d_toff.p, ctx->d_tp.p, ctx->M, v1t, v2t,
                       ctx->d_moff.p, ctx->d_qmask.p, c32, nullptr, nullptr, nullptr, ctx->nsm, st);
    for (uint32_t t = 0; t < ntl; ++t)
      ctx->cull_tests += (hoff[t + 1] - hoff[t]) * (uint64_t)std::min<uint32_t>(ts, qn - ts * t);
    size_t tbytes = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tbytes, c32, ctx->d_offsets.p + 1, (int64_t)qn, st));
    CK(ctx->d_temp.ensure(tbytes));
    CK(cudaMemsetAsync(ctx->d_offsets.p, 0, sizeof(unsigned long long), st));
    CK(cub::DeviceScan::InclusiveSum(ctx->d_temp.p, tbytes, c32, ctx->d_offsets.p + 1, (int64_t)qn, st));
    unsigned long long tot = 0;
    CK(cudaMemcpyAsync(&tot, ctx->d_offsets.p + qn, sizeof(tot), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(ctx->d_pq.ensure(tot));
    CK(ctx->d_pt.ensure(2 * tot));
    launch_query_pairs(1, endpoints, nq_total, order, q0, qn, ts, ctx->d_toff.p, ctx->d_tp.p, ctx->M, v1t, v2t,
                       ctx->d_moff.p, ctx->d_qmask.p, nullptr, ctx->d_offsets.p, ctx->d_pq.p, ctx->d_pt.p, ctx->nsm,
                       st);
    ctx->launches += 5;
    nf = tot;
    if (tot > 4 * budget) {  // bound the chunk's coarse list (memory, refinement) like the frontiers
      *over = tot;
      return SPOLY_OK;
    }
  }
  const uint64_t npairs = nf;
  *ncoarse = npairs;
  *nkept = npairs;
  *kq = ctx->d_pq.p;
  *kt = ctx->d_pt.p;
  *kv = nullptr;
  if (ctx->cfg.cull_levels > 0 && npairs) {
    // barycentric subdivision refinement, then an order-preserving compaction (deterministic)
    CK(ctx->d_keep.ensure(npairs));
    CK(ctx->d_pq2.ensure(npairs));
    CK(ctx->d_pt2.ensure(2 * npairs));
    CK(ctx->d_vr2.ensure(2 * npairs));
    CK(ctx->d_nsel.ensure(4));
    {
      const uint64_t fcap = std::min<uint64_t>(std::max<uint64_t>(16 * npairs, 1ull << 20), 1ull << 27);
      CK(ctx->d_front.ensure(2 * fcap));
      CK(ctx->d_fcount.ensure(16));
      // blocks of coarse pairs small enough that a level's frontier (<= 16 children per entry) stays under the cap
      // (an overflowing entry keeps its pair: sound but loose)
      const uint64_t blk = std::max<uint64_t>(fcap / 16, 1);
      for (uint64_t b0 = 0; b0 < npairs; b0 += blk) {
        const uint64_t nb = std::min(blk, npairs - b0);
        RefineScratch RW{{ctx->d_front.p, ctx->d_front.p + fcap}, fcap, ctx->d_fcount.p, 0};
        launch_refine_pairs(ctx->d_pq.p + b0, ctx->d_pt.p + 2 * b0, nb, ctx->M, endpoints, ctx->cfg.cull_levels, v1t,
                            v2t, ctx->d_keep.p + b0, nullptr, RW, ctx->nsm, st);
        ctx->launches += RW.launches;
        unsigned long long fc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int lv = std::min(ctx->cfg.cull_levels, 5);
        CK(cudaMemcpyAsync(fc, ctx->d_fcount.p, sizeof(unsigned long long) * (size_t)lv, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        uint64_t entries = nb;  // level 0 runs on every coarse pair
        for (int l = 0; l < lv; ++l) {
          ctx->cull_tests += 16ull * entries;
          entries = std::min<uint64_t>(fc[l], fcap);
        }
      }
    }
    const uint2* pt_in = reinterpret_cast<const uint2*>(ctx->d_pt.p);
    uint2* pt_out = reinterpret_cast<uint2*>(ctx->d_pt2.p);
    size_t tb1 = 0, tb2 = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, tb1, ctx->d_pq.p, ctx->d_keep.p, ctx->d_pq2.p, ctx->d_nsel.p,
                                  (int64_t)npairs, st));
    CK(cub::DeviceSelect::Flagged(nullptr, tb2, pt_in, ctx->d_keep.p, pt_out, ctx->d_nsel.p + 1, (int64_t)npairs,
                                  st));
    CK(ctx->d_temp.ensure(std::max(tb1, tb2)));
    tb1 = tb2 = ctx->d_temp.cap;
    CK(cub::DeviceSelect::Flagged(ctx->d_temp.p, tb1, ctx->d_pq.p, ctx->d_keep.p, ctx->d_pq2.p, ctx->d_nsel.p,
                                  (int64_t)npairs, st));
    CK(cub::DeviceSelect::Flagged(ctx->d_temp.p, tb2, pt_in, ctx->d_keep.p, pt_out, ctx->d_nsel.p + 1,
                                  (int64_t)npairs, st));
    ctx->launches += 2;
    unsigned long long ns = 0;
    CK(cudaMemcpyAsync(&ns, ctx->d_nsel.p, sizeof(ns), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *nkept = ns;
    *kq = ctx->d_pq2.p;
    *kt = ctx->d_pt2.p;
    if (ns) {
      // reading R25: the v-range of T_1's surviving cells of every kept pair (the same refinement on the kept pairs
      // only, walking every surviving branch instead of stopping at the first)
      const uint64_t fcap = std::min<uint64_t>(std::max<uint64_t>(16 * ns, 1ull << 20), 1ull << 27);
      const uint64_t blk = std::max<uint64_t>(fcap / 16, 1);
      for (uint64_t b0 = 0; b0 < ns; b0 += blk) {
        const uint64_t nb = std::min<uint64_t>(blk, ns - b0);
        RefineScratch RW{{ctx->d_front.p, ctx->d_front.p + fcap}, fcap, ctx->d_fcount.p, 0};
        launch_refine_pairs(ctx->d_pq2.p + b0, ctx->d_pt2.p + 2 * b0, nb, ctx->M, endpoints, ctx->cfg.cull_levels, v1t,
                            v2t, ctx->d_keep.p + b0, ctx->d_vr2.p + 2 * b0, RW, ctx->nsm, st);
        ctx->launches += RW.launches + 1;
      }
      *kv = ctx->d_vr2.p;
    }
  }
  return SPOLY_OK;
}

// queries sorted along a 30-bit Morton code of their endpoints (k=1 and k=2 query tiles): *order[i] = query id
static spoly_status sort_queries(spoly_ctx* ctx, const double* endpoints, uint32_t nq, const uint32_t** order) {
  cudaStream_t st = ctx->st;
  CK(ctx->d_qbounds.ensure(12));
  CK(ctx->d_qkeys.ensure(2ull * nq));
  CK(ctx->d_qorder.ensure(2ull * nq));
  launch_query_order(endpoints, nq, ctx->d_qbounds.p, ctx->d_qkeys.p, ctx->d_qorder.p, st);
  ctx->launches += 2;
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ctx->d_qkeys.p, ctx->d_qkeys.p + nq, ctx->d_qorder.p,
                                     ctx->d_qorder.p + nq, (int)nq, 0, 30, st));
  CK(ctx->d_temp.ensure(tb));
  CK(cub::DeviceRadixSort::SortPairs(ctx->d_temp.p, tb, ctx->d_qkeys.p, ctx->d_qkeys.p + nq, ctx->d_qorder.p,
                                     ctx->d_qorder.p + nq, (int)nq, 0, 30, st));
  *order = ctx->d_qorder.p + nq;
  return SPOLY_OK;
}

spoly_status spoly_solve(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces, const double* endpoints,
                         uint32_t nq, const double* inten, const spoly_tuple_list* tuples, spoly_result* out) {
  if (!ctx || !chain || !out) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null argument");
  const int k = (int)strlen(chain);
  if (bounces != k || k < 1) return fail(ctx, SPOLY_ERR_INVALID_ARG, "bounces != strlen(chain)");
  if (strcmp(chain, "R") != 0 && strcmp(chain, "T") != 0 && strcmp(chain, "RR") != 0 && strcmp(chain, "TT") != 0 &&
      strcmp(chain, "RT") != 0 && strcmp(chain, "TR") != 0)
    return fail(ctx, SPOLY_ERR_UNSUPPORTED_CHAIN, "chain not supported by this build");
  if (!ctx->has_mesh || mesh_id != 0) return fail(ctx, SPOLY_ERR_INVALID_ARG, "no such mesh");
  if (nq && !endpoints) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null endpoints");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->st;
  ctx->launches = 0;
  ctx->have_vr = false;
  ctx->npairs_culled = 0;
  ctx->cull_tests = 0;
  memset(out, 0, sizeof(*out));
  out->k = k;
  CK(ctx->d_count.ensure(6));
  CK(ctx->d_counters.ensure(C_NUM));
  CK(ctx->o_per_query.ensure(nq));
  CK(cudaEventRecord(ctx->ev[0], st));

  // ---------------- work list
  uint64_t npairs = 0;
  if (tuples) {
    if (!tuples->offsets || !tuples->tri_ids) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null tuple list");
    uint32_t tot = 0;
    CK(cudaMemcpyAsync(&tot, tuples->offsets + nq, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    npairs = tot;
    CK(ctx->d_pq.ensure(npairs));
    CK(ctx->d_pt.ensure(npairs * k));
    CK(ctx->d_lerr.ensure(1));
    CK(cudaMemsetAsync(ctx->d_lerr.p, 0, sizeof(unsigned int), st));
    launch_expand_list(tuples->offsets, tuples->tri_ids, nq, k, ctx->M.perm_of, ctx->M.ntris, npairs, ctx->d_pq.p,
                       ctx->d_pt.p, ctx->d_lerr.p, ctx->nsm, st);
    ctx->launches++;
    unsigned int lerr = 0;
    CK(cudaMemcpyAsync(&lerr, ctx->d_lerr.p, sizeof(lerr), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (lerr & 1u) return fail(ctx, SPOLY_ERR_INVALID_ARG, "tuple list holds a triangle id >= ntris");
    if (lerr & 2u) return fail(ctx, SPOLY_ERR_INVALID_ARG, "tuple list offsets are not monotone");
  } else if (ctx->cfg.cull && k == 2) {
    // queries are culled in chunks whose node-pair frontiers fit cfg.max_pairs entries; the refined pair
    // lists of the chunks are appended in query order, so the work list equals the unchunked one
    uint32_t P = 0;
    const int top = cull_split_level(ctx->M, &P);
    if (top < 1) return fail(ctx, SPOLY_ERR_UNSUPPORTED_CHAIN, "two-bounce cull supports at most 2^22 triangles");
    const uint64_t budget = std::max<uint64_t>(ctx->cfg.max_pairs, 2ull * P);
    // query tiles (reading R14 on tiles): Morton order of the queries, chunks of whole tiles
    const uint32_t* order = nullptr;
    if (ctx->cfg.k2_tiles) {
      spoly_status os = sort_queries(ctx, endpoints, nq, &order);
      if (os != SPOLY_OK) return os;
    }
    uint32_t ts = order ? 32 : 1;  // queries per tile (halved when one tile alone exceeds the budget)
    uint32_t unit = ts;            // chunks in whole tiles
    uint32_t chunk = std::max<uint32_t>(unit, std::min<uint32_t>(ctx->k2_chunk ? ctx->k2_chunk : nq, nq));
    chunk = (uint32_t)std::max<uint64_t>(unit, std::min<uint64_t>(chunk, unit * std::max<uint64_t>(1, budget / P)));
    chunk = (chunk + unit - 1) / unit * unit;
    uint64_t acc = 0, coarse = 0;
    bool have_vr = ctx->cfg.cull_levels > 0;
    for (uint32_t q0 = 0; q0 < nq;) {
      const uint32_t qn = std::min(chunk, nq - q0);
      uint64_t ncoarse = 0, nkept = 0, over = 0;
      const uint32_t *kq = nullptr, *kt = nullptr, *kv = nullptr;
      spoly_status s = cull_k2_chunk(ctx, chain, endpoints, q0, qn, top, P, budget, &ncoarse, &nkept, &kq, &kt, &kv,
                                     &over, order, nq, ts);
      if (s != SPOLY_OK) return s;
      if (over) {  // a frontier of this chunk exceeded the budget: shrink the chunk (then the tiles) and redo it
        if (qn <= unit) {
          if (ts == 1) return fail(ctx, SPOLY_ERR_CAPACITY, "two-bounce cull frontier of one query exceeds max_pairs");
          ts /= 2;  // smaller tiles (their spheres are tighter, their union of pairs smaller); kept for the rest
          unit = ts;
          chunk = ts;
          continue;
        }
        chunk = (uint32_t)std::max<double>(1.0, std::min<double>(qn / 2, 0.9 * qn * (double)budget / (double)over));
        chunk = std::max<uint32_t>(unit, chunk / unit * unit);
        continue;
      }
      CK(grow_keep(ctx->d_pqa, acc, acc + nkept, st));
      CK(grow_keep(ctx->d_pta, 2 * acc, 2 * (acc + nkept), st));
      CK(grow_keep(ctx->d_vra, 2 * acc, 2 * (acc + nkept), st));
      if (nkept) {
        CK(cudaMemcpyAsync(ctx->d_pqa.p + acc, kq, nkept * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->d_pta.p + 2 * acc, kt, 2 * nkept * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        if (kv)
          CK(cudaMemcpyAsync(ctx->d_vra.p + 2 * acc, kv, 2 * nkept * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
      }
      if (nkept && !kv) have_vr = false;  // (cull_levels == 0: no cells, no ranges)
      acc += nkept;
      coarse += ncoarse;
      q0 += qn;
    }
    ctx->k2_chunk = chunk;
    CK(ctx->d_pqa.ensure(1));
    CK(ctx->d_pta.ensure(2));
    CK(ctx->d_vra.ensure(2));
    std::swap(ctx->d_pq, ctx->d_pqa);
    std::swap(ctx->d_pt, ctx->d_pta);
    ctx->have_vr = have_vr && acc > 0;
    ctx->npairs_culled = ctx->cfg.cull_levels > 0 ? coarse : 0;
    npairs = acc;
  } else if (ctx->cfg.cull) {
    // query order (Morton of the endpoints), tile cull, per-query cull on the tile survivors
    const uint32_t ntiles = (nq + 31) / 32;
    const uint32_t* order = nullptr;
    {
      spoly_status os = sort_queries(ctx, endpoints, nq, &order);
      if (os != SPOLY_OK) return os;
    }
    CK(ctx->d_tcount.ensure(ntiles + 1));
    for (int attempt = 0; attempt < 2; ++attempt) {
      const uint32_t cap = std::max<uint32_t>(64, std::min<uint32_t>(ctx->tile_cap, ctx->M.ntris));
      CK(ctx->d_tlist.ensure((uint64_t)ntiles * cap));
      CK(cudaMemsetAsync(ctx->d_tcount.p + ntiles, 0, sizeof(uint32_t), st));
      launch_tile_cull(endpoints, nq, order, ctx->M, chain[0] == 'T', cap, ctx->d_tlist.p, ctx->d_tcount.p,
                       reinterpret_cast<unsigned int*>(ctx->d_tcount.p + ntiles), ctx->nsm, st);
      ctx->launches++;
      uint32_t mx = 0;
      CK(cudaMemcpyAsync(&mx, ctx->d_tcount.p + ntiles, sizeof(mx), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (mx <= cap) {
        ctx->tile_used_cap = cap;
        break;
      }
      ctx->tile_cap = mx + mx / 8 + 64;  // regrow and redo (kept for later solves)
    }
    const uint32_t cap = ctx->tile_used_cap;
    CK(ctx->d_counts.ensure(nq));
    CK(ctx->d_offsets.ensure((uint64_t)nq + 1));
    uint32_t* c32 = reinterpret_cast<uint32_t*>(ctx->d_counts.p);
    CK(ctx->d_qmask.ensure((uint64_t)nq * ((cap + 31) / 32)));
    launch_query_cull(0, endpoints, nq, order, ctx->M, chain[0] == 'T', cap, ctx->d_tlist.p, ctx->d_tcount.p, c32,
                      ctx->d_qmask.p, nullptr, nullptr, nullptr, ctx->nsm, st);
    ctx->launches++;
    size_t tbytes = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tbytes, c32, ctx->d_offsets.p + 1, (int)nq, st));
    CK(ctx->d_temp.ensure(tbytes));
    CK(cudaMemsetAsync(ctx->d_offsets.p, 0, sizeof(unsigned long long), st));
    CK(cub::DeviceScan::InclusiveSum(ctx->d_temp.p, tbytes, c32, ctx->d_offsets.p + 1, (int)nq, st));
    unsigned long long tot = 0;
    CK(cudaMemcpyAsync(&tot, ctx->d_offsets.p + nq, sizeof(tot), cudaMemcpyDeviceToHost, st));
    {
      // cull work: every query tests its tile's surviving triangles (32 queries per tile; the last tile ragged)
      std::vector<uint32_t> tc(ntiles);
      CK(cudaMemcpyAsync(tc.data(), ctx->d_tcount.p, sizeof(uint32_t) * ntiles, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (uint32_t t = 0; t < ntiles; ++t) ctx->cull_tests += (uint64_t)tc[t] * std::min<uint32_t>(32, nq - 32 * t);
    }
    CK(cudaStreamSynchronize(st));
    npairs = tot;
    CK(ctx->d_pq.ensure(npairs));
    CK(ctx->d_pt.ensure(npairs * k));
    launch_query_cull(1, endpoints, nq, order, ctx->M, chain[0] == 'T', cap, ctx->d_tlist.p, ctx->d_tcount.p,
                      nullptr, ctx->d_qmask.p, ctx->d_offsets.p, ctx->d_pq.p, ctx->d_pt.p, ctx->nsm, st);
    ctx->launches++;
  } else {
    npairs = k == 1 ? (uint64_t)nq * ctx->M.ntris : (uint64_t)nq * ctx->M.ntris * (ctx->M.ntris - 1);
    CK(ctx->d_pq.ensure(npairs));
    CK(ctx->d_pt.ensure(npairs * k));
    if (k == 1)
      launch_all_pairs_k1(nq, ctx->M.ntris, ctx->d_pq.p, ctx->d_pt.p, st);
    else
      launch_all_pairs_k2(nq, ctx->M.ntris, ctx->d_pq.p, ctx->d_pt.p, st);
    ctx->launches++;
  }
  ctx->npairs = npairs;
  ctx->last_k = k;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[1], st));

  // ---------------- solve (regrow the sink once on overflow)
  SolveParams prm;
  prm.bisect_tol = ctx->cfg.bisect_tol;
  prm.theta_admit = ctx->cfg.theta_admit;
  prm.theta_final = ctx->cfg.theta_final;
  prm.eps_domain = ctx->cfg.eps_domain;
  prm.eps_flag = ctx->cfg.eps_flag;
  prm.tau_trunc = ctx->cfg.tau_trunc;
  prm.pieces = ctx->cfg.pieces;
  prm.scan_bisect_iters = ctx->cfg.scan_bisect_iters;
  prm.polish_iters = ctx->cfg.polish_iters;
  prm.eta_front = ctx->M.eta_front;
  prm.eta_back = ctx->M.eta_back;
  // initial sink capacities from the work list (an overflow re-runs the whole solve once): solutions
  // ~0.3 per pair on C2 (k=1), ~0.2% per refined pair for k=2; flagged tuples ~1e-5 (k=1) / ~1.3% (k=2)
  const uint64_t sol_guess = k == 1 ? npairs / 2 : npairs / 32;
  const uint64_t flag_guess = k == 1 ? npairs / 64 : npairs / 8;
  spoly_status s = ensure_sink(ctx, std::max({ctx->d_key.cap, (uint64_t)ctx->cfg.max_solutions, sol_guess}),
                               std::max({ctx->d_fkey.cap, (uint64_t)(1ull << 16), flag_guess}), k);
  if (s != SPOLY_OK) return s;
  CK(ctx->d_count.ensure(6));
  CK(ctx->d_jpair.ensure(k == 1 ? npairs : 1));
  CK(ctx->d_jmeta.ensure(k == 1 ? npairs : 1));
  CK(ctx->d_jr.ensure(k == 1 ? npairs * kJobStride : kJobStride));
  CK(ctx->d_jroot.ensure(k == 1 ? npairs : 1));
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  for (int attempt = 0; attempt < 2; ++attempt) {
    CK(cudaMemsetAsync(ctx->d_count.p, 0, 6 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(ctx->d_counters.p, 0, C_NUM * sizeof(unsigned long long), st));
    SolSink S = raw_sink(ctx);
    JobSink J;
    J.count = ctx->d_count.p + 2;
    J.capacity = std::min({ctx->d_jpair.cap, ctx->d_jr.cap / kJobStride, ctx->d_jroot.cap});
    J.pair = ctx->d_jpair.p;
    J.meta = ctx->d_jmeta.p;
    J.r = ctx->d_jr.p;
    J.root = ctx->d_jroot.p;
    CK(cudaEventRecord(ctx->ev[4], st));
    if (k == 1) {
      launch_solve_k1(1, chain[0] == 'T', ctx->d_pq.p, ctx->d_pt.p, npairs, ctx->M, endpoints, inten, prm, S, J,
                      ctx->nsm, st);
      CK(cudaEventRecord(ctx->ev[5], st));
      launch_solve_k1(2, chain[0] == 'T', ctx->d_pq.p, ctx->d_pt.p, npairs, ctx->M, endpoints, inten, prm, S, J,
                      ctx->nsm, st);
      CK(cudaEventRecord(ctx->ev[6], st));
      launch_solve_k1(3, chain[0] == 'T', ctx->d_pq.p, ctx->d_pt.p, npairs, ctx->M, endpoints, inten, prm, S, J,
                      ctx->nsm, st);
      ctx->launches += 4;
    } else {
      CK(cudaEventRecord(ctx->ev[5], st));
      {
        const uint64_t rb = k2_record_bytes(chain[0] == 'T', chain[1] == 'T') / sizeof(double);
        const uint64_t budget = (3ull << 30) / sizeof(double);  // <= 3 GiB of system records per chunk
        const uint64_t per = std::max<uint64_t>(1, std::min<uint64_t>(npairs, budget / rb));
        CK(ctx->d_rec.ensure(per * rb));
        CK(ctx->d_plist.ensure(per));
        CK(ctx->d_clist.ensure(8 * per));
        CK(ctx->d_nsel.ensure(4 + 24));
        K2Scratch W{ctx->d_rec.p, (ctx->d_rec.cap / rb) * rb, ctx->d_plist.p, ctx->d_clist.p, ctx->d_nsel.p + 4, 0};
        if (W.rec_cap / rb > ctx->d_plist.cap) W.rec_cap = ctx->d_plist.cap * rb;
        if (W.rec_cap / rb > ctx->d_clist.cap / 8) W.rec_cap = (ctx->d_clist.cap / 8) * rb;
        // the pairs' surviving-cell v-ranges restrict the determinant scan (reading R25); the d_vra buffer holds
        // them while the work list is the accumulated one (swapped into d_pq / d_pt above)
        launch_solve_k2(chain[0] == 'T', chain[1] == 'T', ctx->d_pq.p, ctx->d_pt.p,
                        ctx->have_vr && ctx->cfg.scan_restrict ? ctx->d_vra.p : nullptr, npairs, ctx->M, endpoints,
                        inten, prm, S, W, ctx->nsm, st);
        ctx->launches += W.launches - 1;
      }
      ctx->launches += 1;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(cnt, ctx->d_count.p, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cnt[2] + cnt[3] > J.capacity) return fail(ctx, SPOLY_ERR_CUDA, "job list overflow");
    if (cnt[0] <= S.capacity && cnt[1] <= S.fcapacity) break;
    if (attempt == 1) {
      out->report.required_solutions = cnt[0];
      return fail(ctx, SPOLY_ERR_CAPACITY, "solution buffer overflow after regrow");
    }
    s = ensure_sink(ctx, (uint64_t)(cnt[0] * 1.25) + 1024, (uint64_t)(cnt[1] * 1.25) + 1024, k);
    if (s != SPOLY_OK) return s;
  }
  // ---------------- visibility: drop chains with a blocked segment, keys preserved
  uint64_t n_raw = cnt[0];
  if (ctx->cfg.visibility && n_raw) {
    CK(ctx->d_vkeep.ensure(n_raw));
    CK(ctx->d_vsel.ensure(n_raw));
    CK(ctx->d_vn.ensure(1));
    launch_visibility(k, n_raw, raw_sink(ctx), ctx->d_pq.p, ctx->d_pt.p, endpoints, ctx->mesh_tree, ctx->occ_tree,
                      ctx->d_vkeep.p, ctx->nsm, st);
    size_t tb = 0;
    cub::CountingInputIterator<uint32_t> iota(0);
    CK(cub::DeviceSelect::Flagged(nullptr, tb, iota, ctx->d_vkeep.p, ctx->d_vsel.p, ctx->d_vn.p, (int64_t)n_raw, st));
    CK(ctx->d_temp.ensure(tb));
    CK(cub::DeviceSelect::Flagged(ctx->d_temp.p, tb, iota, ctx->d_vkeep.p, ctx->d_vsel.p, ctx->d_vn.p, (int64_t)n_raw,
                                  st));
    unsigned long long nk = 0;
    CK(cudaMemcpyAsync(&nk, ctx->d_vn.p, sizeof(nk), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(ctx->d_vkey.ensure(ctx->d_key.cap));
    CK(ctx->d_vbary.ensure(ctx->d_bary.cap));
    CK(ctx->d_vcontrib.ensure(ctx->d_contrib.cap));
    CK(ctx->d_vresid.ensure(ctx->d_resid.cap));
    launch_gather_raw(ctx->d_vsel.p, nk, k, raw_sink(ctx), ctx->d_vkey.p, ctx->d_vbary.p, ctx->d_vcontrib.p,
                      ctx->d_vresid.p, st);
    std::swap(ctx->d_key, ctx->d_vkey);
    std::swap(ctx->d_bary, ctx->d_vbary);
    std::swap(ctx->d_contrib, ctx->d_vcontrib);
    std::swap(ctx->d_resid, ctx->d_vresid);
    ctx->launches += 4;
    n_raw = nk;
  }
  CK(cudaEventRecord(ctx->ev[2], st));

  // ---------------- deterministic order + per-query sums
  const uint64_t n = n_raw, nf_raw = cnt[1];
  CK(ctx->o_query.ensure(n));
  CK(ctx->o_tuple.ensure(n * k));
  CK(ctx->o_bary.ensure(n * 2 * k));
  CK(ctx->o_contrib.ensure(n));
  CK(ctx->o_resid.ensure(n));
  CK(ctx->o_flags.ensure(n));
  CK(ctx->d_key2.ensure(n));
  CK(ctx->d_perm_in.ensure(n));
  CK(ctx->d_perm_out.ensure(n));
  CK(ctx->d_fkey2.ensure(nf_raw));
  CK(ctx->d_fflags2.ensure(nf_raw));
  CK(ctx->d_upair.ensure(nf_raw));
  CK(ctx->d_uflags.ensure(nf_raw));
  CK(ctx->d_nruns.ensure(1));
  SolSink in = raw_sink(ctx);
  OutArrays o;
  memset(&o, 0, sizeof(o));
  o.query = ctx->o_query.p;
  o.tuple = ctx->o_tuple.p;
  o.flags = ctx->o_flags.p;
  o.bary = ctx->o_bary.p;
  o.contrib = ctx->o_contrib.p;
  o.resid = ctx->o_resid.p;
  const int end_bit = std::min(64, 6 + bits_for(npairs));
  const int fbits = std::min(64, bits_for(npairs));
  // flags: sort the per-pair records, OR-reduce by pair
  uint64_t nf = 0;
  if (nf_raw) {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ctx->d_fkey.p, ctx->d_fkey2.p, ctx->d_fflags.p, ctx->d_fflags2.p,
                                       (int64_t)nf_raw, 0, fbits, st));
    CK(ctx->d_temp.ensure(tb));
    CK(cub::DeviceRadixSort::SortPairs(ctx->d_temp.p, tb, ctx->d_fkey.p, ctx->d_fkey2.p, ctx->d_fflags.p,
                                       ctx->d_fflags2.p, (int64_t)nf_raw, 0, fbits, st));
    tb = 0;
    CK(cub::DeviceReduce::ReduceByKey(nullptr, tb, ctx->d_fkey2.p, ctx->d_upair.p, ctx->d_fflags2.p, ctx->d_uflags.p,
                                      ctx->d_nruns.p, BitOr(), (int64_t)nf_raw, st));
    CK(ctx->d_temp.ensure(tb));
    CK(cub::DeviceReduce::ReduceByKey(ctx->d_temp.p, tb, ctx->d_fkey2.p, ctx->d_upair.p, ctx->d_fflags2.p,
                                      ctx->d_uflags.p, ctx->d_nruns.p, BitOr(), (int64_t)nf_raw, st));
    unsigned long long nr = 0;
    CK(cudaMemcpyAsync(&nr, ctx->d_nruns.p, sizeof(nr), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    nf = nr;
    CK(ctx->o_fquery.ensure(nf));
    CK(ctx->o_ftuple.ensure(nf * k));
    CK(ctx->o_fflags.ensure(nf));
    o.fquery = ctx->o_fquery.p;
    o.ftuple = ctx->o_ftuple.p;
    o.fflags = ctx->o_fflags.p;
    launch_gather_flagged(ctx->d_upair.p, ctx->d_uflags.p, nf, k, ctx->d_pq.p, ctx->d_pt.p, ctx->M.orig_id, o, st);
    ctx->launches++;
  }
  // counting order (same order as the key sort, without its radix passes) when the per-pair arrays (16 B
  // per pair, memset + scan) cost less than sorting the solutions: measured on B200, C3 (1.3 M pairs, 0.26 M
  // solutions) 0.46 -> 0.41 ms, C2 (24.5 M pairs, 7.7 M solutions) 0.71 -> 0.77 ms, i.e. counting pays
  // while npairs <~ 2 n + 4 M.  SPOLY_SORT_ORDER=1 / =0 forces the sort / the counting order (A/B, tests).
  const char* force = getenv("SPOLY_SORT_ORDER");
  const bool counting_fits = n && n < (1ull << 32) && npairs <= (1ull << 30);
  const bool counting = counting_fits && (force && force[0] == '1'   ? false
                                          : force && force[0] == '0' ? true
                                                                     : npairs <= 2 * n + (1ull << 22));
  if (counting) {
    CK(ctx->d_pmask.ensure(npairs));
    CK(ctx->d_pcnt.ensure(2 * npairs));
    CK(cudaMemsetAsync(ctx->d_pmask.p, 0, npairs * sizeof(unsigned long long), st));
    launch_slot_masks(ctx->d_key.p, n, ctx->d_pmask.p, npairs, ctx->d_pcnt.p, st);
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, ctx->d_pcnt.p, ctx->d_pcnt.p + npairs, (int64_t)npairs, st));
    CK(ctx->d_temp.ensure(tb));
    CK(cub::DeviceScan::ExclusiveSum(ctx->d_temp.p, tb, ctx->d_pcnt.p, ctx->d_pcnt.p + npairs, (int64_t)npairs, st));
    launch_scatter_solutions(ctx->d_key.p, n, ctx->d_pmask.p, ctx->d_pcnt.p + npairs, k, in, ctx->d_pq.p,
                             ctx->d_pt.p, ctx->M.orig_id, o, ctx->d_key2.p, st);
    launch_solution_flags(ctx->d_key2.p, nullptr, n, ctx->d_upair.p, ctx->d_uflags.p, nf, o.flags, st);
    ctx->launches += 4;
  } else if (n) {
    launch_iota(ctx->d_perm_in.p, n, st);
    ctx->launches++;
    size_t tb = 0;
    const uint32_t* k32 = nullptr;
    if (end_bit <= 32) {
      CK(ctx->d_k32.ensure(2 * n));
      launch_key32(ctx->d_key.p, n, ctx->d_k32.p, st);
      ctx->launches++;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ctx->d_k32.p, ctx->d_k32.p + n, ctx->d_perm_in.p,
                                         ctx->d_perm_out.p, (int64_t)n, 0, end_bit, st));
      CK(ctx->d_temp.ensure(tb));
      CK(cub::DeviceRadixSort::SortPairs(ctx->d_temp.p, tb, ctx->d_k32.p, ctx->d_k32.p + n, ctx->d_perm_in.p,
                                         ctx->d_perm_out.p, (int64_t)n, 0, end_bit, st));
      k32 = ctx->d_k32.p + n;
    } else {
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ctx->d_key.p, ctx->d_key2.p, ctx->d_perm_in.p,
                                         ctx->d_perm_out.p, (int64_t)n, 0, end_bit, st));
      CK(ctx->d_temp.ensure(tb));
      CK(cub::DeviceRadixSort::SortPairs(ctx->d_temp.p, tb, ctx->d_key.p, ctx->d_key2.p, ctx->d_perm_in.p,
                                         ctx->d_perm_out.p, (int64_t)n, 0, end_bit, st));
    }
    launch_gather_solutions(ctx->d_perm_out.p, ctx->d_key2.p, k32, n, k, in, ctx->d_pq.p, ctx->d_pt.p,
                            ctx->M.orig_id, o, st);
    launch_solution_flags(ctx->d_key2.p, k32, n, ctx->d_upair.p, ctx->d_uflags.p, nf, o.flags, st);
    ctx->launches += 2;
  }
  CK(ctx->d_qrange.ensure(2ull * nq));
  launch_per_query_sorted(ctx->o_query.p, ctx->o_contrib.p, n, nq, ctx->o_per_query.p, ctx->d_qrange.p, st);
  ctx->launches += n ? 2 : 1;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[3], st));
  unsigned long long counters[C_NUM];
  CK(cudaMemcpyAsync(counters, ctx->d_counters.p, sizeof(counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));

  out->n_solutions = n;
  out->n_flagged = nf;
  out->query = ctx->o_query.p;
  out->tuple = ctx->o_tuple.p;
  out->bary = ctx->o_bary.p;
  out->contribution = ctx->o_contrib.p;
  out->residual = ctx->o_resid.p;
  out->flags = ctx->o_flags.p;
  out->flagged_query = ctx->o_fquery.p;
  out->flagged_tuple = ctx->o_ftuple.p;
  out->flagged_flags = ctx->o_fflags.p;
  out->per_query = ctx->o_per_query.p;
  spoly_report& R = out->report;
  R.n_pairs_in = counters[C_PAIRS];
  R.n_systems = counters[C_SYSTEMS];
  R.n_vroots = counters[C_VROOTS];
  R.n_candidates = counters[C_CANDIDATES];
  R.n_rej_domain = counters[C_REJ_DOMAIN];
  R.n_rej_constraint = counters[C_REJ_CONSTRAINT];
  R.n_rej_side = counters[C_REJ_SIDE];
  R.n_rej_kappa = counters[C_REJ_KAPPA];
  R.n_flagged = nf;
  R.n_admissible = counters[C_ADMISSIBLE];
  cudaEventElapsedTime(&R.ms_cull, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&R.ms_solve, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&R.ms_reduce, ctx->ev[2], ctx->ev[3]);
  R.ms_phase1 = R.ms_phase2 = 0.f;
  if (npairs) {
    cudaEventElapsedTime(&R.ms_phase1, ctx->ev[4], ctx->ev[5]);
    cudaEventElapsedTime(&R.ms_phase2, ctx->ev[5], ctx->ev[2]);
  }
  R.ms_roots = R.ms_path = 0.f;
  if (npairs && k == 1) {
    cudaEventElapsedTime(&R.ms_roots, ctx->ev[5], ctx->ev[6]);
    cudaEventElapsedTime(&R.ms_path, ctx->ev[6], ctx->ev[2]);
  }
  R.n_rebuilds = counters[C_REBUILDS];
  R.alg_kflop = counters[C_KFLOP];
  R.n_elims = counters[C_ELIMS];
  R.n_pairs_coarse = ctx->npairs_culled;
  R.n_jobs_mono = counters[C_CAND_JOBS];
  R.n_jobs_deep = cnt[3];
  R.n_launches = ctx->launches;
  R.n_eval_terms = counters[C_EVAL_TERMS];
  R.n_refined = counters[C_REFINED];
  R.n_cand_jobs = counters[C_CAND_JOBS];
  R.n_path_jobs = cnt[2] + cnt[3];
  R.n_eval_deep = counters[C_EVAL_DEEP];
  R.n_rej_visibility = counters[C_REJ_VIS];
  R.n_cull_tests = ctx->cull_tests;
  R.n_truncated = counters[C_TRUNCATED];
  R.n_big_scan = counters[C_BIG_SCAN];
  return SPOLY_OK;
}

spoly_status spoly_solve_host(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces,
                              const double* ep_host, uint32_t nq, const double* int_host, double* per_query_host,
                              spoly_result* out) {
  if (!ctx || !ep_host || !per_query_host) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null argument");
  CK(cudaSetDevice(ctx->device));
  const size_t need = 7ull * nq;
  if (ctx->h_pinned_cap < need) {
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    ctx->h_pinned = nullptr;
    CK(cudaMallocHost(&ctx->h_pinned, need * sizeof(double)));
    ctx->h_pinned_cap = need;
  }
  CK(ctx->d_ep.ensure(6ull * nq));
  memcpy(ctx->h_pinned, ep_host, sizeof(double) * 6ull * nq);
  CK(cudaMemcpyAsync(ctx->d_ep.p, ctx->h_pinned, sizeof(double) * 6ull * nq, cudaMemcpyHostToDevice, ctx->st));
  const double* dint = nullptr;
  if (int_host) {
    CK(ctx->d_int.ensure(nq));
    memcpy(ctx->h_pinned + 6ull * nq, int_host, sizeof(double) * nq);
    CK(cudaMemcpyAsync(ctx->d_int.p, ctx->h_pinned + 6ull * nq, sizeof(double) * nq, cudaMemcpyHostToDevice, ctx->st));
    dint = ctx->d_int.p;
  }
  spoly_result tmp;
  spoly_result* r = out ? out : &tmp;
  spoly_status s = spoly_solve(ctx, mesh_id, chain, bounces, ctx->d_ep.p, nq, dint, nullptr, r);
  if (s != SPOLY_OK) return s;
  CK(cudaMemcpyAsync(ctx->h_pinned, r->per_query, sizeof(double) * nq, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  memcpy(per_query_host, ctx->h_pinned, sizeof(double) * nq);
  return SPOLY_OK;
}

spoly_status spoly_set_normal_offsets(spoly_ctx* ctx, const double* slopes, uint32_t ntris) {
  if (!ctx) return SPOLY_ERR_INVALID_ARG;
  if (!ctx->has_mesh) return fail(ctx, SPOLY_ERR_INVALID_ARG, "no mesh uploaded");
  const uint32_t n = ctx->M.ntris;
  if (slopes && ntris != n) return fail(ctx, SPOLY_ERR_INVALID_ARG, "slopes must hold 2 values per mesh triangle");
  for (uint64_t i = 0; slopes && i < 2ull * n; ++i)
    if (!std::isfinite(slopes[i])) return fail(ctx, SPOLY_ERR_INVALID_ARG, "non-finite slope");
  CK(cudaSetDevice(ctx->device));
  if (!slopes) {
    if (ctx->has_base)
      CK(cudaMemcpyAsync(ctx->d_tris.p, ctx->d_tris_base.p, sizeof(TriRec) * n, cudaMemcpyDeviceToDevice, ctx->st));
  } else {
    if (!ctx->has_base) {
      CK(ctx->d_tris_base.ensure(n));
      CK(cudaMemcpyAsync(ctx->d_tris_base.p, ctx->d_tris.p, sizeof(TriRec) * n, cudaMemcpyDeviceToDevice, ctx->st));
      ctx->has_base = true;
    }
    CK(ctx->d_slopes.ensure(2ull * n));
    CK(cudaMemcpyAsync(ctx->d_slopes.p, slopes, sizeof(double) * 2ull * n, cudaMemcpyHostToDevice, ctx->st));
  }
  if (ctx->has_base) {
    if (slopes)
      launch_perturb_tris(ctx->d_tris_base.p, ctx->d_slopes.p, ctx->M.orig_id, n, ctx->cfg.cull_margin, ctx->d_tris.p,
                          ctx->d_tcull.p, ctx->st);
    else
      launch_rebuild_tcull(ctx->d_tris.p, n, ctx->cfg.cull_margin, ctx->d_tcull.p, ctx->st);
    spoly_status bs = build_bounds(ctx, n);
    if (bs != SPOLY_OK) return bs;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st));
  return SPOLY_OK;
}

spoly_status spoly_render(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces, const double* endpoints,
                          uint32_t width, uint32_t height, const double* light_intensity, uint32_t nsamples,
                          const double* slopes, double albedo, double exposure, double* radiance, uint8_t* srgb) {
  if (!ctx || !endpoints || !radiance) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null argument");
  if (!ctx->has_mesh) return fail(ctx, SPOLY_ERR_INVALID_ARG, "no mesh uploaded");
  const uint64_t nq64 = (uint64_t)width * height;
  if (nq64 == 0 || nq64 > 0xffffffffull) return fail(ctx, SPOLY_ERR_INVALID_ARG, "bad image size");
  if (!(albedo >= 0) || !std::isfinite(albedo) || !(exposure >= 0)) return fail(ctx, SPOLY_ERR_INVALID_ARG, "bad albedo/exposure");
  const uint32_t nq = (uint32_t)nq64, S = nsamples ? nsamples : 1;
  CK(cudaSetDevice(ctx->device));
  CK(ctx->d_acc.ensure(nq));
  CK(cudaMemsetAsync(ctx->d_acc.p, 0, sizeof(double) * nq, ctx->st));
  const double scale = albedo / 3.14159265358979323846 / S;
  spoly_status s = SPOLY_OK;
  for (uint32_t i = 0; i < S && s == SPOLY_OK; ++i) {
    if (slopes) {
      s = spoly_set_normal_offsets(ctx, slopes + 2ull * ctx->M.ntris * i, ctx->M.ntris);
      if (s != SPOLY_OK) break;
    }
    spoly_result r;
    s = spoly_solve(ctx, mesh_id, chain, bounces, endpoints, nq, light_intensity, nullptr, &r);
    if (s == SPOLY_OK) launch_splat(r.per_query, nq, scale, ctx->d_acc.p, ctx->st);
  }
  if (slopes) {
    spoly_status r2 = spoly_set_normal_offsets(ctx, nullptr, 0);
    if (s == SPOLY_OK) s = r2;
  }
  if (s != SPOLY_OK) return s;
  CK(cudaMemcpyAsync(radiance, ctx->d_acc.p, sizeof(double) * nq, cudaMemcpyDeviceToDevice, ctx->st));
  if (srgb) launch_tonemap(ctx->d_acc.p, nq, exposure, srgb, ctx->st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st));
  return SPOLY_OK;
}

spoly_status spoly_last_worklist(const spoly_ctx* ctx, const uint32_t** pq, const uint32_t** pt, uint64_t* n) {
  if (!ctx || !pq || !pt || !n) return SPOLY_ERR_INVALID_ARG;
  spoly_ctx* c = const_cast<spoly_ctx*>(ctx);
  if (c->d_pt_orig.ensure(std::max<uint64_t>(c->npairs * c->last_k, 1)) != cudaSuccess) return SPOLY_ERR_OOM;
  launch_map_ids(c->d_pt.p, c->npairs * c->last_k, c->M.orig_id, c->d_pt_orig.p, c->st);
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return SPOLY_ERR_CUDA;
  *pq = c->d_pq.p;
  *pt = c->d_pt_orig.p;
  *n = c->npairs;
  return SPOLY_OK;
}

spoly_status spoly_sqrt_table(spoly_ctx* ctx, int from_device, double* out30) {
  if (!out30 || (from_device && !ctx)) return fail(ctx, SPOLY_ERR_INVALID_ARG, "null argument");
  if (from_device) CK(cudaSetDevice(ctx->device));
  cudaError_t e = k2_sqrt_table(from_device, out30);
  if (e != cudaSuccess) {
    if (ctx) ctx->err = cudaGetErrorString(e);
    return SPOLY_ERR_CUDA;
  }
  return SPOLY_OK;
}

spoly_status spoly_bench_fma(spoly_ctx* ctx, int fp64, double seconds, double* flops) {
  if (!ctx || !flops) return SPOLY_ERR_INVALID_ARG;
  CK(cudaSetDevice(ctx->device));
  double* sink = nullptr;
  CK(cudaMalloc(&sink, sizeof(double)));
  int blocks, threads, fpt;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 256;
  float ms = 0;
  for (int rep = 0; rep < 8; ++rep) {
    cudaEventRecord(a, ctx->st);
    launch_fma_peak(fp64, iters, sink, ctx->nsm, ctx->st, &blocks, &threads, &fpt);
    cudaEventRecord(b, ctx->st);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    if (ms > 1000.0 * seconds * 0.5) break;
    iters = (int)std::min(1e9, iters * std::max(2.0, 1000.0 * seconds / std::max(ms, 0.01f)));
  }
  *flops = (double)blocks * threads * fpt * (double)iters / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return SPOLY_OK;
}

}  // extern "C"
