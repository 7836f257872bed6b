// Host-visible launchers of the CUDA kernels (implemented in the .cu files of csrc/).
#pragma once
#include "common.cuh"

namespace spoly {

// mesh.cu
void launch_build_tris(const float* pos, const float* nrm, const uint32_t* tri, const uint32_t* order, uint32_t ntris,
                       float margin, TriRec* recs, TriCull* tc, uint32_t* orig_id, uint32_t* perm_of,
                       cudaStream_t st);
void launch_build_upper(const TriRec* recs, uint32_t ntris, float margin, int level, ClusterRec* out, uint32_t n,
                        cudaStream_t st);
void launch_build_clusters(const TriRec* recs, uint32_t ntris, float margin, ClusterRec* l1, ClusterRec* l2,
                           cudaStream_t st);
void launch_perturb_tris(const TriRec* base, const double* slopes, const uint32_t* orig_id, uint32_t ntris,
                         float margin, TriRec* recs, TriCull* tc, cudaStream_t st);
void launch_rebuild_tcull(const TriRec* recs, uint32_t ntris, float margin, TriCull* tc, cudaStream_t st);
void launch_splat(const double* per_query, uint32_t nq, double scale, double* acc, cudaStream_t st);
void launch_tonemap(const double* L, uint32_t nq, double exposure, uint8_t* rgb, cudaStream_t st);

// cull.cu: query-coherent hierarchical cone cull (tiles of 32 Morton-sorted queries, then per query)
void launch_query_order(const double* ep, uint32_t nq, float* bounds, uint32_t* keys, uint32_t* idx,
                        cudaStream_t st);
void launch_tile_cull(const double* ep, uint32_t nq, const uint32_t* order, const DeviceMesh& M, int refract,
                      uint32_t cap, uint32_t* tile_list, uint32_t* tile_count, unsigned int* max_count, int nsm,
                      cudaStream_t st);
// pass 0: tests -> keep masks + per-query counts; pass 1: query-major list from the masks
void launch_query_cull(int pass, const double* ep, uint32_t nq, const uint32_t* order, const DeviceMesh& M,
                       int refract, uint32_t cap, const uint32_t* tile_list, const uint32_t* tile_count,
                       uint32_t* counts, uint32_t* masks, const unsigned long long* offsets, uint32_t* pq,
                       uint32_t* pt, int nsm, cudaStream_t st);
void launch_all_pairs_k1(uint32_t nq, uint32_t ntris, uint32_t* pair_query, uint32_t* pair_tpos, cudaStream_t st);
// explicit tuple list -> work list; *err |= 1 for an id >= ntris, 2 for a malformed CSR row (err zeroed by the caller)
void launch_expand_list(const uint32_t* offsets, const uint32_t* tri_ids, uint32_t nq, int k, const uint32_t* perm_of,
                        uint32_t ntris, uint64_t total, uint32_t* pair_query, uint32_t* pair_tpos, unsigned int* err,
                        int nsm, cudaStream_t st);

// solve_k1.cu
void launch_solve_k1(int phase, int refract, const uint32_t* pq, const uint32_t* pt, uint64_t npairs,
                     const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                     const SolSink& S, const JobSink& J, int nsm, cudaStream_t st);

// solve_k2.cu
// two-bounce scratch: per-pair system records (chunked), path list, counters
struct K2Scratch {
  double* rec;
  uint64_t rec_cap;  // doubles
  uint32_t* plist;   // >= rec_cap / stride entries
  uint32_t* clist;   // 8 * (rec_cap / stride) entries: per order class
  unsigned long long* ctr;  // 24
  int launches;
};
uint64_t k2_record_bytes(int v1t, int v2t);
// the Eq. 20 sqrt surrogate table (6 x (lo, hi, c0, c1, d1)): host copy, or read back from constant memory
cudaError_t k2_sqrt_table(int from_device, double* out30);
// vrange: per pair [lo, hi] v-range (1/32 units) of the surviving cull cells, or NULL (whole [0, 1])
void launch_solve_k2(int v1t, int v2t, const uint32_t* pq, const uint32_t* pt, const uint32_t* vrange, uint64_t npairs,
                     const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                     const SolSink& S, K2Scratch& W, int nsm, cudaStream_t st);
// two-bounce pair cull: split level of the implicit hierarchy (-1: > 2^22 triangles) and one expansion pass
int cull_split_level(const DeviceMesh& M, uint32_t* pairs_per_query);
void launch_pair_expand(int pass, int cl, const double* ep, uint32_t qbase, const uint32_t* fq, const uint32_t* fa,
                        const uint32_t* fb, uint64_t nf, const DeviceMesh& M, int v1t, int v2t, uint32_t* counts,
                        unsigned long long* masks, const unsigned long long* offsets, uint32_t* oq, uint32_t* oa, uint32_t* ob, int nsm,
                        cudaStream_t st, const float4* tsph = nullptr);
// two-bounce query tiles (32 Morton-sorted queries): endpoint spheres of tiles [0, ntiles) starting at sorted
// position s0; per-query exact test of the tile's triangle pairs (pass 0 masks + counts, pass 1 list)
void launch_tile_spheres(const double* ep, uint32_t nq, const uint32_t* order, uint32_t s0, uint32_t ntiles,
                         uint32_t ts, float4* tsph, int nsm, cudaStream_t st);
void launch_query_pairs(int pass, const double* ep, uint32_t nq, const uint32_t* order, uint32_t s0, uint32_t sn,
                        uint32_t ts, const unsigned long long* toff, const uint32_t* tpair, const DeviceMesh& M,
                        int v1t, int v2t, const unsigned long long* moff, uint32_t* masks, uint32_t* counts,
                        const unsigned long long* offsets, uint32_t* oq, uint32_t* ot, int nsm, cudaStream_t st);
void launch_tile_hist(const uint32_t* tq, uint64_t n, unsigned long long* cnt, int nsm, cudaStream_t st);
struct RefineScratch {
  uint64_t* front[2];  // frontier ping-pong, cap entries each
  uint64_t cap;
  unsigned long long* count;  // >= 2 * levels
  int launches;
};
// keep[i] = 1 for the pairs some subdivision cell pair survives `levels` deep; vrange (optional, 2 x uint32 per pair):
// [lo, hi] v-range of T_1's surviving cells in units of 1/32 (reading R25)
void launch_refine_pairs(const uint32_t* pq, const uint32_t* pt, uint64_t n, const DeviceMesh& M, const double* ep,
                         int levels, int v1t, int v2t, uint8_t* keep, uint32_t* vrange, RefineScratch& W, int nsm,
                         cudaStream_t st);
void launch_all_pairs_k2(uint32_t nq, uint32_t ntris, uint32_t* pair_query, uint32_t* pair_tpos, cudaStream_t st);

// reduce.cu
struct OutArrays {
  uint32_t *query, *tuple, *flags, *fquery, *ftuple, *fflags;
  double *bary, *contrib;
  float* resid;
};
void launch_map_ids(const uint32_t* tpos, uint64_t n, const uint32_t* orig_id, uint32_t* out, cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st);
void launch_gather_solutions(const uint32_t* perm, const unsigned long long* skey, const uint32_t* skey32, uint64_t n,
                             int k, const SolSink& in, const uint32_t* pq, const uint32_t* pt, const uint32_t* orig_id,
                             const OutArrays& out, cudaStream_t st);
void launch_slot_masks(const unsigned long long* key, uint64_t n, unsigned long long* mask, uint64_t npairs,
                       uint32_t* cnt, cudaStream_t st);
void launch_scatter_solutions(const unsigned long long* key, uint64_t n, const unsigned long long* mask,
                              const uint32_t* off, int k, const SolSink& in, const uint32_t* pq, const uint32_t* pt,
                              const uint32_t* orig_id, const OutArrays& out, unsigned long long* skey,
                              cudaStream_t st);
void launch_key32(const unsigned long long* key, uint64_t n, uint32_t* out, cudaStream_t st);
void launch_gather_flagged(const unsigned long long* upair, const uint32_t* uflags, uint64_t n, int k,
                           const uint32_t* pq, const uint32_t* pt, const uint32_t* orig_id, const OutArrays& out,
                           cudaStream_t st);
void launch_solution_flags(const unsigned long long* skey, const uint32_t* skey32, uint64_t n,
                           const unsigned long long* upair, const uint32_t* uflags, uint64_t nf, uint32_t* flags,
                           cudaStream_t st);
void launch_per_query_sorted(const uint32_t* query, const double* contrib, uint64_t n, uint32_t nq, double* per_query,
                             unsigned long long* range, cudaStream_t st);

// visibility.cu
int aabb_levels(uint32_t ntris, uint32_t* n);  // fills n[0..top], returns top
void launch_build_aabbs(const TriRec* recs, AabbTree& T, cudaStream_t st);
void launch_occ_tris(const float* pos, const uint32_t* tri, const uint32_t* order, uint32_t ntris, TriRec* recs,
                     cudaStream_t st);
void launch_visibility(int k, uint64_t n, const SolSink& S, const uint32_t* pq, const uint32_t* pt, const double* ep,
                       const AabbTree& mesh, const AabbTree& occ, uint8_t* keep, int nsm, cudaStream_t st);
void launch_gather_raw(const uint32_t* sel, uint64_t n, int k, const SolSink& in, unsigned long long* okey,
                       double* obary, double* ocontrib, float* oresid, cudaStream_t st);

// fma_peak.cu
void launch_fma_peak(int fp64, int iters, double* sink, int nsm, cudaStream_t st, int* blocks_out, int* threads_out,
                     int* flops_per_thread_iter);

}  // namespace spoly
