// Host-visible launchers of the CUDA kernels (implemented in the .cu files of csrc/).
#pragma once
#include "common.cuh"

namespace spoly {

// mesh.cu
void launch_build_tris(const float* pos, const float* nrm, const uint32_t* tri, const uint32_t* order, uint32_t ntris,
                       TriRec* recs, float4* tricone, uint32_t* orig_id, uint32_t* perm_of, cudaStream_t st);
void launch_build_clusters(const TriRec* recs, const float4* tricone, uint32_t ntris, ClusterRec* cl, cudaStream_t st);

// cull.cu: pass 0 counts survivors per query, pass 1 writes the query-major work list
struct CullParams {
  float margin;
  int refract;  // 0: R, 1: T
  float eta_front, eta_back;
};
void launch_cull_k1(int pass, const double* ep, uint32_t nq, const DeviceMesh& M, const CullParams& cp,
                    uint32_t* counts, const unsigned long long* offsets, uint32_t* pair_query, uint32_t* pair_tpos,
                    int nsm, cudaStream_t st);
void launch_all_pairs_k1(uint32_t nq, uint32_t ntris, uint32_t* pair_query, uint32_t* pair_tpos, cudaStream_t st);
void launch_expand_list(const uint32_t* offsets, const uint32_t* tri_ids, uint32_t nq, int k, const uint32_t* perm_of,
                        uint32_t* pair_query, uint32_t* pair_tpos, int nsm, cudaStream_t st);

// solve_k1.cu
void launch_solve_R_list(const uint32_t* pq, const uint32_t* pt, uint64_t npairs, uint64_t pair_base,
                         const DeviceMesh& M, const double* ep, const double* inten, const SolveParams& prm,
                         const SolSink& S, int nsm, cudaStream_t st);

// reduce.cu
void launch_map_ids(const uint32_t* tpos, uint64_t n, const uint32_t* orig_id, uint32_t* out, cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st);
void launch_gather_solutions(const uint32_t* perm, uint64_t n, int k, const SolSink& in, const SolSink& out,
                             cudaStream_t st);
void launch_gather_flagged(const uint32_t* perm, uint64_t n, int k, const SolSink& in, const SolSink& out,
                           cudaStream_t st);
void launch_per_query_sorted(const uint32_t* query, const double* contrib, uint64_t n, uint32_t nq, double* per_query,
                             cudaStream_t st);

// fma_peak.cu
void launch_fma_peak(int fp64, int iters, double* sink, int nsm, cudaStream_t st, int* blocks_out, int* threads_out,
                     int* flops_per_thread_iter);

}  // namespace spoly
