// Deterministic compaction: sort the appended solutions by their key
// (pair index << 6 | root slot), gather the records into that order (query / triangle ids from the work
// list), OR-reduce the per-pair flag records, then sum the contributions per query in a fixed order
// ("we sum the contributions from all of them").
#include "kernels.cuh"

namespace spoly {

__global__ void k_iota(uint32_t* v, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st) {
  if (n) k_iota<<<1024, 256, 0, st>>>(v, n);
}

__global__ void k_map_ids(const uint32_t* __restrict__ tpos, uint64_t n, const uint32_t* __restrict__ orig,
                          uint32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = orig[tpos[i]];
}
void launch_map_ids(const uint32_t* tpos, uint64_t n, const uint32_t* orig_id, uint32_t* out, cudaStream_t st) {
  if (n) k_map_ids<<<1024, 256, 0, st>>>(tpos, n, orig_id, out);
}

template <class KeyT>
__global__ void k_gather_solutions(const uint32_t* __restrict__ perm, const KeyT* __restrict__ skey,
                                   uint64_t n, int k, SolSink in, const uint32_t* __restrict__ pq,
                                   const uint32_t* __restrict__ pt, const uint32_t* __restrict__ orig, OutArrays out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = perm[i];
    const uint64_t pair = (uint64_t)skey[i] >> 6;
    out.query[i] = pq[pair];
    for (int j = 0; j < k; ++j) out.tuple[(uint64_t)k * i + j] = orig[pt[(uint64_t)k * pair + j]];
    for (int j = 0; j < 2 * k; ++j) out.bary[(uint64_t)2 * k * i + j] = in.bary[(uint64_t)2 * k * s + j];
    out.contrib[i] = in.contrib[s];
    out.resid[i] = in.resid[s];
  }
}
void launch_gather_solutions(const uint32_t* perm, const unsigned long long* skey, const uint32_t* skey32, uint64_t n,
                             int k, const SolSink& in, const uint32_t* pq, const uint32_t* pt, const uint32_t* orig_id,
                             const OutArrays& out, cudaStream_t st) {
  if (!n) return;
  if (skey32)
    k_gather_solutions<uint32_t><<<2048, 256, 0, st>>>(perm, skey32, n, k, in, pq, pt, orig_id, out);
  else
    k_gather_solutions<unsigned long long><<<2048, 256, 0, st>>>(perm, skey, n, k, in, pq, pt, orig_id, out);
}

// Counting order (replaces the key sort when the per-pair arrays fit): keys are unique and slot < 64, so
// the rank of a solution in key order is (solutions of lower pairs) + (lower slots of its own pair).
// k_slot_masks sets one bit per (pair, slot); the pair counts (popcounts) are exclusive-scanned; the
// scatter writes every record straight to its rank -- the same order as the sort, no sort passes.
__global__ void k_slot_masks(const unsigned long long* __restrict__ key, uint64_t n, unsigned long long* mask) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long kk = key[i];
    atomicOr(mask + (kk >> 6), 1ull << (kk & 63));
  }
}
__global__ void k_mask_counts(const unsigned long long* __restrict__ mask, uint64_t np, uint32_t* __restrict__ cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x)
    cnt[i] = (uint32_t)__popcll(mask[i]);
}
__global__ void k_scatter_solutions(const unsigned long long* __restrict__ key, uint64_t n,
                                    const unsigned long long* __restrict__ mask, const uint32_t* __restrict__ off,
                                    int k, SolSink in, const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                    const uint32_t* __restrict__ orig, OutArrays out, unsigned long long* skey) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long kk = key[i];
    const uint64_t pair = kk >> 6;
    const uint64_t p = (uint64_t)off[pair] + __popcll(mask[pair] & ((1ull << (kk & 63)) - 1ull));
    skey[p] = kk;
    out.query[p] = pq[pair];
    for (int j = 0; j < k; ++j) out.tuple[(uint64_t)k * p + j] = orig[pt[(uint64_t)k * pair + j]];
    for (int j = 0; j < 2 * k; ++j) out.bary[(uint64_t)2 * k * p + j] = in.bary[(uint64_t)2 * k * i + j];
    out.contrib[p] = in.contrib[i];
    out.resid[p] = in.resid[i];
  }
}
void launch_slot_masks(const unsigned long long* key, uint64_t n, unsigned long long* mask, uint64_t npairs,
                       uint32_t* cnt, cudaStream_t st) {
  if (n) k_slot_masks<<<1024, 256, 0, st>>>(key, n, mask);
  if (npairs) k_mask_counts<<<2048, 256, 0, st>>>(mask, npairs, cnt);
}
void launch_scatter_solutions(const unsigned long long* key, uint64_t n, const unsigned long long* mask,
                              const uint32_t* off, int k, const SolSink& in, const uint32_t* pq, const uint32_t* pt,
                              const uint32_t* orig_id, const OutArrays& out, unsigned long long* skey,
                              cudaStream_t st) {
  if (n) k_scatter_solutions<<<2048, 256, 0, st>>>(key, n, mask, off, k, in, pq, pt, orig_id, out, skey);
}

// keys below 2^32 (pair index << 6 | slot): sorted as 32-bit keys (two thirds of the radix-sort traffic)
__global__ void k_key32(const unsigned long long* __restrict__ key, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)key[i];
}
void launch_key32(const unsigned long long* key, uint64_t n, uint32_t* out, cudaStream_t st) {
  if (n) k_key32<<<1024, 256, 0, st>>>(key, n, out);
}

__global__ void k_gather_flagged(const unsigned long long* __restrict__ upair, const uint32_t* __restrict__ uflags,
                                 uint64_t n, int k, const uint32_t* __restrict__ pq, const uint32_t* __restrict__ pt,
                                 const uint32_t* __restrict__ orig, OutArrays out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pair = upair[i];
    out.fquery[i] = pq[pair];
    for (int j = 0; j < k; ++j) out.ftuple[(uint64_t)k * i + j] = orig[pt[(uint64_t)k * pair + j]];
    out.fflags[i] = uflags[i];
  }
}
void launch_gather_flagged(const unsigned long long* upair, const uint32_t* uflags, uint64_t n, int k,
                           const uint32_t* pq, const uint32_t* pt, const uint32_t* orig_id, const OutArrays& out,
                           cudaStream_t st) {
  if (n) k_gather_flagged<<<256, 256, 0, st>>>(upair, uflags, n, k, pq, pt, orig_id, out);
}

// every solution carries its tuple's (OR-reduced) flags: binary search of its pair in the sorted list
template <class KeyT>
__global__ void k_solution_flags(const KeyT* __restrict__ skey, uint64_t n,
                                 const unsigned long long* __restrict__ upair, const uint32_t* __restrict__ uflags,
                                 uint64_t nf, uint32_t* flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long pair = (unsigned long long)skey[i] >> 6;
    uint64_t lo = 0, hi = nf;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (upair[m] < pair) lo = m + 1; else hi = m;
    }
    flags[i] = (lo < nf && upair[lo] == pair) ? uflags[lo] : 0u;
  }
}
void launch_solution_flags(const unsigned long long* skey, const uint32_t* skey32, uint64_t n,
                           const unsigned long long* upair, const uint32_t* uflags, uint64_t nf, uint32_t* flags,
                           cudaStream_t st) {
  if (!n) return;
  if (skey32)
    k_solution_flags<uint32_t><<<2048, 256, 0, st>>>(skey32, n, upair, uflags, nf, flags);
  else
    k_solution_flags<unsigned long long><<<2048, 256, 0, st>>>(skey, n, upair, uflags, nf, flags);
}

// query ranges of the query-sorted solution list in one pass: a run of equal query ids starts / ends where
// the neighbour differs (queries without solutions keep the zeroed empty range [0, 0))
__global__ void k_query_ranges(const uint32_t* __restrict__ query, uint64_t n, unsigned long long* range) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = query[i];
    if (i == 0 || query[i - 1] != q) range[2ull * q] = i;
    if (i + 1 == n || query[i + 1] != q) range[2ull * q + 1] = i + 1;
  }
}
// one warp per query over its range: fixed-order sum (lane-strided partial sums + fixed xor tree) ->
// bit-reproducible per-query totals.
__global__ void k_per_query_sorted(const unsigned long long* __restrict__ range, const double* __restrict__ contrib,
                                   uint32_t nq, double* per_query) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t q = gw; q < nq; q += nw) {
    const uint64_t b = range[2 * q], e = range[2 * q + 1];
    double s = 0.0;
    for (uint64_t i = b + lane; i < e; i += 32) s += contrib[i];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) per_query[q] = s;
  }
}
void launch_per_query_sorted(const uint32_t* query, const double* contrib, uint64_t n, uint32_t nq, double* per_query,
                             unsigned long long* range, cudaStream_t st) {
  if (!nq) return;
  cudaMemsetAsync(range, 0, 2ull * nq * sizeof(unsigned long long), st);
  if (n) k_query_ranges<<<1024, 256, 0, st>>>(query, n, range);
  uint64_t blocks = ((uint64_t)nq * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_per_query_sorted<<<(int)blocks, 256, 0, st>>>(range, contrib, nq, per_query);
}

}  // namespace spoly
