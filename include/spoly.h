/* spoly.h — C ABI of the B200-native Specular Polynomials hot path (libspoly.so).
 *
 * Problem (Sec. 3.1): given two separators x_0, x_{k+1} (a "query") and a tuple
 * of k specular triangles T_1..T_k (positions P_i, shading normals N_i, Eqs. 1-2),
 * return ALL admissible specular chains x_1..x_k satisfying h_i x n_i = 0 (Eq. 3), and, when
 * several connect the same separators, the sum of their contributions.
 *
 * Method on the device (all sm_100a kernels, FP64 where the tolerance needs it):
 *   cull (replaces the Wang20 pruning PAPER.md:680)  ->  coefficient phase (Eqs. 6, 9, 12, 13-20;
 *   Sec. 5.3)  ->  elimination phase (hidden-variable Bezout resultant, Eq. 24)  ->  univariate
 *   roots (Laplace expansion + derivative-recursion root isolation for k=1, PAPER.md:604-608;
 *   determinant-sign bisection over 100 pieces for k=2)  ->  path phase
 *   (back-substitution, validation, contribution)  ->  deterministic compaction.
 *
 * Conventions
 *  - Every call returns spoly_status; no exception crosses the ABI.  Errors are sticky only for the
 *    call that reports them.
 *  - Pointers documented "device" are CUDA device pointers valid on the ctx's device (e.g. a torch
 *    CUDA tensor's data_ptr()); pointers documented "host" are ordinary host memory.
 *  - The ctx owns every output buffer; they stay valid until the next spoly_solve* on the same ctx
 *    or spoly_destroy.
 *  - All work is enqueued on the ctx's stream; spoly_solve returns after the stream has completed
 *    (it synchronises once to read the solution count), so outputs are ready on return.
 *  - Per-tuple degeneracies (near-tangent roots, boundary roots, degenerate systems) are FLAGS on
 *    the tuple, never errors.
 */
#ifndef SPOLY_H
#define SPOLY_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPOLY_OK = 0,
  SPOLY_ERR_INVALID_ARG = 1,       /* NULL pointer, bounces != strlen(chain), bad sizes        */
  SPOLY_ERR_BAD_MESH = 2,          /* index out of range or degenerate triangle (|e1xe2| tiny) */
  SPOLY_ERR_UNSUPPORTED_CHAIN = 3, /* chain not in {"R","T","RR","TT","RT","TR"}              */
  SPOLY_ERR_OOM = 4,               /* device allocation failed                                 */
  SPOLY_ERR_CAPACITY = 5,          /* max_solutions too small even after one regrow            */
  SPOLY_ERR_CUDA = 6               /* any other CUDA runtime error (message: spoly_last_error) */
} spoly_status;

/* tuple flags: excluded from exact-count parity, reported per tuple */
#define SPOLY_FLAG_NEAR_TANGENT 1u /* root pair closer than eps_flag, tiny critical value, or
                                      non-transversal (a,b) intersection                        */
#define SPOLY_FLAG_BOUNDARY 2u     /* a valid chain within eps_flag of a triangle edge           */
#define SPOLY_FLAG_RESIDUAL 4u     /* accepted chain with residual in [1e-7, theta_final)        */
#define SPOLY_FLAG_DEGENERATE 8u   /* a or b identically zero, u-free system, degenerate basis   */
#define SPOLY_FLAG_TRUNCATED 16u   /* a fixed per-tuple capacity of the kernels was exceeded (more v-roots,
                                      u-roots or admissible chains than the kernel keeps): the tuple's
                                      solution set may be incomplete; counted in report.n_truncated  */

typedef struct spoly_ctx spoly_ctx;

typedef struct {
  int pieces;            /* k>=2 determinant scan pieces; 100                 */
  int scan_bisect_iters; /* k>=2 bisections per sign-changing piece; 10       */
  double bisect_tol;     /* k=1 root bracket threshold; 1e-9                  */
  int polish_iters;      /* Newton steps on the exact shooting residual (k=2); 5 (reading R23) */
  double theta_admit;    /* raw-root residual gate before polish (k=2); 3e-2 (reading R24)   */
  double theta_final;    /* final Eq. 3 residual gate; 1e-6 (north_star)                     */
  double eps_domain;     /* barycentric slack of the inside test; 1e-9                       */
  double eps_flag;       /* near-tangent / boundary flag distance; 1e-6                      */
  double tau_trunc;      /* numerical u-degree truncation threshold; 1e-12       */
  int cull;              /* 1: run the cull pre-pass when no tuple list is given             */
  int deterministic;     /* ignored: the output is always in the deterministic (query, tuple,
                            root) order and bit-identical run to run (kept for ABI stability) */
  float cull_margin;     /* angular slack (rad) of the FP32 cull; 1e-4                       */
  uint64_t max_solutions;/* minimum initial solution-buffer capacity; the library also sizes the
                            solution / flag sinks from the work list (k=1: pairs/2, pairs/64;
                            k=2: pairs/32, pairs/8) and regrows them once on overflow       */
  uint64_t max_pairs;    /* k=2 cull: max node-pair frontier entries per query chunk; 2^27.
                            Queries are culled in chunks that fit (order-preserving, so the
                            work list is the unchunked one); SPOLY_ERR_CAPACITY if one query
                            alone exceeds it                                                */
  int cull_levels;       /* k=2: barycentric subdivision levels re-testing each kept pair; 3 */
  int visibility;        /* 1: the path phase's visibility test: a chain with a blocked segment
                            x_i -> x_{i+1} is dropped (scene = the specular mesh + the occluders of
                            spoly_upload_occluders; the chain's own triangles at a segment's ends are skipped;
                            a hit is t in (1e-7, 1 - 1e-7) inside the closed triangle); 0 (default)          */
  int scan_restrict;     /* k=2 with the cull: the 100-piece determinant scan skips the pieces outside
                            the v-range of T_1's surviving subdivision cells (+1 piece each side): the cull
                            predicate is sound, so no admissible chain lies there (reading R25); 1 (default)    */
  int k2_tiles;          /* k=2 cull: expand the node-pair hierarchy once per tile of 32 Morton-sorted queries
                            (endpoint spheres), then test each query exactly on its tile's triangle pairs; the
                            work list is query-major in that order; 1 (default), 0: per-query expansion     */
} spoly_config;

/* Fills cfg with the defaults listed above.  Never fails for a non-NULL cfg. */
spoly_status spoly_default_config(spoly_config* cfg);

/* Creates a context on CUDA device `cuda_device`.  cfg NULL -> defaults.  cuda_stream: a
 * cudaStream_t to enqueue on (NULL -> the ctx creates and owns a non-blocking stream).
 * On success *out owns device memory until spoly_destroy. */
spoly_status spoly_create(int cuda_device, const spoly_config* cfg, void* cuda_stream, spoly_ctx** out);
void spoly_destroy(spoly_ctx* ctx);
/* Human-readable message of the last failing call on this ctx (static storage of the ctx). */
const char* spoly_last_error(const spoly_ctx* ctx);

/* Uploads a triangle mesh (HOST pointers, copied): pos/nrm are nverts x 3 float32 (positions and
 * per-vertex shading normals; normals need not be unit, Eq. 2 interpolates them un-normalised),
 * tri is ntris x 3 uint32 vertex indices; the winding defines the geometric normal e1 x e2 whose
 * side has index of refraction eta_front (the other side eta_back).  Builds the per-triangle FP32
 * records, the spatial (Morton) cluster hierarchy and the cluster bounds used by the cull.
 * Replaces any previously uploaded mesh; *mesh_id receives its id (always 0 in this version). */
spoly_status spoly_upload_mesh(spoly_ctx* ctx, const float* pos, const float* nrm, uint32_t nverts,
                               const uint32_t* tri, uint32_t ntris, float eta_front, float eta_back,
                               uint32_t* mesh_id);

/* Uploads (HOST pointers, copied) an occluder-only mesh for the visibility test (cfg.visibility): triangles that
 * block segments but are never specular (no normals).  pos: nverts x 3 float32, tri: ntris x 3 uint32.  ntris = 0
 * removes the occluders.  The specular mesh always occludes as well. */
spoly_status spoly_upload_occluders(spoly_ctx* ctx, const float* pos, uint32_t nverts, const uint32_t* tri,
                                    uint32_t ntris);

/* Optional explicit tuple list (device pointers): CSR offsets[nqueries+1] into tri_ids, which holds
 * k uint32 triangle ids per tuple (ORIGINAL mesh indices). */
typedef struct {
  const uint32_t* offsets;
  const uint32_t* tri_ids;
} spoly_tuple_list;

typedef struct {
  /* telescoping counters */
  uint64_t n_pairs_in, n_systems, n_vroots, n_candidates, n_rej_domain, n_rej_constraint, n_rej_side,
      n_rej_kappa, n_flagged, n_admissible;
  float ms_cull, ms_solve, ms_reduce; /* CUDA-event times of the phases of the last solve       */
  uint32_t n_launches;                /* kernels this library launched in the last solve        */
  uint64_t n_eval_terms;              /* FMA terms of the univariate root-finding evaluations of the
                                         monotone jobs in phase 1 (FLOP model)      */
  uint64_t required_solutions;        /* set with SPOLY_ERR_CAPACITY                            */
  float ms_phase1, ms_phase2;         /* CUDA-event times of the two solve kernels (phase 2 incl.
                                         the count read-back)                                    */
  uint64_t n_rebuilds;                /* phase-2 coefficient-phase recomputations (FLOP model)   */
  uint64_t alg_kflop;                 /* two-bounce kernel: algorithmic kFLOP (coefficient phase +
                                         determinant evaluations)                   */
  uint64_t n_jobs_mono, n_jobs_deep;  /* one-bounce jobs: monotone r with a root in [0,1] (solved in
                                         phase 1) / deeper derivative recursion (deep-job kernel)  */
  uint64_t n_elims;                   /* one-bounce pairs that reached the elimination phase       */
  uint64_t n_pairs_coarse;            /* pairs kept before the last exact filter: two-bounce pair cull
                                         before the subdivision refinement; one-bounce R before the
                                         product-form sign test (n_pairs_in counts the final list)   */
  float ms_roots, ms_path;            /* one-bounce phase 2 split: deep-job root isolation and the
                                         path kernel (incl. the count read-back)                    */
  uint64_t n_refined;                 /* one-bounce candidates past the domain pre-check (refined,
                                         reading R2; FLOP model)                                     */
  uint64_t n_cand_jobs, n_path_jobs;  /* one-bounce monotone jobs with a root (back-substitution
                                         pre-check in phase 1) / jobs the path kernel ran           */
  uint64_t n_cull_tests;              /* cull work of the last solve: one bounce, triangle tests of the
                                         per-query cull; two bounces, node-pair tests of the pair
                                         expansion + sub-pair tests of the subdivision refinement    */
  uint64_t n_truncated;               /* roots / chains dropped at a per-tuple kernel capacity (each such
                                         tuple carries SPOLY_FLAG_TRUNCATED)                          */
  uint64_t n_big_scan;                /* two bounces: tuples whose Bezout order n > 32 took the
                                         shared-memory determinant                                    */
  uint64_t n_eval_deep;               /* one bounce: FMA terms of the deep jobs' root isolation (the
                                         monotone jobs' Newton terms are in n_eval_terms)              */
  uint64_t n_rej_visibility;          /* admissible chains dropped by the visibility test             */
} spoly_report;

typedef struct {
  uint64_t n_solutions; /* admissible chains                                                */
  uint64_t n_flagged;   /* tuples carrying a flag                                           */
  int k;                /* bounces                                                          */
  /* device pointers owned by the ctx, sorted by (query, tuple position, root) when
   * deterministic=1.  The order comes from a radix sort of the (pair << 6 | slot) keys or, when the
   * work list is small relative to the solution count, from an equivalent counting order (identical
   * output); the environment variable SPOLY_SORT_ORDER=1 / =0 forces the sort / the counting order. */
  const uint32_t* query;        /* [n_solutions]                                            */
  const uint32_t* tuple;        /* [n_solutions * k] original triangle ids                  */
  const double* bary;           /* [n_solutions * 2k] (u_1, v_1[, u_2, v_2]), Eq. 1          */
  const double* contribution;   /* [n_solutions] I / J (geometric point-light factor, c15)  */
  const float* residual;        /* [n_solutions] max_i |h_i^ x n_i^| (Eq. 3)                */
  const uint32_t* flags;        /* [n_solutions] flags of the solution's tuple              */
  const uint32_t* flagged_query;/* [n_flagged]                                              */
  const uint32_t* flagged_tuple;/* [n_flagged * k]                                          */
  const uint32_t* flagged_flags;/* [n_flagged]                                              */
  const double* per_query;      /* [nqueries] sum of contributions           */
  spoly_report report;
} spoly_result;

/* Solves every (query, tuple) pair.  chain: "R", "T", "RR" or "TT" (Heckbert notation,
 * PAPER.md:479); bounces must equal strlen(chain).  endpoints: DEVICE, nqueries x 2 x 3 float64
 * (x_0 then x_{k+1}).  light_intensity: DEVICE, nqueries float64, or NULL (= 1).  tuples: DEVICE
 * CSR list, or NULL -> the cull pre-pass enumerates candidate tuples itself (cfg.cull=1) or all
 * tuples (cfg.cull=0).  out: filled with ctx-owned device pointers. */
spoly_status spoly_solve(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces,
                         const double* endpoints, uint32_t nqueries, const double* light_intensity,
                         const spoly_tuple_list* tuples, spoly_result* out);

/* Same as spoly_solve but from/to HOST memory: copies endpoints/intensity host->device (through
 * ctx-owned pinned staging), solves, and copies the per-query contribution sums (nqueries float64)
 * back into per_query_host.  out (optional) receives the device-side result as spoly_solve. */
spoly_status spoly_solve_host(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces,
                              const double* endpoints_host, uint32_t nqueries,
                              const double* light_intensity_host, double* per_query_host,
                              spoly_result* out);

/* Glossy (near-specular) vertices, PAPER.md:857-859 ("After sampling the normal offset for glossy vertices, the
 * admissible chains corresponding to the offset remain finite, and the problem reduces to pure specular
 * situations"), reading R28.  slopes: HOST, ntris x 2 float64 (p, q) in ORIGINAL triangle order,
 * microfacet slopes sampled by the caller (e.g. Beckmann: p, q ~ N(0, alpha^2 / 2)).  Every triangle's three
 * shading normals become n_j' = fl32(n_j + p T + q B), (T, B) the orthonormal frame of the triangle plane
 * (T = e1 / |e1|, B = g^ x T, g = e1 x e2), computed in FP64 on the device from the UPLOADED normals (offsets do
 * not accumulate); the cull bounds are rebuilt.  Later solves see the perturbed surface.  slopes = NULL restores
 * the uploaded normals.  Errors: INVALID_ARG (no mesh, ntris != mesh triangle count, non-finite slope). */
spoly_status spoly_set_normal_offsets(spoly_ctx* ctx, const double* slopes, uint32_t ntris);

/* Deterministic splat renderer (the application layer of PAPER.md:680 "apply it on both glints rendering and
 * caustics rendering"; SPEC S:661-669 cmd_render without Monte Carlo): the width x height queries (row-major
 * pixels; endpoints DEVICE nqueries x 2 x 3 float64 as spoly_solve: x_0 = the pixel's diffuse receiver point,
 * x_{k+1} = the light) are solved once per sample s < nsamples with the sample's normal offsets (slopes: HOST,
 * nsamples x ntris x 2 float64 as spoly_set_normal_offsets, or NULL = pure specular, one solve), and
 *     radiance[q] = sum_s (albedo / pi / nsamples) * per_query_s[q]      (accumulated in sample order)
 * radiance: DEVICE, nqueries float64 (linear).  srgb: DEVICE, nqueries x 3 uint8 or NULL:
 *     c = rint(255 * min(1, max(0, exposure * radiance))^(1 / 2.2)) in every channel (gray).
 * light_intensity as spoly_solve.  The uploaded normals are restored on return.  Errors: as spoly_solve,
 * INVALID_ARG for a zero or > 2^32 image, negative albedo or exposure. */
spoly_status spoly_render(spoly_ctx* ctx, uint32_t mesh_id, const char* chain, int bounces, const double* endpoints,
                          uint32_t width, uint32_t height, const double* light_intensity, uint32_t nsamples,
                          const double* slopes, double albedo, double exposure, double* radiance, uint8_t* srgb);

/* Device pointers of the (query, tuple) work list of the LAST solve (cull output or the given list),
 * query-major: pair_query[n_pairs], pair_tuple[n_pairs * k] (original ids).  A chunked two-bounce cull
 * keeps every chunk's pairs, concatenated in chunk order (*n_pairs counts them all). */
spoly_status spoly_last_worklist(const spoly_ctx* ctx, const uint32_t** pair_query,
                                 const uint32_t** pair_tuple, uint64_t* n_pairs);

/* The piecewise rational sqrt surrogate of Eq. 20 the two-bounce kernels use for a
 * refracting first vertex: 6 rows of (lo, hi, c0, c1, d1), sqrt(x) ~ (c0 + c1 x) / (1 + d1 x) on [lo, hi]
 * (our minimax fit, reading R8).  out30: HOST, 30 doubles.  from_device = 0: the host copy
 * compiled into the library (ctx may be NULL, no GPU needed); 1: the table read back from the device's
 * constant memory (needs a ctx).  Lets the tests pin the kernels' copy to tests/golden/sqrt_table.txt. */
spoly_status spoly_sqrt_table(spoly_ctx* ctx, int from_device, double* out30);

/* FMA-throughput microbenchmark on the ctx's device (roofline denominator): independent FMA
 * chains on every SM for about `seconds`.  fp64=1: double, 0: float.  Returns FLOP/s. */
spoly_status spoly_bench_fma(spoly_ctx* ctx, int fp64, double seconds, double* flops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* SPOLY_H */
