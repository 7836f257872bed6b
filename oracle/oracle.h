/* ORACLE — test infrastructure only.
 *
 * Plain, slow, FP64 CPU transcription of Specular Polynomials (Mo et al. 2024,
 * arXiv 2405.13409; PAPER.md).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code with the
 * CUDA path (paper_2405_13409_b200/csrc) and never calls it.
 *
 * Every step cites the PAPER.md passage it follows; readings of silent/ambiguous passages
 * are the SURVEY.md §8(c) readings, listed in DESIGN.md §3.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tuple flags — excluded from exact-count parity */
#define ORC_FLAG_NEAR_TANGENT 1u
#define ORC_FLAG_BOUNDARY 2u
#define ORC_FLAG_RESIDUAL 4u
#define ORC_FLAG_DEGENERATE 8u

typedef struct {
  int pieces;            /* k>=2 scan pieces, 100 */
  int scan_bisect_iters; /* 10 */
  double bisect_tol;     /* 1e-9 */
  int polish_iters;      /* 5 ("one iteration"; c13, DESIGN reading R23) */
  double theta_admit;    /* 3e-2 raw-root residual gate (k>=2; DESIGN reading R24) */
  double theta_final;    /* 1e-6 final residual gate (north_star) */
  double eps_domain;     /* 1e-9 */
  double eps_flag;       /* 1e-6 */
  double tau_trunc;      /* 1e-12 numerical u-degree truncation (c5-ii) */
  int cull;              /* 1: oracle cull predicate when no tuple list is given */
  double cull_margin;    /* radians, 1e-9 */
  int cull_levels;       /* k=2 barycentric subdivision levels of the cull, 3 */
  int visibility;        /* 1: reject chains with a blocked segment, 0 */
} orc_config;

void orc_default_config(orc_config* cfg);

/* --- whole pipeline ---------------------------------------------------- */
typedef struct orc_result orc_result;

/* mesh: pos/nrm V x 3 float32, tri T x 3 uint32.  endpoints Q x 2 x 3 (x0, x_{k+1}).
 * intensity: Q values or NULL (=1).  offsets/tri_ids: CSR tuple list (k ids per tuple) or
 * NULL -> all tuples (k=1: every triangle; k=2: every ordered pair) filtered by the oracle
 * cull if cfg->cull.  nthreads<=0 -> hardware concurrency.  Returns NULL on bad input. */
orc_result* orc_solve(const float* pos, const float* nrm, uint32_t nverts, const uint32_t* tri,
                      uint32_t ntris, float eta_front, float eta_back, const char* chain,
                      const double* endpoints, uint32_t nq, const double* intensity,
                      const uint32_t* offsets, const uint32_t* tri_ids, const orc_config* cfg,
                      int nthreads, const float* occ_pos, uint32_t occ_nverts, const uint32_t* occ_tri,
                      uint32_t occ_ntris /* optional non-specular occluders for the visibility test (may be 0) */);
void orc_free(orc_result*);
/* sizes */
uint64_t orc_n_solutions(const orc_result*);
uint64_t orc_n_flagged(const orc_result*);
int orc_k(const orc_result*);
/* copies out: query[n], tuple[n*k], bary[n*2k], contribution[n], residual[n], flags[n] */
void orc_get_solutions(const orc_result*, uint32_t* query, uint32_t* tuple, double* bary,
                       double* contribution, double* residual, uint32_t* flags);
/* flagged tuples: query[m], tuple[m*k], flags[m] */
void orc_get_flagged(const orc_result*, uint32_t* query, uint32_t* tuple, uint32_t* flags);
void orc_get_per_query(const orc_result*, double* per_query /* Q */);
/* the (query, tuple) pairs the oracle solved (after its cull): query[n], tuple[n*k] */
uint64_t orc_n_worklist(const orc_result*);
void orc_get_worklist(const orc_result*, uint32_t* query, uint32_t* tuple);
/* counters: pairs_in, systems, vroots, candidates, rej_domain, rej_constraint, rej_side,
 *           rej_kappa, flagged, admissible, rej_visibility */
void orc_get_report(const orc_result*, uint64_t counters[11]);

/* --- pieces, exported for the pins in tests/ ---------------------------- */
/* Build the bivariate system (a,b) for one tuple (Sec. 4.5, Eqs. 21-23).
 * tris: k triangles x (p0,p1,p2,n0,n1,n2) x 3 doubles (18 per triangle), ORIGINAL labeling.
 * Outputs dense (deg+1)^2 grids (index i*(deg+1)+j = coefficient of u^i v^j) BEFORE
 * normalisation/truncation, plus the decisions taken.  a_out/b_out capacity: 64*64.
 * info[0]=relabel(0/1) info[1]=eta0*1000 info[2]=degenerate-basis(0/1) */
int orc_build_system(const char* chain, const double* tris, const double* x0, const double* xk1,
                     double eta_front, double eta_back, const double* sqrt_table,
                     double* a_out, int* deg_a, double* b_out, int* deg_b, int* info);
/* Bezout matrix (Eq. 24) of two bivariate grids, hiding v: returns n and, for entry (i,j),
 * coefficients in ent[(i*n+j)*maxc + l] (maxc = 2*64). */
int orc_bezout(const double* a, int deg_a, const double* b, int deg_b, int n, double* ent, int* ent_deg);
/* determinant polynomial of an n x n matrix of univariate polynomials by Laplace expansion */
int orc_det_laplace(const double* ent, const int* ent_deg, int n, double* r_out);
/* determinant of the numeric Bezout matrix at v by Gaussian elimination (partial pivoting) */
double orc_det_at(const double* a, int deg_a, const double* b, int deg_b, int n, double v);
/* derivative-recursion isolation + bisection */
int orc_isolate(const double* p, int deg, double lo, double hi, double tol, double* roots_out);
/* cull predicate: 1 = keep.  tris as in orc_build_system. */
int orc_cull_keep(const char* chain, const double* tris, const double* x0, const double* xk1,
                  double eta_front, double eta_back, double margin, int levels /* k=2 subdivision */);
/* exact forward light-side trace Jacobian J (c15) at a solved chain; returns J (<=0 on failure) */
double orc_jacobian(const char* chain, const double* tris, const double* x0, const double* xk1,
                    double eta_front, double eta_back, const double* bary);
/* piecewise rational sqrt surrogate (Eq. 20) table used by the oracle: 6 x (lo, hi, c0, c1, d1) */
void orc_sqrt_table(double* out30);
double orc_sqrt_approx(double x);

#ifdef __cplusplus
}
#endif
