/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 path.
 *
 * Plain-C restatement of the reference hot path (blockfv, /root/reference/proj/core):
 * LDU->BSR plan and permutation, BSR SpMV, block LU, LUSGS, DILU, pairwise
 * aggregation, Galerkin coarsening, AMG V-cycle with dense coarsest LU,
 * restarted right-preconditioned GMRES (MGS) and BiCGStab, the topology
 * signature, and the RCB decomposition / partition / consolidation layer.
 * Each function cites the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker.  The product (libbcs.so) never links
 * or calls it.  It is pinned bit-for-bit against the reference itself
 * (oracle/_ref/libbcs_ref.so) and against tests/golden/* by
 * tests/test_oracle.py.
 */
#ifndef BCS_ORACLE_H
#define BCS_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Same leading fields/order as bcs_solver_config (include/bcs.h). */
typedef struct {
    int method;   /* 0 GMRES, 1 BiCGStab */
    int precond;  /* 0 none, 1 LUSGS, 2 DILU, 3 AMG */
    double rel_tol;
    double abs_tol;
    int max_iters;
    int gmres_restart;
    int amg_max_levels;
    int amg_min_coarse_rows;
    int amg_pre_sweeps;
    int amg_post_sweeps;
} or_cfg;

typedef struct {
    int iterations;
    int converged;
    int breakdown;
    int amg_levels;
    double initial_residual;
    double final_residual;
} or_report;

const char* or_last_error(void);
/* 0: reference sequential dot (default); 1: pairwise re-association */
void or_set_dot_mode(int mode);

/* block_csr.cpp:56-80 — src[k] encodes the LDU source of slot k:
 * c (diag of cell c), nc+f (upper of face f), nc+nf+f (lower of face f). */
int or_csr_plan(int nc, int nf, const int* owner, const int* neigh, int* row_off, int* cols, int* src);
/* block_csr.cpp:97-109 value permutation */
void or_csr_values(int nc, int nf, int n, const int* src, const double* diag, const double* upper,
                   const double* lower, double* vals);
/* block_csr.cpp:146-160 */
unsigned long long or_signature(int nc, int nf, const int* owner, const int* neigh);
/* block_csr.cpp:129-137 */
void or_csr_matvec(int rows, int n, const int* row_off, const int* cols, const double* vals, const double* x,
                   double* y);
/* block_matrix.cpp:104-119 (LDU addressing) */
void or_ldu_matvec(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                   const double* upper, const double* lower, const double* x, double* y);
/* amg.cpp:10-37; returns nCoarse */
int or_aggregate(int rows, int n, const int* row_off, const int* cols, const double* vals, int* agg);

/* one z = M^{-1} r with the configured preconditioner (engine.cpp:21-29) */
int or_precond_apply(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                     const double* upper, const double* lower, const or_cfg* cfg, const double* r, double* z);

/* SolvePipeline::solve EngineCsr (engine.cpp:47-120) + residual history.
 * hist[k] = relative residual after Arnoldi step / BiCGStab iteration k
 * (implicit |g_{j+1}|/beta0, replaced by the true residual at each restart/exit). */
int or_solve(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag, const double* upper,
             const double* lower, const double* b, const double* x0, const or_cfg* cfg, double* x, or_report* rep,
             double* hist, int hist_cap, int* hist_n);

/* AMG hierarchy (amg.cpp:73-105) handle */
void* or_amg_build(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                   const double* upper, const double* lower, int max_levels, int min_coarse_rows);
int or_amg_depth(void* h);
void or_amg_level_sizes(void* h, int l, int* rows, int* nnz, int* agg_len);
void or_amg_level_get(void* h, int l, int* row_off, int* cols, double* vals, int* agg);
void or_amg_free(void* h);

/* partition.cpp:21-85 */
int or_decompose(int nc, const double* centroids, int n_ranks, int* cell_to_rank, int* rank_row_offset,
                 int* old_to_new);

#ifdef __cplusplus
}
#endif
#endif
