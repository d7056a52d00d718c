// Host-side launch wrappers for the sm_100a kernels (one translation unit
// per subsystem: k_csr.cu, k_sweep.cu, k_amg.cu, k_krylov.cu).  Every wrapper
// enqueues on the given stream and increments the launch counter.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>

namespace bcs {

// guards the lazily initialised per-process launch parameters (occupancy
// capacities, function attributes): contexts on different host threads may
// make their first launches at the same time
std::recursive_mutex& lazy_init_mutex();


struct LaunchCounter {
    long long launches = 0;
};
extern thread_local LaunchCounter* g_launches;
inline void count_launch(int k = 1) {
    if (g_launches) g_launches->launches += k;
}

int num_sms();

// ---------------------------------------------------------------- scan
// exclusive prefix sum of n ints in place; *total (device) = sum. tmp >= scan_tmp_ints(n)
size_t scan_tmp_ints(size_t n);
void exclusive_scan(int* data, int n, int* d_total, int* tmp, cudaStream_t s);

// ---------------------------------------------------- LDU -> BSR (K1, K2)
// rowcnt must be zeroed, size nc+1
void plan_count(int nc, int nf, const int* owner, const int* neigh, int* rowcnt, cudaStream_t s);
// fill: ro (nc+1) already scanned; fill counters zeroed (nc)
void plan_fill(int nc, int nf, const int* owner, const int* neigh, const int* ro, int* fillc, int* ci, int* src,
               cudaStream_t s);
void plan_sort_rows(int nc, const int* ro, int* ci, int* src, cudaStream_t s);
void find_diag(int rows, const int* ro, const int* ci, int* dg, cudaStream_t s);
void transpose_pos(int rows, const int* ro, const int* ci, int* tpos, int* asym_flag, cudaStream_t s);
void gather_values(int n, int nnz, int nc, int nf, const int* src, const double* diag, const double* upper,
                   const double* lower, double* vals, cudaStream_t s);

// -------------------------------- performance mode: multicolouring (k_color.cu)
// Jones-Plassmann colouring (deterministic); colA receives the colours.
// Returns the number of rounds, -1 when a row would need more than 64 colours.
int mc_color(int rows, const int* ro, const int* ci, int* colA, int* colB, int* counters, int* hostCounters,
             cudaStream_t s);
// perm[new] = old, inv[old] = new, rows ordered by (colour, index); returns #colours (syncs)
int mc_permutation(int rows, const int* color, int* perm, int* inv, int* scratch, size_t scratchInts, int* hostBuf,
                   cudaStream_t s);
// permuted BSR pattern (nro: rows+1, nci/sv: nnz; sv = source slot of each new slot)
void mc_permute_pattern(int rows, const int* ro, const int* ci, const int* perm, const int* inv, int* nro, int* nci,
                        int* sv, int* scanTmp, int* dTotal, cudaStream_t s);
void mc_permute_values(int n, size_t nnz, const int* sv, const double* v, double* nv, cudaStream_t s);
void mc_vec_gather(int n, int rows, const int* perm, const double* x, double* xp, cudaStream_t s);
void mc_vec_scatter(int n, int rows, const int* perm, const double* sp, double* z, int acc, cudaStream_t s);
// performance mode, block-Jacobi smoothing: z (=|+=) omega * D^-1 r per block row
void block_jacobi(int n, int rows, const double* lu, const double* rcp, const int* perm, const double* r, double* z,
                  int acc, double omega, cudaStream_t s);
// colour-synchronous DILU sweep of a coloured level (coff: device, ncol + 1 colour boundaries)
// performance mode: one colour [i0, i1) of the colour-permuted level as a
// streaming pass (rows of a colour are independent); forward colours in
// increasing order, backward in decreasing order, one launch each
// rowmap != null: the forward reads rin in the original numbering (fused
// gather); the backward also writes zfinal[rowmap[i]] with k_vec_scatter's
// acc semantics (fused scatter)
void mc_colour_sweep(int n, bool fwd, int i0, int i1, const int* ro, const int* dg, const int* ci, const double* v,
                     const double* lu, const double* rcp, const int* perm, const double* rin, double* out,
                     const int* rowmap, double* zfinal, int acc, cudaStream_t s);
void mc_sweep(int n, bool fwd, int rows, int ncol, const int* coff, const int* ro, const int* dg, const int* ci,
              const double* v, const double* lu, const double* rcp, const int* perm, const double* rin, double* out,
              cudaStream_t s);

// ------------------------------------------------------------- SpMV (K3)
// y = A x  (sub == nullptr)   or   y = sub - A x
void spmv(int n, int rows, const int* ro, const int* ci, const double* v, const double* x, const double* sub,
          double* y, cudaStream_t s);

// ------------------------------------------------- LU / sweeps (K5-K8)
void factor_diag_blocks(int n, int rows, const int* dg, const double* v, double* lu, int* piv, int* err_cell,
                        cudaStream_t s);
// Level-synchronous Kahn over the lower-triangular DAG.  dilu != 0 also
// computes the DILU modified diagonals (preconditioner.cpp:101-126) into lu/piv.
// order (rows) receives the level-sorted row permutation; returns depth.
struct KahnWork {
    int* cnt;    // rows
    int* tail;   // >= 5 ints of counters
    int* lvl;    // rows+1 (level offsets into order / active list A)
    int* lvl2;   // rows (active list B, aggregation only)
};
extern int last_agg_rounds;  // rounds of the last aggregation (diagnostics)
// T: scratch of nnz*n*n doubles (producer-side D~_j^{-1} A_ji blocks), DILU only
int kahn_schedule(int n, int rows, const int* ro, const int* ci, const int* dg, const int* tpos, const double* v,
                  bool dilu, double* lu, int* piv, double* T, int* order, KahnWork w, int* err_cell,
                  cudaStream_t s);
// sync-free level schedule (rows bucketed by dependency level); returns depth.
// level: rows ints, cnt: rows+2 ints, small: >= 3 ints
int level_schedule(int rows, const int* ro, const int* ci, const int* dg, int* order, int* level, int* cnt,
                   int* scan_tmp, int* small, int* err, cudaStream_t s);
// DILU setup (preconditioner.cpp:101-126) of several matrices at once (the
// AMG levels but the coarsest), sync-free: tickets ordered by (dependency
// level, matrix).  dlev: the matrix's dependency levels (level_schedule);
// T: scratch of sum(nnz)*n*n doubles, matrix l at Tbase + tOff; keys/order:
// sum(rows) ints; cnt: maxdepth*nl+1 ints; desc_dev: dilu_desc_bytes().
// *err_cell = min over singular rows of (matrix << 26 | row).
struct DiluLevelHost {
    int rows;
    const int *ro, *dg, *tpos, *tc, *lpre, *dlev;
    const double* v;
    double* lu;
    int* piv;
    size_t tOff;
};
void dilu_setup_multi(int n, int nl, const DiluLevelHost* levels, int maxdepth, int* keys, int* order, int* cnt,
                      int* scan_tmp, int* small, void* desc_dev, double* Tbase, size_t tcount, int* err_cell,
                      int* err, cudaStream_t s);
size_t dilu_desc_bytes();
// lower-slot prefix lpre[rows+1] and compact transposed index tc[nnz] of the
// DILU setup's T (lower slots only); returns the number of lower slots (syncs)
size_t dilu_compact_index(int rows, const int* ro, const int* dg, const int* ci, const int* tpos, int* lpre, int* tc,
                          int* d_total, int* scan_tmp, cudaStream_t s);
// dependency levels + level-ordered schedules of several matrices in one
// sync-free pass; depth[l] out; small >= 2 + nl ints; cnt >= max depth + 2.
struct LevelsHost {
    int rows;
    const int *ro, *ci, *dg;
    int* level;
    int* order;
};
void level_schedule_multi(int nl, const LevelsHost* lv, int* depth, int* cnt, int* scan_tmp, int* small,
                          void* desc_dev, int* err, cudaStream_t s);
// sync-free sweeps (preconditioner.cpp:128-156 / :29-57). y, zb pre-filled
// with the pending pattern (0xFF bytes).  accumulate: 0 none, 1 z = 0 + zb,
// 2 z += zb.  rcp: per-row diagonal reciprocals (make_reciprocals).
void make_reciprocals(int n, int rows, const double* lu, const int* piv, double* rcp, int* perm, cudaStream_t s);
// ticket-order records (int4: row, first slot, #deps) for both sweeps
// order: forward tickets -> rows; border: backward tickets -> rows, or
// nullptr for the forward order reversed (the level schedule)
void sweep_records(int rows, const int* order, const int* border, const int* ro, const int* dg, int* fwd4,
                   int* bwd4, cudaStream_t s);
// chain schedule (k_sweep.cu): W = warps of the chain kernel's cooperative
// grid; order (rows) = tickets -> rows, woff (W+1) = warp ticket ranges;
// *bad |= 1 when the schedule's progress check fails on this pattern.
// Launch the level's sweeps with depth = -1 and woff.
int sweep_chunk_warps(int n, bool fwd);
// cluster variant spread over G > 1 clusters: the level's rows must be
// ticketed range-major (rows/G contiguous row ranges, each in level order):
// out = order stably sorted by range.  G = 0: not the cluster variant.
int sweep_cluster_parts(int n, int rows, int depth);
void cluster_part_order(int rows, int G, const int* order, int* out, cudaStream_t s);
void chain_schedule(int rows, bool fwd, int depth, const int* ro, const int* dg, const int* ci, const int* dlev, int W,
                    int* order, int* woff, int* bad, cudaStream_t s);
void chain_count(int rows, const int* ro, const int* dg, const int* ci, int* cnt, cudaStream_t s);
// per-ticket slots (the sweep program): slot sizes in 16-byte units into
// off16 (rows entries; the caller scans them, off16[rows] = total), then the
// packed slots of one direction (rec4 = that direction's records).
void sweep_slot_sizes(int n, bool fwd, int rows, int depth, const int* rec4, int* off16, cudaStream_t s);
void sweep_pack(int n, bool fwd, int rows, int depth, const int* rec4, const int* ci, const double* v,
                const double* lu, const int* perm, const double* rcp, const int* off16, unsigned char* pk,
                cudaStream_t s);
// rec4: the sweep's ticket records, woff: warp ticket ranges (both read by
// the chain variant only, depth = -1)
void sweep_forward(int n, int rows, int depth, const int* off16, const unsigned char* pk, const int* rec4,
                   const int* woff, const int* ci, const double* v, const double* r, double* y, int* err,
                   cudaStream_t s);
void sweep_backward(int n, int rows, int depth, const int* off16, const unsigned char* pk, const int* rec4,
                    const int* woff, const int* ci, const double* v, const double* y, double* zb, double* z,
                    int accumulate, int* err, cudaStream_t s);
// number of mismatches of the reciprocal-based division against __ddiv_rn
unsigned long long selftest_division(unsigned long long n, unsigned long long seed);
unsigned long long selftest_latency(int op, int n);  // cycles of n dependent ops (0 dadd 1 dmul 2 dfma 3 shfl.f64 4 shfl.b32)
// total ns of n ping-pong round trips between two SMs (signalling flavour `mode`)
unsigned long long selftest_pingpong(int mode, int n);
void set_sweep_trace(unsigned long long* d, long long filter);  // filter: 0 any, else rows*2+fwd
unsigned long long selftest_chain(int variant, int L, int warps);  // total ns  // diagnostics: per-ticket timing trace

// ------------------------------------------------- device assembly (§8(f))
void assemble_inverse_src(int nnzb, const int* src, int* inv, cudaStream_t s);
// bkind: PatchKind per boundary face in bco order, or nullptr (all farfield)
// fsL/fsR: reconstructed face states (5 per internal face) or nullptr (first order);
// scheme: riemannFlux of the residual, 0 Roe, 1 HLLC, 2 Rusanov; *firstBad = min(*firstBad, first
// cell whose state is non-physical)
void assemble_euler(int nc, int nf, const int* owner, const int* neigh, const double* area, const int* cfo,
                    const int* cfl, const int* bco, const double* barea, const int* bkind, const double* fsL,
                    const double* fsR, int scheme, const double* q, const double* qinf, double cfl_num,
                    const int* inv, double* vals, double* rhs, int* firstBad, cudaStream_t s);
// musclReconstruct (euler.cpp:236-312): grad 15 per cell, psi 5 per cell, fsL/fsR 5 per face;
// limiter 0 none, 1 Barth-Jespersen
void assemble_euler_muscl(int nc, int nf, const int* owner, const int* neigh, const int* cfo, const int* cfl,
                          const double* cen, const double* fx, const double* q, int limiter, double* grad, double* psi,
                          double* fsL, double* fsR, cudaStream_t s);

void assemble_coupled(int nc, int nf, const int* owner, const int* neigh, const double* area, const double* fx,
                      const double* vol, const double* cen, const int* cfo, const int* cf, const int* bco,
                      const double* barea, const double* bu, const int* bkind, const double* bp,
                      const double* state, const double* phi, double nu, int pin, double pinValue, const int* inv,
                      double* D, double* grad, double* vals, double* rhs, cudaStream_t s);

// ------------------------------------------------------------ AMG (K9-K12)
void strengths(int n, int rows, const int* ro, const int* ci, const int* dg, const double* v, double* dn,
               double* str, int nnz, cudaStream_t s);
// greedy pairwise matching (amg.cpp:10-37), exact; choice[r]: -2 taken, -1 singleton, >=0 partner
void aggregate_kahn(int rows, const int* ro, const int* ci, const int* dg, const int* tpos, const double* str,
                    int* choice, KahnWork w, int* err, cudaStream_t s);
// same result, sync-free (no grid barriers); err set if a row could not decide
void aggregate_syncfree(int rows, const int* ro, const int* ci, const int* dg, const int* tpos, const double* str,
                        int* choice, int* err, cudaStream_t s);
// numbering: agg (rows), members (2 per coarse row); returns nCoarse (sync)
int aggregate_number(int rows, const int* choice, int* flag_tmp, int* agg, int* members, int* d_total,
                     int* scan_tmp, cudaStream_t s);
// Galerkin coarse operator (amg.cpp:39-71)
struct GalerkinTmp {
    int* seg_off;            // nCoarse+1
    unsigned long long* keys;// total
    unsigned long long* sorted;
    int* big;                // list of big segments
    int* nbig;               // 1
};
size_t galerkin_keys_size(int rows_coarse, const int* d_dummy);
// step 1: segment lengths into seg_off[c] (then caller scans)
void galerkin_seg_len(int nCoarse, const int* ro, const int* members, int* seg_off, cudaStream_t s);
void galerkin_keys(int nCoarse, const int* ro, const int* ci, const int* agg, const int* members,
                   const int* seg_off, unsigned long long* keys, cudaStream_t s);
void galerkin_sort(int nCoarse, const int* seg_off, const unsigned long long* keys, unsigned long long* sorted,
                   int* big, int* nbig, int* err, cudaStream_t s);
// coarse row lengths into cro[c] (then caller scans)
void galerkin_count(int nCoarse, const int* seg_off, const unsigned long long* sorted, int* cro, cudaStream_t s);
void galerkin_fill(int n, int nCoarse, const int* ro, const int* members, const int* seg_off,
                   const unsigned long long* sorted, const double* v, const int* cro, int* cci, double* cv,
                   cudaStream_t s);
void restrict_vec(int n, int nCoarse, const int* members, const double* res, double* rc, cudaStream_t s);
void prolong_vec(int n, int rows, const int* agg, const double* zc, double* z, cudaStream_t s);
// dense coarsest level (amg.cpp:91-104, smallmat.hpp:134-174)
void dense_build(int n, int rows, const int* ro, const int* ci, const double* v, double* dense, cudaStream_t s);
void dense_factor(int m, double* a, int* piv, int* err, cudaStream_t s);
void dense_solve(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s);
// the coarse tail of the V-cycle in one CTA (k_tail.cu).  Levels of the
// tail, top (largest) first, coarsest last; phase 0 = down path of all but the
// coarsest (pre-smoothing, residual, restriction), phase 1 = up path
// (prolongation, post-smoothing); the coarsest dense solve runs in between.
// rtop/ztop replace lv[0].r / lv[0].z.
struct TailLevelDev {
    int rows, ncoarse;
    const int *ro, *ci, *dg, *order, *agg, *members;
    const double *v, *lu, *rcp;
    const int* perm;
    double *r, *z, *res;
};
constexpr int kTailMaxRows = 512;
size_t tail_smem_bytes(int n, int rows);
void vcycle_tail(int n, int nl, const TailLevelDev* lv, int top_rows, const double* rtop, double* ztop, int pre,
                 int post, int phase, int* err, cudaStream_t s);
// blocked variants for large coarsest levels (k_dense.cu); piv: 2m ints
// (pivots, then the composed permutation the solve uses)
constexpr int kDenseBlockedMin = 256;
void dense_factor_blocked(int m, double* a, int* piv, int* err, cudaStream_t s);
// tolerance-level (tiled backward substitution) for large m; forward in reference order
void dense_solve_tiled(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s);
void dense_solve_big(int m, const double* lu, const int* piv, const double* r, double* z, cudaStream_t s);

// ------------------------------------------------------ Krylov (K13-K15)
int reduce_blocks();
// out[0] = dot(a, b)   (sqrt_out: out[0] = sqrt(dot)); deterministic.  The
// vector is nseg contiguous segments seg[0..nseg] (device int64 offsets);
// segment sums are folded with the reference's pairwise engine tree.
// partials >= reduce_blocks() + 4*nseg doubles.
void dot(const double* a, const double* b, const long long* seg, int nseg, double* out, bool sqrt_out,
         double* partials, int* ticket, cudaStream_t s, int bps = 0);
// w -= (*h) * v ; out = dot(w, nextv) (nextv == nullptr: out = sqrt(dot(w,w)))
void axpy_dot(double* w, const double* h, const double* v, const double* nextv, const long long* seg, int nseg,
              double* out, double* partials, int* ticket, cudaStream_t s, int bps = 0, int sqrt_mode = -1);
// Mode-R halo adds after the local product (partition.cpp:335-350)
// blocks per segment of the segmented reductions with nseg segments
int seg_blocks(int nseg);
// multi-process Mode R: engine partials folded in the reference's tree; rows packed for a halo send
void fold_engines(const double* parts, int G, double* out, bool sqrt_out, cudaStream_t s);
// exact mode: the reference's sequential dot order per segment + engine tree
void dot_seq(const double* a, const double* b, const long long* seg, int nseg, double* out, bool sqrt_out,
             double* partials, cudaStream_t s);
void axpy_dot_seq(double* w, const double* h, const double* v, const double* nextv, size_t N, const long long* seg,
                  int nseg, double* out, double* partials, bool sqrt_out, cudaStream_t s);
// the reference libm's hypot (glibc algorithm) on n device pairs
void hypot_eval(const double* x, const double* y, double* out, int n, cudaStream_t s);
void pack_rows(int n, int cnt, const int* idx, const double* x, double* out, cudaStream_t s);
void halo_spmv(int n, int nhr, const int* hrow, const int* hoff, const int* hcol, const double* hv, const double* x,
               double* y, int rowStart, cudaStream_t s);
// y = x / (*den) if (*den > thr) ; else untouched
void scale_by(const double* x, const double* den, double thr, double* y, size_t N, cudaStream_t s);
void copy_vec(const double* x, double* y, size_t N, cudaStream_t s);
void sub_vec(const double* b, const double* y, double* r, size_t N, cudaStream_t s);  // r = b - y
void add_to(double* x, const double* z, size_t N, cudaStream_t s);                     // x += z
// w = sum_{i<j} y_i V_i  (in i order, from 0.0)
void lincomb(const double* V, size_t ld, const double* y, int j, double* w, size_t N, cudaStream_t s);
// GMRES Givens step on device (krylov.cpp:104-117); status[0]=|g_{j+1}|, status[1]=happy
void givens_step(double* H, int m, int j, double* cs, double* sn, double* g, double* status, cudaStream_t s);
void back_subst(const double* H, int m, int j, const double* g, double* y, cudaStream_t s);
// BiCGStab elementwise updates (krylov.cpp:174-200)
void bicg_p(double* p, const double* r, const double* v, double bf, double omega, size_t N, cudaStream_t s);
void bicg_s(double* sv, const double* r, const double* v, double alpha, size_t N, cudaStream_t s);
void bicg_x_half(double* x, const double* ph, double alpha, size_t N, cudaStream_t s);
void bicg_x_r(double* x, double* r, const double* ph, const double* sh, const double* sv, const double* t,
              double alpha, double omega, size_t N, cudaStream_t s);

}  // namespace bcs
