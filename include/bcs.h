/*
 * bcs.h — C ABI of the B200-native block-coupled linear-solve path.
 *
 * One context drives one B200.  The boundary mirrors the reference's
 * SolvePipeline (proj/core/include/blockfv/engine.hpp:28-38,
 * proj/core/src/engine.cpp:47-120): face-addressed LDU upload, setup-or-
 * replace by topology signature, AMG/DILU/LUSGS-preconditioned GMRES or
 * BiCGStab to a relative tolerance, residual query.  Plain pointers and
 * sizes only; no exceptions cross the ABI (status codes + bcs_last_error),
 * which the C++ (include/bcs.hpp) and Python (paper_2403_07882_b200.bcs)
 * wrappers turn back into the reference's std::invalid_argument /
 * std::runtime_error semantics with the reference's message text.
 *
 * Layouts are exactly the reference host layouts:
 *   owner/neighbour : int32 per internal face, owner < neighbour (mesh.cpp:84-89)
 *   diag            : n_cells * n * n doubles, row-major n x n per cell
 *   upper / lower   : n_faces * n * n doubles (upper = (owner row, neighbour col),
 *                     lower = (neighbour row, owner col); block_matrix.hpp:40-87)
 *   vectors         : n_cells * n doubles, AoS per cell (block_matrix.hpp:20-30)
 * Block sizes 1..5 are supported on the device (hot configs: 4 and 5).
 *
 * Ownership: the caller owns every host array; it is read (or, for x,
 * written) during the call only.  *_device entry points take device pointers
 * on the context's device and enqueue on the context stream.
 * Threading: a context is not thread-safe (the reference solve is not
 * reentrant either); distinct contexts may be used from distinct
 * host threads at the same time.  Calls return with results valid.
 */
#ifndef BCS_H
#define BCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bcs_ctx bcs_ctx;

typedef enum {
    BCS_OK = 0,
    BCS_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    BCS_RUNTIME_ERROR = 2,    /* reference: std::runtime_error    */
    BCS_CUDA_ERROR = 3,
    BCS_NCCL_ERROR = 4,
    BCS_OUT_OF_MEMORY = 5
} bcs_status;

/* KrylovMethod / PrecondKind (krylov.hpp:15-16) */
enum { BCS_GMRES = 0, BCS_BICGSTAB = 1,
       /* Flexible GMRES (north_star "FGMRES"): the reference's Arnoldi process with
        * z_j = M^-1 v_j kept, x += Z y at restart/exit instead of x += M^-1(V y).
        * Identical Arnoldi scalars (residual history), one V-cycle fewer per
        * restart cycle; the update differs from GMRES only by rounding. */
       BCS_FGMRES = 2 };
enum { BCS_PRECOND_NONE = 0, BCS_PRECOND_LUSGS = 1, BCS_PRECOND_DILU = 2, BCS_PRECOND_AMG = 3 };
/* Backend (engine.hpp:17).  HOST_LDU keeps the reference's contract (only
 * none/LUSGS allowed, zero convert/setup/retrieve timings) but executes on the
 * device like every other path: there is no CPU fallback. */
enum { BCS_BACKEND_HOST_LDU = 0, BCS_BACKEND_ENGINE_CSR = 1 };

/* SolverConfig + AmgConfig (krylov.hpp:18-37).  The leading fields are
 * layout-identical to the oracle's or_cfg. */
typedef struct {
    int method;              /* BCS_GMRES | BCS_BICGSTAB | BCS_FGMRES (default GMRES) */
    int precond;             /* BCS_PRECOND_*                        (default LUSGS) */
    double rel_tol;          /* (default 1e-6)  */
    double abs_tol;          /* (default 1e-300) */
    int max_iters;           /* (default 500)   */
    int gmres_restart;       /* (default 30)    */
    int amg_max_levels;      /* (default 10)    */
    int amg_min_coarse_rows; /* (default 8)     */
    int amg_pre_sweeps;      /* (default 1)     */
    int amg_post_sweeps;     /* (default 1)     */
    int mode;                /* BCS_MODE_* (default BCS_MODE_PARITY) */
} bcs_solver_config;

/* Execution modes.
 * PARITY (default): every element-wise, block and per-row operation in the
 *   reference's order (bit-identical BSR, SpMV, LU, LUSGS/DILU, Galerkin,
 *   V-cycle, vector updates; the reference libm's hypot in the Givens
 *   rotation); global dot products are deterministic two-level trees, the
 *   only association that differs from the reference.
 * PERF: the north_star performance smoothers -- multicolour block DILU on
 *   every AMG level (deterministic colouring, colour-parallel sweeps) instead
 *   of the natural-order sweeps; iteration counts differ from the reference
 *   and are reported, never silently substituted.
 * EXACT: PARITY plus the reference's own dot order (defaultDot,
 *   krylov.cpp:38-42: one sequential chain per engine, engine partials
 *   folded by the pairwise tree of partition.cpp:433-450): residual
 *   histories and solutions are bit-identical to the reference.  A dot is
 *   then a serial chain of N dependent adds (~4.3 ns each): a proof mode. */
enum { BCS_MODE_PARITY = 0, BCS_MODE_PERF = 1, BCS_MODE_EXACT = 2,
       /* PERF with block-Jacobi smoothing (z += 0.8 D^-1 r per block row; of the
        * dampings 0.8 / 0.9 / 1.0 the 128^3 bench needed 18 / 22 / 94 iterations)
        * on every level above the one-CTA tail: dependency-free, HBM-streaming,
        * weaker than DILU (more iterations, fewer seconds). */
       BCS_MODE_PERF_JACOBI = 3 };

/* SolveReport (krylov.hpp:39-50) + per-stage timings (seconds) with the
 * reference keys (engine.cpp:80-112) and device sub-stages. */
typedef struct {
    int iterations;
    int converged;
    int breakdown;
    int setup_branch; /* 1: setup (first call / topology change); 0: replace */
    double initial_residual;
    double final_residual;
    double t_convert, t_setup, t_replace, t_solve, t_retrieve;
    double t_amg_setup; /* preconditioner construction inside "solve" */
    double t_krylov;    /* Krylov iterations inside "solve"          */
    int amg_levels;
    int coarse_rows;    /* rows of the coarsest level (dense LU is coarse_rows*n) */
    /* kernel-level accounting (filled when bcs_set_kernel_timing(ctx,1)) */
    int spmv_launches;
    double spmv_ms;     /* summed CUDA-event time of the fine-level SpMV launches */
    int kernel_launches;/* device kernels launched during the call */
    int sweep_launches; /* smoother sweeps (every level) bracketed by events */
    double sweep_ms;    /* their summed CUDA-event time */
    double sweep_bytes; /* their summed algorithmic bytes (sweeps) */
} bcs_report;

void bcs_default_config(bcs_solver_config* cfg);
const char* bcs_version(void);

bcs_status bcs_create(bcs_ctx** out, int device);
bcs_status bcs_destroy(bcs_ctx* ctx);
const char* bcs_last_error(const bcs_ctx* ctx);
/* Run all device work of this context on `stream` (a cudaStream_t); NULL
 * restores the context's own stream. */
bcs_status bcs_set_stream(bcs_ctx* ctx, void* stream);
bcs_status bcs_set_kernel_timing(bcs_ctx* ctx, int enable);

/* Page-locked host buffers from a process-wide cache (cudaHostAlloc'd blocks
 * are kept on free and reused by the next request of the same size class), so
 * a caller that allocates its result vectors here gets full-rate DMA and no
 * page faults on every call.  The Python mirror allocates the BlockVector
 * returned by SolvePipeline::solve this way. */
bcs_status bcs_host_alloc(size_t bytes, void** out);
void bcs_host_free(void* p);

/* Binary LDU dump (the reference only has a text mesh
 * format, mesh.cpp:214-283): one file per system, host only.
 *   header 64 bytes: "BCSLDU01", int32 version (1), n_cells, n_faces,
 *   block_size, flags (bit 0: b present, bit 1: x0 present), uint64 FNV-1a of
 *   the payload, zero padding;
 *   payload, little endian: owner[n_faces], neighbour[n_faces] (int32),
 *   diag[n_cells n^2], upper[n_faces n^2], lower[n_faces n^2] (float64,
 *   row-major blocks), then b[n_cells n] and x0[n_cells n] when flagged.
 * b / x0 may be NULL on save (not stored) and on load (skipped).  A file that
 * is truncated, has another magic or fails the checksum -> BCS_RUNTIME_ERROR. */
bcs_status bcs_ldu_save(const char* path, int n_cells, int n_faces, int block_size, const int32_t* owner,
                        const int32_t* neighbour, const double* diag, const double* upper, const double* lower,
                        const double* b, const double* x0);
bcs_status bcs_ldu_load_sizes(const char* path, int* n_cells, int* n_faces, int* block_size, int* has_b,
                              int* has_x0);
bcs_status bcs_ldu_load(const char* path, int32_t* owner, int32_t* neighbour, double* diag, double* upper,
                        double* lower, double* b, double* x0);

/* topologySignature (block_csr.cpp:146-160), exact; host only. */
uint64_t bcs_topology_signature(int n_cells, int n_faces, const int32_t* owner, const int32_t* neighbour);

/* ---- drop-in: one SolvePipeline::solve call (engine.cpp:47-120) ---------
 * Host arrays.  b_len / x0_len are the element counts of b / x0 (the
 * reference's BlockVector dimension check, engine.cpp:50-52).  x receives
 * n_cells*n doubles.  Setup-or-replace is decided as the reference does, by
 * topology signature against the previous call on this context. */
bcs_status bcs_pipeline_solve(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                              const int32_t* neighbour, const double* diag, const double* upper,
                              const double* lower, const double* b, size_t b_len, const double* x0,
                              size_t x0_len, double* x, int backend, const bcs_solver_config* cfg,
                              bcs_report* report);

/* ---- Mode R: the reference's distributed semantics --------------------------
 * distributedSolve(buildPartitioned(A, decompose(mesh, n_ranks)), ...) with
 * makeConsolidationPlan(dec, n_engines) (partition.cpp:21-479): RCB on the
 * cell centroids (n_cells*3 doubles), rank-major renumbering, ranks
 * consolidated onto engines, one local preconditioner per engine, global
 * Krylov with halo couplings and the fixed pairwise engine tree for dot
 * products.  All engines run on this context's device; b, x0 and x are in
 * the original cell order.  Timings use the reference keys convert / setup /
 * solve / retrieve (partition.cpp:474-477). */
bcs_status bcs_dist_solve(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                          const int32_t* neighbour, const double* centroids, const double* diag, const double* upper,
                          const double* lower, const double* b, const double* x0, double* x, int n_ranks,
                          int n_engines, const bcs_solver_config* cfg, bcs_report* report);

/* distributedSolve(rankParts, b, x0, cfg, plan, dec, net) itself
 * (partition.hpp, partition.cpp:370-479) on partitions the caller already
 * built (e.g. the reference's buildPartitioned): rank r owns the global rows
 * [rank_row_offset[r], rank_row_offset[r+1]) (new, rank-major numbering),
 * with its local BSR (local_row_offsets[r]: rows+1, local_cols[r] local
 * column ids, local_values[r] n*n blocks row-major) and halo_counts[r]
 * off-rank couplings (halo_rows[r] local row, halo_cols[r] global column,
 * halo_peers[r] owning rank, halo_values[r] blocks).  The ranks are
 * consolidated onto n_engines engines by the caller's ConsolidationPlan
 * (rank_to_engine, engine_row_offset: partition.cpp:184-199) exactly as the
 * reference's consolidate (partition.cpp:201-248).  b, x0 and x are global
 * vectors in the new numbering (the rank slices of a DistributedVector
 * concatenated in rank order).  Same engine semantics, timing keys and
 * EXACT-mode bit-identity as bcs_dist_solve. */
bcs_status bcs_dist_solve_parts(bcs_ctx* ctx, int n_ranks, int block_size, const int32_t* rank_row_offset,
                                const int32_t* const* local_row_offsets, const int32_t* const* local_cols,
                                const double* const* local_values, const int32_t* halo_counts,
                                const int32_t* const* halo_rows, const int32_t* const* halo_cols,
                                const int32_t* const* halo_peers, const double* const* halo_values, int n_engines,
                                const int32_t* rank_to_engine, const int32_t* engine_row_offset, const double* b,
                                const double* x0, double* x, const bcs_solver_config* cfg, bcs_report* report);

/* Host-side partition layer (no device needed): decompose + buildPartitioned
 * (+ consolidate when n_engines > 0).  Local slots and halo entries carry the
 * id of their LDU source block: cell c -> c, upper of face f -> n_cells + f,
 * lower of face f -> n_cells + n_faces + f. */
typedef struct bcs_partition bcs_partition;
bcs_status bcs_partition_create(bcs_partition** out, int n_cells, int n_faces, const int32_t* owner,
                                const int32_t* neighbour, const double* centroids, int n_ranks, int n_engines);
void bcs_partition_destroy(bcs_partition* p);
int bcs_partition_count(const bcs_partition* p);
bcs_status bcs_partition_decomposition(const bcs_partition* p, int32_t* cell_to_rank, int32_t* rank_row_offset,
                                       int32_t* old_to_new);
bcs_status bcs_partition_sizes(const bcs_partition* p, int part, int* row_start, int* row_end, int* nnz, int* n_halo,
                               int* n_send);
bcs_status bcs_partition_get(const bcs_partition* p, int part, int32_t* row_offsets, int32_t* cols, int32_t* src,
                             int32_t* halo_row, int32_t* halo_col, int32_t* halo_peer, int32_t* halo_src,
                             int32_t* send_peer, int32_t* send_row);

/* Exchange plan of engine `part` for one process per engine (host only):
 * n_send rows it packs (send_row, local rows; send_count[peer], peers
 * ascending), n_recv rows it receives (recv_global_row, renumbered global
 * rows; recv_count[peer]) and, per halo entry, the position of its column
 * in the receive buffer.  Counts arrays have count() entries. */
bcs_status bcs_partition_exchange_sizes(const bcs_partition* p, int part, int* n_send, int* n_recv);
bcs_status bcs_partition_exchange_get(const bcs_partition* p, int part, int32_t* send_row, int32_t* send_count,
                                      int32_t* recv_global_row, int32_t* recv_count, int32_t* halo_recv_idx);

/* The reference's per-rank upload (partition.cpp:384-407) of engine `part`:
 * the LDU blocks of its local slots (slot order, nnz * n^2 doubles) and of
 * its halo entries (entry order, n_halo * n^2 doubles) gathered on the host
 * from the face-addressed arrays; bcs_dist_solve_mp ships exactly these to
 * the engine's GPU.  Either output may be NULL. */
bcs_status bcs_partition_gather_values(const bcs_partition* p, int part, int n_cells, int n_faces, int block_size,
                                       const double* diag, const double* upper, const double* lower,
                                       double* local_values, double* halo_values);

/* ---- Mode R with one process per GPU (NCCL) -------------------------------
 * bcs_comm_unique_id fills 128 bytes on one rank; every rank passes them to
 * bcs_comm_init (collective).  bcs_dist_solve_mp is then called collectively
 * with the whole system on every rank (LinearDispatch's inputs): rank r owns
 * engine r (n_engines = number of processes), builds its local matrix,
 * halo plan and preconditioner, and the global Krylov exchanges halos with
 * NCCL send/recv and folds per-engine dot partials (NCCL all-gather) in the
 * reference's engine tree — the same arithmetic as bcs_dist_solve with the
 * engines on one device.  x (original cell order) is complete on every rank. */
bcs_status bcs_comm_unique_id(unsigned char id[128]);
bcs_status bcs_comm_init(bcs_ctx* ctx, int rank, int n_ranks_total, const unsigned char id[128]);
bcs_status bcs_dist_solve_mp(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                             const int32_t* neighbour, const double* centroids, const double* diag,
                             const double* upper, const double* lower, const double* b, const double* x0, double* x,
                             int n_ranks, const bcs_solver_config* cfg, bcs_report* report);

/* ---- staged interface (device-resident workflows) ------------------------ */
/* Builds the LDU->BSR plan (block_csr.cpp:56-80) on the device. */
bcs_status bcs_set_topology(bcs_ctx* ctx, int n_cells, int n_faces, int block_size, const int32_t* owner,
                            const int32_t* neighbour);
/* Value permutation LDU->BSR (replaceValues, block_csr.cpp:120-127). */
bcs_status bcs_upload_ldu(bcs_ctx* ctx, const double* diag, const double* upper, const double* lower);
bcs_status bcs_upload_ldu_device(bcs_ctx* ctx, const double* d_diag, const double* d_upper,
                                 const double* d_lower);
/* Preconditioner build + Krylov on the current matrix; x holds x0 on entry. */
/* Device assembly of the 5x5 density-based system:
 * replaces assembleJacobian + computeResidual (euler.cpp:361-455) for
 * first-order reconstruction, the Roe flux and farfield patches (ghost state
 * = freestream).  Mesh: owner/neighbour per internal face (sets the topology
 * when it differs), face_area 3 per internal face (owner -> neighbour), the
 * boundary faces in patch order (cell, outward area vector), q the primitive
 * state (rho, u, v, w, p) per cell, q_inf the freestream, cfl the pseudo-time
 * CFL (<= 0: none).  The matrix goes straight into the context's block-CSR
 * (as bcs_upload_ldu would put it, bit-identical); rhs (host, 5 per cell)
 * receives the permuted residual. */
bcs_status bcs_assemble_euler(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner, const int32_t* neighbour,
                              const double* face_area, int n_bfaces, const int32_t* bface_cell,
                              const double* bface_area, const double* q, const double* q_inf, double cfl,
                              double* rhs);
/* bcs_assemble_euler with a patch kind per boundary face (ghostState,
 * euler.cpp:320-341; EulerCase::patchOverride resolved by the caller):
 * bface_kind = the reference's PatchKind order, 0 wall, 1 inlet, 2 outlet,
 * 3 farfield, 4 slip, 5 symmetry.  Wall/slip/symmetry reflect the interior
 * velocity, inlet/farfield take q_inf, outlet the interior state.  Any other
 * value: BCS_INVALID_ARGUMENT "unknown patch kind" (euler.cpp:340).
 * bface_kind == NULL is bcs_assemble_euler (all farfield). */
bcs_status bcs_assemble_euler_patches(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                      const int32_t* neighbour, const double* face_area, int n_bfaces,
                                      const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                      const double* q, const double* q_inf, double cfl, double* rhs);
/* The general Euler assembly: bcs_assemble_euler_patches plus the
 * EulerCase choices that shape the residual.  recon (ReconstructionConfig,
 * euler.hpp:62-65): 0 first order, 1 MUSCL without limiter, 2 MUSCL +
 * Barth-Jespersen (musclReconstruct, euler.cpp:236-312: least-squares
 * primitive gradients :205-234, first order where a reconstructed state is
 * non-physical); flux (FluxScheme order, euler.hpp:51): 0 Roe, 1 HLLC,
 * 2 Rusanov (riemannFlux :195-203, used on internal and boundary faces).
 * The Jacobian stays the first-order Roe-dissipation one, as in
 * assembleJacobian.  face_fx (owner-side weight per internal face; face
 * centre = fx c_owner + (1 - fx) c_neighbour, mesh.hpp:55-59) and
 * cell_centroid (3 per cell) are read only when recon > 0; bface_kind may
 * be NULL (all farfield).  Unknown flux: "unknown flux scheme". */
bcs_status bcs_assemble_euler_ex(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                 const int32_t* neighbour, const double* face_area, const double* face_fx,
                                 const double* cell_centroid, int n_bfaces, const int32_t* bface_cell,
                                 const double* bface_area, const int32_t* bface_kind, const double* q,
                                 const double* q_inf, int recon, int flux, double cfl, double* rhs);
/* Device assembly of the 4x4 pressure-based coupled p-U system: replaces
 * assembleCoupled (incompressible.cpp:143-250: momentumDiagCoeff, least-
 * squares pressure gradients, upwind + diffusion momentum, fx-interpolated
 * pressure gradient, negated continuity with the Rhie-Chow compact Laplacian)
 * followed by pinPressure(pin_cell, pin_value) (:252-264), for wall (kind 0)
 * and moving-wall (kind 1, wall velocity bface_u) patches.  face_fx: the
 * owner-side interpolation weight per internal face; cell_vol, cell_centroid
 * (3 per cell); state (u, v, w, p per cell); phi the face fluxes; nu the
 * viscosity; pin_cell < 0: no pinning.  Values go straight into the context's
 * block-CSR, bit-identical to uploading the reference's LDU matrix; rhs (host,
 * 4 per cell) receives the right-hand side. */
bcs_status bcs_assemble_coupled(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                const int32_t* neighbour, const double* face_area, const double* face_fx,
                                const double* cell_vol, const double* cell_centroid, int n_bfaces,
                                const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                const double* bface_u, const double* state, const double* phi, double nu,
                                int pin_cell, double pin_value, double* rhs);
/* bcs_assemble_coupled for every IncompressibleBc kind (incompressible.hpp:24-29;
 * momentumDiagCoeff's and assembleCoupled's patch terms, incompressible.cpp:70-86,
 * 203-247): bface_kind 0 wall, 1 moving wall, 2 inlet (velocity bface_u,
 * known flux), 3 outlet (zero-gradient velocity, fixed pressure bface_p, one
 * per boundary face; may be NULL when there is no outlet). */
bcs_status bcs_assemble_coupled_ex(bcs_ctx* ctx, int n_cells, int n_faces, const int32_t* owner,
                                   const int32_t* neighbour, const double* face_area, const double* face_fx,
                                   const double* cell_vol, const double* cell_centroid, int n_bfaces,
                                   const int32_t* bface_cell, const double* bface_area, const int32_t* bface_kind,
                                   const double* bface_u, const double* bface_p, const double* state,
                                   const double* phi, double nu, int pin_cell, double pin_value, double* rhs);
bcs_status bcs_solve(bcs_ctx* ctx, const double* b, double* x, const bcs_solver_config* cfg, bcs_report* report);
bcs_status bcs_solve_device(bcs_ctx* ctx, const double* d_b, double* d_x, const bcs_solver_config* cfg,
                            bcs_report* report);

/* ---- residual query and per-kernel entry points (parity tests / bench) --- */
bcs_status bcs_residual(bcs_ctx* ctx, const double* b, const double* x, double* norm);
/* relative residual per Krylov step of the last solve (same definition as
 * the oracle: |g_{j+1}|/beta0, true residual at restarts/exit). */
bcs_status bcs_residual_history(bcs_ctx* ctx, double* out, int cap, int* n);
bcs_status bcs_spmv(bcs_ctx* ctx, const double* x, double* y);                  /* host arrays   */
bcs_status bcs_spmv_device(bcs_ctx* ctx, const double* d_x, double* d_y);        /* device arrays */
bcs_status bcs_csr_get(bcs_ctx* ctx, int32_t* row_offsets, int32_t* cols, double* values);
bcs_status bcs_precond_setup(bcs_ctx* ctx, const bcs_solver_config* cfg);
bcs_status bcs_precond_apply(bcs_ctx* ctx, const double* r, double* z);          /* host arrays   */
bcs_status bcs_amg_depth(bcs_ctx* ctx, int* depth);
bcs_status bcs_amg_level_sizes(bcs_ctx* ctx, int level, int* rows, int* nnz);
bcs_status bcs_amg_level_get(bcs_ctx* ctx, int level, int32_t* row_offsets, int32_t* cols, double* values,
                             int32_t* aggregate /* rows entries, or NULL; coarsest has none */);
/* Level schedule of the last DILU/LUSGS setup of `level`: number of
 * dependency levels of its lower-triangular DAG (critical path). */
bcs_status bcs_level_schedule_depth(bcs_ctx* ctx, int level, int* depth);

/* Diagnostics: the device restatement of the reference libm's hypot (used by
 * the Givens rotation) on n host pairs -- the test pins it against libm. */
bcs_status bcs_selftest_hypot(const double* x, const double* y, double* out, int n);

/* Device memory held by the context, per category (bytes), as a JSON object
 * {"bsr_fine": .., "bsr_coarse": .., "sweep_programs": .., ..., "total": ..}.
 * *needed = length + 1; buf may be NULL (size query). */
bcs_status bcs_memory_report(bcs_ctx* ctx, char* buf, size_t cap, size_t* needed);

/* Performance mode: the multicolouring of level `level`'s smoother after a
 * BCS_MODE_PERF setup: *n_colors (0 when the level is smoothed in natural
 * order), if perm != NULL its row order perm[new] = row (rows sorted by
 * (colour, row)) and if color_offsets != NULL the n_colors + 1 boundaries of
 * the colours in that order; the smoother is the natural-order DILU of the
 * symmetrically permuted level matrix. */
bcs_status bcs_level_coloring(bcs_ctx* ctx, int level, int* n_colors, int32_t* perm, int32_t* color_offsets);

/* Device self-tests (diagnostics).  what = 0: the sweeps' reciprocal-based
 * exact division against IEEE __ddiv_rn on n random operand pairs; *result =
 * number of bit mismatches (must be 0).  what = 10..14: total ns of n cross-SM
 * ping-pong round trips with signalling flavour what-10 (0 relaxed, 1 relaxed +
 * fence, 2 atomic exchange, 3 volatile, 4 release/acquire).  what = 20: per-row
 * sweep trace into the device buffer at address seed (10 u64 per ticket), n = 0
 * removes it, n = 1 traces every sweep, n > 1 only sweeps with rows*2+fwd == n.
 * what = 30/31: n-hop minimal chain, total ns.  what = 40..44: cycles of n
 * dependent dadd / dmul / dfma / f64 shuffle / b32 shuffle on one warp. */
bcs_status bcs_selftest(int what, unsigned long long n, unsigned long long seed, unsigned long long* result);

#ifdef __cplusplus
}
#endif
#endif /* BCS_H */
