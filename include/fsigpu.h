/* SPDX-License-Identifier: Apache-2.0
 *
 * fsigpu — B200 (sm_100a) solve path for the monolithic FSI Jacobians of
 * arXiv:1909.13201 (reference "fsibench", /root/reference/proj).
 *
 * C ABI: plain pointers and sizes, int status codes, thread-local last
 * error string.  Every entry point replaces a reference interface on the
 * solve path; the reference symbol each one stands in for is cited
 * (file:line into proj/).  Host-pointer entry points copy in/out; the *_dev
 * variants take device pointers and an optional cudaStream_t (NULL = the
 * handle's own stream) for fully device-resident use.
 *
 * Error behaviour mirrors the reference's exceptions:
 *   FSIGPU_ERR_INVALID   <- std::invalid_argument (bad sizes / config)
 *   FSIGPU_ERR_SINGULAR  <- fsi::SingularBlockError (label via
 *                           fsigpu_last_singular_block(): lowest failing block
 *                           of the batch, and fsigpu_last_singular_level():
 *                           its GMG level; block -1 = a non-block failure
 *                           named by the message, e.g. "gmg-coarse" or
 *                           "fs lumped mass row <i>", precond.cpp:239-241)
 *   FSIGPU_ERR_CUDA      <- device failure (no reference analogue)
 * GMRES non-convergence is reported in fsigpu_gmres_result, not as an error
 * (krylov.hpp:49-55).
 */
#ifndef FSIGPU_H
#define FSIGPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define FSIGPU_OK 0
#define FSIGPU_ERR_INVALID 1
#define FSIGPU_ERR_SINGULAR 2
#define FSIGPU_ERR_CUDA 3

typedef struct fsigpu_csr_t* fsigpu_csr;
typedef struct fsigpu_blocks_t* fsigpu_blocks;
typedef struct fsigpu_gmg_t* fsigpu_gmg;
typedef struct fsigpu_gmres_t* fsigpu_gmres;

/* One multigrid level as the reference driver fills GmgLevel + the FS
 * smoother inputs (driver.cpp:229-256, gmg.hpp:60-68, precond.hpp:95-124).
 * Level 0 uses only n, a_*, row_mask, col_mask. */
typedef struct {
  int n;
  const int* a_ptr; /* frame (J2) CSR, int32 offsets/cols, fp64 values */
  const int* a_idx;
  const double* a_val;
  const unsigned char* row_mask; /* GmgLevel::constrained_rows */
  const unsigned char* col_mask; /* GmgLevel::constrained_cols */
  int nc;                        /* size of level l-1 */
  const int* p_ptr;              /* GmgLevel::p, n x nc */
  const int* p_idx;
  const double* p_val;
  const int* r_ptr; /* GmgLevel::r, nc x n */
  const int* r_idx;
  const double* r_val;
  int g1;                /* FsPreconditioner::group1_size()          */
  int n_us;              /* FsPreconditioner::solid_velocity_size()  */
  const double* lumped;  /* FsPreconditioner::lumped(), n_us values  */
  int as1_n;             /* AS1 blocks: frame positions in [0, g1)   */
  const int* as1_ptr;
  const int* as1_idx;
  int as2_n; /* AS2 fluid blocks: group-2 local positions */
  const int* as2_ptr;
  const int* as2_idx;
} fsigpu_level_desc;

typedef struct {
  int iterations; /* Arnoldi steps (GmresResult::iterations)  */
  int converged;
  int breakdown;
  int n_history;  /* history[0] = ||r0||, then one entry per step */
  long long m_applies; /* GMG V-cycles applied */
  double true_residual; /* ||b - A x|| at exit */
} fsigpu_gmres_result;

/* ---- runtime ------------------------------------------------------- */
const char* fsigpu_last_error(void);
int fsigpu_last_singular_block(void);
int fsigpu_last_singular_level(void);
int fsigpu_init(int device);
int fsigpu_version(void);
/* number of libfsigpu kernel launches issued so far (graph replays included) */
long long fsigpu_launch_count(void);

/* ---- CSR SpMV: SparseMatrix::multiply (sparse.cpp:70-76),
 *      CsrOperator::apply (krylov.cpp:16) -------------------------------- */
int fsigpu_csr_create(int rows, int cols, const int* ptr, const int* idx, const double* val,
                      fsigpu_csr* out);
int fsigpu_csr_multiply(fsigpu_csr a, const double* x, double* y);
int fsigpu_csr_multiply_dev(fsigpu_csr a, const double* d_x, double* d_y, void* stream);
/* average device time (ms) of `reps` back-to-back SpMV launches (CUDA events) */
int fsigpu_csr_time(fsigpu_csr a, int reps, double* ms_per_launch);
void fsigpu_csr_destroy(fsigpu_csr a);

/* ---- batched dense blocks: DenseFactorization ctor / solve
 *      (dense.cpp:31-86), factor_principal_block (precond.cpp:13-21) ----- */
/* principal blocks A[dofs, dofs] of a CSR matrix, batched extract + LU */
int fsigpu_blocks_factor_csr(fsigpu_csr a, int n_blocks, const int* block_ptr,
                             const int* block_idx, fsigpu_blocks* out);
/* dense row-major blocks concatenated, sizes[b] x sizes[b] each */
int fsigpu_blocks_factor_dense(int n_blocks, const int* sizes, const double* mats,
                               fsigpu_blocks* out);
/* config-1 generator on the device: n54 blocks of m=54 then n59 of m=59,
 * entries uniform[-1,1] from a counter hash of (seed, block, i, j), diagonal
 * shifted by the row's absolute sum; rhs sets generated alike. */
int fsigpu_blocks_generate_dominant(long long n54, long long n59, unsigned long long seed,
                                    fsigpu_blocks* out);
int fsigpu_blocks_generate_rhs(fsigpu_blocks b, unsigned long long seed, double* d_rhs);
int fsigpu_blocks_copy_matrix(fsigpu_blocks b, long long block, double* rowmajor);
long long fsigpu_blocks_count(fsigpu_blocks b);
long long fsigpu_blocks_total_rows(fsigpu_blocks b);
long long fsigpu_blocks_factor_bytes(fsigpu_blocks b);
int fsigpu_blocks_solve(fsigpu_blocks b, const double* rhs, double* x);
int fsigpu_blocks_solve_dev(fsigpu_blocks b, const double* d_rhs, double* d_x, void* stream);
/* refactor in place from the retained matrices (config-1 LU timing) */
int fsigpu_blocks_refactor(fsigpu_blocks b, void* stream);
/* LU factors back to the host: row-major per block like DenseFactorization,
 * plus LAPACK-style pivots piv[k] (dense.cpp:45-51) */
int fsigpu_blocks_get_lu(fsigpu_blocks b, double* lu_rowmajor, int* piv);
void fsigpu_blocks_destroy(fsigpu_blocks b);

/* Block-solve mode of the FS smoothers of GMG hierarchies created after the
 * call: 0 = LU forward/back substitution (tiled), 1 = explicit block inverse
 * computed at setup from the same LU (one batched GEMV + combine per sweep),
 * 2 = the additive FS operator assembled from those inverses as one sparse
 * matrix (default; one fused SpMV "x += omega FS r" per sweep). */
#define FSIGPU_MODE_LU 0
#define FSIGPU_MODE_INVERSE 1
#define FSIGPU_MODE_ASSEMBLED 2
int fsigpu_set_block_mode(int mode);
/* programmatic dependent launch of the solve-path kernels (default on: each kernel fetches its
 * setup data before griddepcontrol.wait; config 0: 8.45 -> 7.96 ms per solve) */
int fsigpu_set_pdl(int enable);

/* Level smoother of every smoothed level: 0 = damped Richardson with the
 * create() omega (reference richardson_smooth, src/precond.cpp:305-317; the
 * default), 1 = GMRES(1) minimal-residual step  x += alpha FS(b - A x),
 * alpha = (w.r)/(w.w), w = A FS r  (BASELINE.json configs[0] "1 pre- and 1
 * post-step GMRES(1)"; not in the reference). GMRES(1) makes the
 * V-cycle non-linear: use it under the flexible device solver
 * (fsigpu_gmres_*). Invalidates graphs captured by existing solvers. */
int fsigpu_gmg_set_smoother(fsigpu_gmg g, int kind);

/* ---- GMG with additive FS smoothers: GmgPreconditioner (gmg.cpp:178-246),
 *      FsPreconditioner (precond.cpp:119-303, additive per SURVEY §8c),
 *      richardson_smooth (precond.cpp:305-317) ---------------------------- */
int fsigpu_gmg_create(int n_levels, const fsigpu_level_desc* levels, double omega, int pre,
                      int post, char cycle, fsigpu_gmg* out);
/* The same with the Schwarz mode of the FS smoothers (SchwarzMode,
 * include/fsi/precond.hpp): additive (the default above) or
 * multiplicative, the reference's shipped FsPreconditioner::apply
 * (precond.cpp:59-77,271-303) with the blocks run in multicolour order:
 * same-colour blocks share no dof and do not couple, so each colour is one
 * parallel step (block order differs from the reference's; the CPU
 * restatement runs the same order). */
#define FSIGPU_SCHWARZ_ADDITIVE 0
#define FSIGPU_SCHWARZ_MULTIPLICATIVE 1
int fsigpu_gmg_create_ex(int n_levels, const fsigpu_level_desc* levels, double omega, int pre,
                         int post, char cycle, int schwarz, fsigpu_gmg* out);
int fsigpu_gmg_size(fsigpu_gmg g);
/* the cudaStream_t every GMG / GMRES kernel of this handle is launched on */
void* fsigpu_gmg_stream(fsigpu_gmg g);
int fsigpu_gmg_apply(fsigpu_gmg g, const double* r, double* z);
int fsigpu_gmg_apply_dev(fsigpu_gmg g, const double* d_r, double* d_z, void* stream);
int fsigpu_fs_apply(fsigpu_gmg g, int level, const double* r, double* z);
int fsigpu_coarse_solve(fsigpu_gmg g, const double* b, double* x);
void fsigpu_gmg_destroy(fsigpu_gmg g);
/* Device time (ms, CUDA events on the hierarchy stream) of one launch of a
 * V-cycle kernel on `level` and its algorithmic bytes. which: 0 FS smoother
 * SpMV, 1 level residual SpMV, 2 prolongation + fused residual, 3
 * restriction, 4 coarse GEMV (level 0). cold: flush L2 (256 MB) before each
 * launch; else back to back. */
/* tuning: lanes per row and batch depth of a level matrix's SpMV launches
 * (which: 0 A, 1 FS, 2 A*P, 3 P, 4 R) */
int fsigpu_gmg_set_launch(fsigpu_gmg g, int level, int which, int lpr, int unroll);
int fsigpu_gmg_time_kernel(fsigpu_gmg g, int which, int level, int reps, int cold, double* ms,
                           double* bytes);

/* ---- block sets built on the device: FsPreconditioner's field-split
 *      sets (precond.cpp:119-269) and the Vanka sets of the pure-DD smoother
 *      (build_vanka_blocks, ordering.cpp:77-115, as AsPreconditioner maps
 *      them, precond.cpp:99-117), from the mesh-side index maps in the
 *      solver's frame. Replaces constructing (and CPU-factorising) the
 *      reference FsPreconditioner / AsPreconditioner to obtain the sets. --- */
typedef struct fsigpu_sets_t* fsigpu_sets;
typedef struct {
  int n_elements;
  int n_nodes;                      /* Q2 nodes (DofMap::n_q2_nodes)                  */
  int nodes_per_element;            /* 9 (2D Q2) or 27 (3D Q2)                        */
  int dim;                          /* components of d and u (2 or 3)                 */
  int p_per_element;                /* P1disc modes per element (3 in 2D, 4 in 3D)    */
  const int* element_nodes;         /* n_elements x nodes_per_element                 */
  const unsigned char* elem_solid;  /* FieldLayout::elem_solid                        */
  const unsigned char* node_solid;  /* FieldLayout::node_solid                        */
  const int* d_pos;                 /* n_nodes x dim: frame_of(d_dof(node, i))        */
  const int* u_pos;                 /* n_nodes x dim: frame_of(u_dof(node, i))        */
  const int* p_pos;                 /* n_elements x p_per_element: frame_of(p_dof)    */
  const unsigned char* drop;        /* constrained_positions (precond.cpp:90-97), or NULL */
} fsigpu_mesh_desc;
/* level: n, a_* (frame matrix), g1, n_us are read (the sets are ignored).
 * AS1: solid [d^s,p^s] chunks of epb_as1 elements, then fluid d^f chunks of
 * epb_as1 grown by overlap_layers rings; AS2: fluid [u^f,p^f] chunks of
 * epb_as2 (group-2 local); lumped u^s mass (precond.cpp:231-245; a
 * non-positive row sum -> FSIGPU_ERR_SINGULAR "fs lumped mass row <i>"). */
int fsigpu_fs_sets_build(const fsigpu_level_desc* level, const fsigpu_mesh_desc* mesh, int epb_as1,
                         int epb_as2, int overlap_layers, fsigpu_sets* out);
/* Vanka sets (J1 frame positions) as AS1 blocks of a one-group level */
int fsigpu_vanka_sets_build(int n, const fsigpu_mesh_desc* mesh, int epb, fsigpu_sets* out);
int fsigpu_sets_counts(fsigpu_sets s, int* as1_n, int* as1_len, int* as2_n, int* as2_len, int* n_us);
int fsigpu_sets_copy(fsigpu_sets s, int* as1_ptr, int* as1_idx, int* as2_ptr, int* as2_idx,
                     double* lumped);
/* the reference label of block b (AS1 then AS2): fs-solid-dp-<start>, ... */
const char* fsigpu_sets_label(fsigpu_sets s, int block);
void fsigpu_sets_destroy(fsigpu_sets s);

/* ---- outer solver: gmres (krylov.cpp:20-126) on the row-equilibrated
 *      frame operator diag(frame_scale) A_top with M(r) = GMG(r/frame_scale)
 *      (driver.cpp:259-272).  Implemented as FGMRES(restart) with CGS2
 *      Arnoldi (identical to the reference's right-preconditioned GMRES in
 *      exact arithmetic for the fixed linear V-cycle). ------------------- */
int fsigpu_gmres_create(fsigpu_gmg g, const double* frame_scale, int restart, fsigpu_gmres* out);
int fsigpu_gmres_solve(fsigpu_gmres s, const double* b, const double* x0, double* x, int max_iters,
                       double rel_tol, double abs_tol, double* history, fsigpu_gmres_result* res);
int fsigpu_gmres_solve_dev(fsigpu_gmres s, const double* d_b, double* d_x, int max_iters,
                           double rel_tol, double abs_tol, double* history,
                           fsigpu_gmres_result* res);
/* graph capture of the Arnoldi step on/off (default on; multi-kernel path) */
int fsigpu_gmres_set_graphs(fsigpu_gmres s, int enable);
void fsigpu_gmres_destroy(fsigpu_gmres s);

/* ---- instrumentation: accumulated device time per kernel class, measured
 *      with CUDA events on the library stream around each launch when
 *      enabled (adds no sync; disables graphs while on). ----------------- */
#define FSIGPU_K_BLOCK_SOLVE 0
#define FSIGPU_K_SPMV 1
#define FSIGPU_K_TRANSFER 2
#define FSIGPU_K_COMBINE 3
#define FSIGPU_K_COARSE 4
#define FSIGPU_K_ARNOLDI 5
#define FSIGPU_K_COUNT 6
int fsigpu_profile_enable(int enable);
int fsigpu_profile_read(double* ms, long long* launches, double* bytes);
/* the same sums restricted to one GMG level (-1: launches outside a cycle) */
int fsigpu_profile_read_level(int cls, int level, double* ms, long long* launches, double* bytes);
int fsigpu_profile_reset(void);
/* Device-clock launch stamps: durations of the solve kernels INSIDE the
 * captured restart-cycle graph (last CTA exit minus dependency release, from
 * %globaltimer), where CUDA events cannot bracket a launch. No reference
 * counterpart (bench instrumentation). enable/disable resets the counters and
 * makes solvers re-capture their graphs. sub: kernel of the class at that
 * level (SPMV/BLOCK_SOLVE 0; TRANSFER 0 = restriction, 1 = prolongation +
 * residual; COARSE 0; ARNOLDI at level -1: 0 = (A) SpMV + dots, 1 = (B), 2 = (C)). */
int fsigpu_stamps_enable(int enable);
int fsigpu_stamps_read(int cls, int level, int sub, double* us_total, long long* launches);

#ifdef __cplusplus
}
#endif
#endif
