/* SPDX-License-Identifier: Apache-2.0
 *
 * fsi_oracle — plain-C CPU restatement of the reference solve path.
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER. The product path
 * (paper_1909_13201_b200 / libfsigpu.so) never links or calls it.
 *
 * Pinned against outputs of the unmodified reference (oracle/_ref, exported
 * to FSIX archives by oracle/ref_harness/harness.cpp) and the reference's own
 * known-answer tests (tests/test_oracle_golden.py).
 */
#ifndef FSI_ORACLE_H
#define FSI_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as fsigpu_level_desc in include/fsigpu.h. */
typedef struct {
  int n;
  const int* a_ptr;
  const int* a_idx;
  const double* a_val;
  const unsigned char* row_mask; /* constrained rows (frame)  */
  const unsigned char* col_mask; /* constrained cols (frame)  */
  int nc;                        /* coarser level size (l > 0) */
  const int* p_ptr;
  const int* p_idx;
  const double* p_val; /* n x nc  */
  const int* r_ptr;
  const int* r_idx;
  const double* r_val; /* nc x n  */
  int g1, n_us;
  const double* lumped; /* n_us */
  int as1_n;
  const int* as1_ptr;
  const int* as1_idx; /* frame positions in [0, g1) */
  int as2_n;
  const int* as2_ptr;
  const int* as2_idx; /* group-2 local positions */
} orc_level_desc;

typedef struct orc_gmg orc_gmg;

/* sparse.cpp:70-76 */
void orc_csr_spmv(int n, const int* ptr, const int* idx, const double* val, const double* x,
                  double* y);
/* dense.cpp:31-67; a row-major m*m, overwritten by LU; returns 0 or 1 (singular) */
int orc_dense_factor(int m, double* a, int* piv);
/* dense.cpp:69-86 */
void orc_dense_solve(int m, const double* lu, const int* piv, const double* b, double* x);
/* sparse.cpp:171-189 + precond.cpp:13-21: dense principal block (row-major) */
void orc_extract_block(const int* ptr, const int* idx, const double* val, int m, const int* dofs,
                       double* dense);

/* GmgPreconditioner ctor (gmg.cpp:178-184) with additive FS smoothers.
 * Returns NULL on a singular block; *err_level/*err_block name it. */
orc_gmg* orc_gmg_create(int n_levels, const orc_level_desc* levels, double omega, int pre,
                        int post, int* err_level, int* err_block);
void orc_gmg_destroy(orc_gmg* g);
/* 'v' (default), 'w' or 'f' (gmg.cpp:215-229) */
void orc_gmg_set_cycle(orc_gmg* g, char mode);
/* level smoother: 0 damped Richardson (precond.cpp:305-317, default),
 * 1 GMRES(1) minimal-residual step (BASELINE configs[0]) */
void orc_gmg_set_smoother(orc_gmg* g, int kind);
/* FS variant: 0 additive (default), 1 multiplicative in the
 * multicolour block order the GPU runs, 2 multiplicative in the
 * reference's block order (FsPreconditioner::apply, precond.cpp:271-303) */
void orc_gmg_set_fs_mode(orc_gmg* g, int mode);
/* colours of the AS1 (group 1) or AS2 (group 2) blocks of a level */
int orc_gmg_colours(const orc_gmg* g, int level, int group);
/* FS apply on level l >= 1 in the current variant */
void orc_fs_apply(const orc_gmg* g, int level, const double* r, double* z);
/* one V-cycle from a zero guess (gmg.cpp:188-246) */
void orc_gmg_apply(const orc_gmg* g, const double* r, double* z);
/* coarse direct solve */
void orc_coarse_solve(const orc_gmg* g, const double* b, double* x);

/* Reference GMRES (krylov.cpp:20-126) on the row-scaled frame operator
 * A_s = diag(frame_scale) A_top with M(r) = GMG(r / frame_scale)
 * (driver.cpp:259-272). history must hold max_iters + 2 doubles. */
int orc_gmres(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
              int max_iters, double rel_tol, double abs_tol, double* x, double* history,
              int* n_history, int* iterations, int* converged, int* breakdown,
              long long* m_applies);

/* Flexible GMRES on the same operators (keeps Z = M V; x += Z y at restart) */
int orc_fgmres(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
               int max_iters, double rel_tol, double abs_tol, double* x, double* history,
               int* n_history, int* iterations, int* converged, int* breakdown,
               long long* m_applies);

#ifdef __cplusplus
}
#endif
#endif
