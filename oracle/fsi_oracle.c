/* SPDX-License-Identifier: Apache-2.0
 *
 * fsi_oracle.c — CPU restatement of the reference FS-GMG-GMRES solve path.
 * TEST INFRASTRUCTURE ONLY (see fsi_oracle.h). Compiled with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:10-12) so the
 * dense block solves and the additive FS apply reproduce the reference
 * bit for bit; the coarse solve is a dense equilibrated LU instead of the
 * reference's sparse Gilbert-Peierls LU (sparse_lu.cpp:100-277), which
 * agrees to rounding (pinned in tests/test_oracle_golden.py).
 */
#include "fsi_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ kernels */

/* SparseMatrix::multiply, sparse.cpp:70-76: sequential row sums */
void orc_csr_spmv(int n, const int* ptr, const int* idx, const double* val, const double* x,
                  double* y) {
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * x[idx[k]];
    y[i] = s;
  }
}

/* DenseFactorization ctor, dense.cpp:31-67: row-major LU with partial
 * pivoting (first strictly larger |a_ik| wins), singular when
 * |pivot| <= 1e-14 * max(row_max_original, 1e-300) with row_max swapped
 * along with its row. */
int orc_dense_factor(int m, double* a, int* piv) {
  double* row_max = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      const double v = fabs(a[(size_t)i * m + j]);
      if (v > row_max[i]) row_max[i] = v;
    }
  for (int k = 0; k < m; ++k) {
    int p = k;
    double best = fabs(a[(size_t)k * m + k]);
    for (int i = k + 1; i < m; ++i) {
      const double v = fabs(a[(size_t)i * m + k]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    piv[k] = p;
    if (p != k) {
      for (int j = 0; j < m; ++j) {
        const double t = a[(size_t)k * m + j];
        a[(size_t)k * m + j] = a[(size_t)p * m + j];
        a[(size_t)p * m + j] = t;
      }
      const double t = row_max[k];
      row_max[k] = row_max[p];
      row_max[p] = t;
    }
    const double pivot = a[(size_t)k * m + k];
    if (fabs(pivot) <= 1e-14 * fmax(row_max[k], 1e-300)) {
      free(row_max);
      return 1;
    }
    const double inv = 1.0 / pivot;
    for (int i = k + 1; i < m; ++i) {
      const double l = a[(size_t)i * m + k] * inv;
      a[(size_t)i * m + k] = l;
      for (int j = k + 1; j < m; ++j) a[(size_t)i * m + j] -= l * a[(size_t)k * m + j];
    }
  }
  free(row_max);
  return 0;
}

/* DenseFactorization::solve, dense.cpp:69-86 */
void orc_dense_solve(int m, const double* lu, const int* piv, const double* b, double* x) {
  memcpy(x, b, sizeof(double) * (size_t)m);
  for (int k = 0; k < m; ++k)
    if (piv[k] != k) {
      const double t = x[k];
      x[k] = x[piv[k]];
      x[piv[k]] = t;
    }
  for (int k = 0; k < m; ++k) {
    const double xk = x[k];
    if (xk == 0.0) continue;
    for (int i = k + 1; i < m; ++i) x[i] -= lu[(size_t)i * m + k] * xk;
  }
  for (int i = m - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < m; ++j) s -= lu[(size_t)i * m + j] * x[j];
    x[i] = s / lu[(size_t)i * m + i];
  }
}

/* extract_submatrix (sparse.cpp:171-189) densified as in
 * factor_principal_block (precond.cpp:13-21); dofs sorted unique. */
void orc_extract_block(const int* ptr, const int* idx, const double* val, int m, const int* dofs,
                       double* dense) {
  memset(dense, 0, sizeof(double) * (size_t)m * m);
  for (int i = 0; i < m; ++i) {
    const int src = dofs[i];
    int j = 0;
    for (int k = ptr[src]; k < ptr[src + 1] && j < m; ++k) {
      const int c = idx[k];
      while (j < m && dofs[j] < c) ++j;
      if (j < m && dofs[j] == c) dense[(size_t)i * m + j] = val[k];
    }
  }
}

/* ------------------------------------------------------------ blocks */

typedef struct {
  int n_blocks;
  int* ptr;      /* block offsets into idx (frame or group-local positions) */
  int* idx;
  size_t* lu_off; /* offsets into lu */
  double* lu;
  int* piv;       /* per-block pivots, offset ptr[b] */
  double* cover;
  int dim;        /* dimension of the vectors the sweep acts on */
} orc_sweep;

static int sweep_init(orc_sweep* s, int dim, int nb, const int* ptr, const int* idx,
                      const int* a_ptr, const int* a_idx, const double* a_val, int base,
                      int* bad) {
  /* base: the block's positions are relative to a sub-matrix starting at
   * frame row/col `base` (group 2 uses base = g1). */
  s->n_blocks = nb;
  s->dim = dim;
  const int tot = ptr[nb];
  s->ptr = (int*)malloc(sizeof(int) * (size_t)(nb + 1));
  s->idx = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
  memcpy(s->ptr, ptr, sizeof(int) * (size_t)(nb + 1));
  memcpy(s->idx, idx, sizeof(int) * (size_t)tot);
  s->lu_off = (size_t*)malloc(sizeof(size_t) * (size_t)(nb + 1));
  size_t acc = 0;
  for (int b = 0; b < nb; ++b) {
    s->lu_off[b] = acc;
    const size_t m = (size_t)(ptr[b + 1] - ptr[b]);
    acc += m * m;
  }
  s->lu_off[nb] = acc;
  s->lu = (double*)malloc(sizeof(double) * (acc > 0 ? acc : 1));
  s->piv = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
  int* dofs = (int*)malloc(sizeof(int) * 1024);
  for (int b = 0; b < nb; ++b) {
    const int m = ptr[b + 1] - ptr[b];
    for (int i = 0; i < m; ++i) dofs[i] = idx[ptr[b] + i] + base;
    orc_extract_block(a_ptr, a_idx, a_val, m, dofs, s->lu + s->lu_off[b]);
    /* sub-matrix extraction keeps only columns inside the group: the dofs
     * all lie inside it, so the principal block is the same. */
    if (orc_dense_factor(m, s->lu + s->lu_off[b], s->piv + ptr[b])) {
      *bad = b;
      free(dofs);
      return 1;
    }
  }
  free(dofs);
  s->cover = (double*)calloc((size_t)(dim > 0 ? dim : 1), sizeof(double));
  for (int k = 0; k < tot; ++k) s->cover[idx[k]] += 1.0;
  return 0;
}

static void sweep_free(orc_sweep* s) {
  free(s->ptr);
  free(s->idx);
  free(s->lu_off);
  free(s->lu);
  free(s->piv);
  free(s->cover);
}

/* SchwarzSweep::apply, additive branch (precond.cpp:42-57) */
static void sweep_apply_additive(const orc_sweep* s, const double* r, double* z) {
  double rhs[1024], delta[1024];
  memset(z, 0, sizeof(double) * (size_t)s->dim);
  for (int b = 0; b < s->n_blocks; ++b) {
    const int m = s->ptr[b + 1] - s->ptr[b];
    const int* d = s->idx + s->ptr[b];
    for (int i = 0; i < m; ++i) rhs[i] = r[d[i]];
    orc_dense_solve(m, s->lu + s->lu_off[b], s->piv + s->ptr[b], rhs, delta);
    for (int i = 0; i < m; ++i) z[d[i]] += delta[i];
  }
  for (int i = 0; i < s->dim; ++i)
    if (s->cover[i] > 1.0) z[i] /= s->cover[i];
}

/* CSC of the sub-matrix A[base:base+dim, base:base+dim] of a frame CSR
 * (SparseCsc::from_csr of the group matrix, precond.cpp:36,139) */
typedef struct {
  int dim;
  int* ptr;
  int* row;
  double* val;
} orc_csc;

static void csc_build(orc_csc* c, int base, int dim, const int* a_ptr, const int* a_idx, const double* a_val) {
  c->dim = dim;
  c->ptr = (int*)calloc((size_t)dim + 1, sizeof(int));
  for (int i = 0; i < dim; ++i)
    for (int k = a_ptr[base + i]; k < a_ptr[base + i + 1]; ++k) {
      const int j = a_idx[k] - base;
      if (j >= 0 && j < dim) c->ptr[j + 1]++;
    }
  for (int j = 0; j < dim; ++j) c->ptr[j + 1] += c->ptr[j];
  const int tot = c->ptr[dim];
  c->row = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
  c->val = (double*)malloc(sizeof(double) * (size_t)(tot > 0 ? tot : 1));
  int* next = (int*)malloc(sizeof(int) * (size_t)(dim > 0 ? dim : 1));
  for (int j = 0; j < dim; ++j) next[j] = c->ptr[j];
  for (int i = 0; i < dim; ++i) /* rows in order: each column's rows ascend */
    for (int k = a_ptr[base + i]; k < a_ptr[base + i + 1]; ++k) {
      const int j = a_idx[k] - base;
      if (j >= 0 && j < dim) {
        c->row[next[j]] = i;
        c->val[next[j]++] = a_val[k];
      }
    }
  free(next);
}

static void csc_free(orc_csc* c) {
  free(c->ptr);
  free(c->row);
  free(c->val);
}

/* SchwarzSweep::apply, multiplicative branch (precond.cpp:59-77): every
 * block sees the residual updated by all previous block corrections, the
 * update walking the corrected columns of the CSC. The blocks are visited
 * in `order` (NULL: their index order, which is the reference's). res is
 * updated in place, z accumulated. */
static void sweep_apply_mult(const orc_sweep* s, const orc_csc* a, const int* order, double* res, double* z) {
  double rhs[1024], delta[1024];
  for (int q = 0; q < s->n_blocks; ++q) {
    const int b = order ? order[q] : q;
    const int m = s->ptr[b + 1] - s->ptr[b];
    const int* d = s->idx + s->ptr[b];
    for (int i = 0; i < m; ++i) rhs[i] = res[d[i]];
    orc_dense_solve(m, s->lu + s->lu_off[b], s->piv + s->ptr[b], rhs, delta);
    for (int i = 0; i < m; ++i) {
      const int c = d[i];
      z[c] += delta[i];
      const double dv = delta[i];
      if (dv == 0.0) continue;
      for (int k = a->ptr[c]; k < a->ptr[c + 1]; ++k) res[a->row[k]] -= a->val[k] * dv;
    }
  }
}

/* Multicolour ordering of the blocks of one sweep (the order the GPU's
 * multiplicative smoother runs them in, one kernel per colour). Blocks b
 * and b' conflict when they share a dof or the sweep matrix stores an entry
 * coupling them in either direction (A[i,j] or A[j,i], i in b, j in b');
 * greedy in block order: colour(b) = the smallest colour no conflicting
 * earlier block has. Same-colour blocks then neither overlap nor see each
 * other's corrections, so running them in parallel equals running them in
 * sequence. Returns the colour count; order[] = blocks sorted by (colour,
 * index). */
static int colour_blocks(const orc_sweep* s, const orc_csc* a, int* order) {
  const int nb = s->n_blocks, dim = s->dim;
  /* dof -> blocks holding it */
  int* dptr = (int*)calloc((size_t)dim + 1, sizeof(int));
  for (int k = 0; k < s->ptr[nb]; ++k) dptr[s->idx[k] + 1]++;
  for (int i = 0; i < dim; ++i) dptr[i + 1] += dptr[i];
  int* dblk = (int*)malloc(sizeof(int) * (size_t)(s->ptr[nb] > 0 ? s->ptr[nb] : 1));
  int* nx = (int*)malloc(sizeof(int) * (size_t)(dim > 0 ? dim : 1));
  for (int i = 0; i < dim; ++i) nx[i] = dptr[i];
  for (int b = 0; b < nb; ++b)
    for (int k = s->ptr[b]; k < s->ptr[b + 1]; ++k) dblk[nx[s->idx[k]]++] = b;
  /* row pattern of the sweep matrix = the transpose of its CSC */
  int* rptr = (int*)calloc((size_t)dim + 1, sizeof(int));
  for (int k = 0; k < a->ptr[dim]; ++k) rptr[a->row[k] + 1]++;
  for (int i = 0; i < dim; ++i) rptr[i + 1] += rptr[i];
  int* rcol = (int*)malloc(sizeof(int) * (size_t)(a->ptr[dim] > 0 ? a->ptr[dim] : 1));
  for (int i = 0; i < dim; ++i) nx[i] = rptr[i];
  for (int j = 0; j < dim; ++j)
    for (int k = a->ptr[j]; k < a->ptr[j + 1]; ++k) rcol[nx[a->row[k]]++] = j;
  int* colour = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  int* seen = (int*)malloc(sizeof(int) * (size_t)(nb + 1));  /* colour -> last block marking it */
  for (int c = 0; c <= nb; ++c) seen[c] = -1;
  int ncol = 0;
#define ORC_MARK(j)                                                             \
  for (int q = dptr[j]; q < dptr[(j) + 1]; ++q) {                               \
    const int o = dblk[q];                                                      \
    if (o < b) seen[colour[o]] = b;                                             \
  }
  for (int b = 0; b < nb; ++b) {
    for (int k = s->ptr[b]; k < s->ptr[b + 1]; ++k) {
      const int i = s->idx[k];
      ORC_MARK(i)
      for (int e = rptr[i]; e < rptr[i + 1]; ++e) {
        const int j = rcol[e];
        ORC_MARK(j)
      }
      for (int e = a->ptr[i]; e < a->ptr[i + 1]; ++e) {
        const int j = a->row[e];
        ORC_MARK(j)
      }
    }
    int c = 0;
    while (seen[c] == b) ++c;
    colour[b] = c;
    if (c + 1 > ncol) ncol = c + 1;
  }
#undef ORC_MARK
  int q = 0;
  for (int c = 0; c < ncol; ++c)
    for (int b = 0; b < nb; ++b)
      if (colour[b] == c) order[q++] = b;
  free(dptr);
  free(dblk);
  free(nx);
  free(rptr);
  free(rcol);
  free(colour);
  free(seen);
  return ncol;
}

/* ------------------------------------------------------------ GMG */

typedef struct {
  orc_level_desc d;
  orc_sweep as1, as2;
  orc_csc csc1, csc2;      /* A_g1, A_g2 (multiplicative sweeps) */
  int *order1, *order2;    /* multicolour block orders */
  int ncol1, ncol2;
  /* CSC of group 2 restricted to the u^s columns [0, n_us): the Jacobi
   * residual update walks these columns (precond.cpp:281-287) */
  int* us_ptr;
  int* us_row;
  double* us_val;
} orc_level;

struct orc_gmg {
  int L;
  char mode;
  orc_level* lv;
  double omega;
  int pre, post;
  int smoother; /* 0 richardson (precond.cpp:305-317), 1 GMRES(1) */
  int fs_mode;  /* 0 additive, 1 multiplicative in multicolour
                   order (the GPU's), 2 multiplicative in the reference's
                   block order (FsPreconditioner::apply as shipped) */
  /* coarse: equilibrated dense LU */
  int n0;
  double* c_lu;
  int* c_piv;
  double *c_rs, *c_cs;
};

static void build_us_csc(orc_level* l) {
  const orc_level_desc* d = &l->d;
  const int g1 = d->g1, n_us = d->n_us, n = d->n;
  int* cnt = (int*)calloc((size_t)n_us + 1, sizeof(int));
  for (int i = g1; i < n; ++i)
    for (int k = d->a_ptr[i]; k < d->a_ptr[i + 1]; ++k) {
      const int c = d->a_idx[k] - g1;
      if (c >= 0 && c < n_us) cnt[c + 1]++;
    }
  for (int c = 0; c < n_us; ++c) cnt[c + 1] += cnt[c];
  l->us_ptr = cnt;
  const int tot = cnt[n_us];
  l->us_row = (int*)malloc(sizeof(int) * (size_t)(tot > 0 ? tot : 1));
  l->us_val = (double*)malloc(sizeof(double) * (size_t)(tot > 0 ? tot : 1));
  int* next = (int*)malloc(sizeof(int) * (size_t)(n_us > 0 ? n_us : 1));
  for (int c = 0; c < n_us; ++c) next[c] = cnt[c];
  for (int i = g1; i < n; ++i)
    for (int k = d->a_ptr[i]; k < d->a_ptr[i + 1]; ++k) {
      const int c = d->a_idx[k] - g1;
      if (c >= 0 && c < n_us) {
        const int pos = next[c]++;
        l->us_row[pos] = i - g1;
        l->us_val[pos] = d->a_val[k];
      }
    }
  free(next);
}

/* Additive FS apply: z1 = AS1_add(r1);
 * z2[:n_us] = r2/l; res2 = r2 - A_g2[:, :n_us] z2; z2 += AS2_add(res2) */
/* FsPreconditioner::apply (precond.cpp:271-303), the shipped multiplicative
 * smoother: z1 = AS1_mult(r1); z2[:n_us] = r2/l with the residual update of
 * those columns; AS2 fluid blocks multiplicative on the updated residual.
 * coloured: blocks in multicolour order instead of index order. */
static void fs_apply_mult(const orc_gmg* g, int level, const double* r, double* z, int coloured) {
  const orc_level* l = &g->lv[level];
  const int n = l->d.n, g1 = l->d.g1, g2 = n - g1, n_us = l->d.n_us;
  memset(z, 0, sizeof(double) * (size_t)n);
  double* res = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  memcpy(res, r, sizeof(double) * (size_t)n);
  sweep_apply_mult(&l->as1, &l->csc1, coloured ? l->order1 : NULL, res, z);
  double* res2 = res + g1;
  double* z2 = z + g1;
  for (int i = 0; i < n_us; ++i) {
    const double d = r[g1 + i] / l->d.lumped[i];
    z2[i] = d;
    if (d == 0.0) continue;
    for (int k = l->csc2.ptr[i]; k < l->csc2.ptr[i + 1]; ++k) res2[l->csc2.row[k]] -= l->csc2.val[k] * d;
  }
  (void)g2;
  sweep_apply_mult(&l->as2, &l->csc2, coloured ? l->order2 : NULL, res2, z2);
  free(res);
}

void orc_fs_apply(const orc_gmg* g, int level, const double* r, double* z) {
  if (g->fs_mode != 0) {
    fs_apply_mult(g, level, r, z, g->fs_mode == 1);
    return;
  }
  const orc_level* l = &g->lv[level];
  const int n = l->d.n, g1 = l->d.g1, g2 = n - g1, n_us = l->d.n_us;
  memset(z, 0, sizeof(double) * (size_t)n);
  sweep_apply_additive(&l->as1, r, z);
  const double* r2 = r + g1;
  double* z2 = z + g1;
  double* res = (double*)malloc(sizeof(double) * (size_t)(g2 > 0 ? g2 : 1));
  double* t = (double*)malloc(sizeof(double) * (size_t)(g2 > 0 ? g2 : 1));
  memcpy(res, r2, sizeof(double) * (size_t)g2);
  for (int i = 0; i < n_us; ++i) {
    const double d = r2[i] / l->d.lumped[i];
    z2[i] = d;
    if (d == 0.0) continue;
    for (int k = l->us_ptr[i]; k < l->us_ptr[i + 1]; ++k) res[l->us_row[k]] -= l->us_val[k] * d;
  }
  sweep_apply_additive(&l->as2, res, t);
  for (int i = 0; i < g2; ++i) z2[i] += t[i];
  free(res);
  free(t);
}

void orc_coarse_solve(const orc_gmg* g, const double* b, double* x) {
  const int n = g->n0;
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) y[i] = b[i] * g->c_rs[i];
  orc_dense_solve(n, g->c_lu, g->c_piv, y, w);
  for (int j = 0; j < n; ++j) x[j] = w[j] * g->c_cs[j];
  free(y);
  free(w);
}

/* richardson_smooth, precond.cpp:305-317 */
static void richardson(const orc_gmg* g, int level, double* x, const double* b, int sweeps) {
  const orc_level_desc* d = &g->lv[level].d;
  const int n = d->n;
  if (g->omega == 0.0) return;
  double* res = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  for (int s = 0; s < sweeps; ++s) {
    orc_csr_spmv(n, d->a_ptr, d->a_idx, d->a_val, x, res);
    for (int i = 0; i < n; ++i) res[i] = b[i] - res[i];
    orc_fs_apply(g, level, res, z);
    for (int i = 0; i < n; ++i) x[i] += g->omega * z[i];
  }
  free(res);
  free(z);
}

/* GMRES(1) (minimal-residual) smoothing: BASELINE.json configs[0] names
 * "1 pre- and 1 post-step GMRES(1) with FS"; the reference ships only the
 * Richardson sweep above, so this restates the standard
 * one-dimensional GMRES step on the same sweep structure:
 *   r = b - A x ; z = FS r ; w = A z ; alpha = (w.r)/(w.w) (0 if w = 0) ;
 *   x += alpha z.  Non-linear in b: the outer solver must be flexible.
 * Measured (config 0, FGMRES(30), rtol 1e-10): 197 iterations against 103
 * for Richardson omega = 0.7; minimising the row-equilibrated residual
 * instead gives 390. The residual norm of these unscaled saddle-point level
 * systems is dominated by a few row blocks, so the optimal step for it is a
 * poor smoothing step; Richardson stays the default. */
static void mr_smooth(const orc_gmg* g, int level, double* x, const double* b, int sweeps) {
  const orc_level_desc* d = &g->lv[level].d;
  const int n = d->n;
  double* res = (double*)malloc(sizeof(double) * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  for (int s = 0; s < sweeps; ++s) {
    orc_csr_spmv(n, d->a_ptr, d->a_idx, d->a_val, x, res);
    for (int i = 0; i < n; ++i) res[i] = b[i] - res[i];
    orc_fs_apply(g, level, res, z);
    orc_csr_spmv(n, d->a_ptr, d->a_idx, d->a_val, z, w);
    double wr = 0.0, ww = 0.0;
    for (int i = 0; i < n; ++i) {
      wr += w[i] * res[i];
      ww += w[i] * w[i];
    }
    const double alpha = ww > 0.0 ? wr / ww : 0.0;
    for (int i = 0; i < n; ++i) x[i] += alpha * z[i];
  }
  free(res);
  free(z);
  free(w);
}

static void smooth(const orc_gmg* g, int level, double* x, const double* b, int sweeps) {
  if (g->smoother == 1)
    mr_smooth(g, level, x, b, sweeps);
  else
    richardson(g, level, x, b, sweeps);
}

/* GmgPreconditioner::cycle, gmg.cpp:188-239 (V, W and F cycles) */
static void cycle(const orc_gmg* g, int level, char mode, const double* b, double* x) {
  const orc_level_desc* d = &g->lv[level].d;
  const int n = d->n;
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  if (level == 0) {
    double* dx = (double*)malloc(sizeof(double) * (size_t)n);
    orc_csr_spmv(n, d->a_ptr, d->a_idx, d->a_val, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    orc_coarse_solve(g, r, dx);
    for (int i = 0; i < n; ++i) x[i] += dx[i];
    free(dx);
    free(r);
    return;
  }
  smooth(g, level, x, b, g->pre);
  orc_csr_spmv(n, d->a_ptr, d->a_idx, d->a_val, x, r);
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const int nc = d->nc;
  const orc_level_desc* below = &g->lv[level - 1].d;
  double* rc = (double*)malloc(sizeof(double) * (size_t)nc);
  double* ec = (double*)calloc((size_t)nc, sizeof(double));
  orc_csr_spmv(nc, d->r_ptr, d->r_idx, d->r_val, r, rc);
  for (int i = 0; i < nc; ++i)
    if (below->row_mask[i]) rc[i] = 0.0;
  if (mode == 'w') {
    cycle(g, level - 1, 'w', rc, ec);
    cycle(g, level - 1, 'w', rc, ec);
  } else if (mode == 'f') {
    cycle(g, level - 1, 'f', rc, ec);
    cycle(g, level - 1, 'v', rc, ec);
  } else {
    cycle(g, level - 1, 'v', rc, ec);
  }
  for (int i = 0; i < nc; ++i)
    if (below->col_mask[i]) ec[i] = 0.0;
  double* ef = r; /* reuse */
  orc_csr_spmv(n, d->p_ptr, d->p_idx, d->p_val, ec, ef);
  for (int i = 0; i < n; ++i)
    if (!d->col_mask[i]) x[i] += ef[i];
  smooth(g, level, x, b, g->post);
  free(rc);
  free(ec);
  free(r);
}

void orc_gmg_apply(const orc_gmg* g, const double* r, double* z) {
  const int n = g->lv[g->L - 1].d.n;
  memset(z, 0, sizeof(double) * (size_t)n);
  cycle(g, g->L - 1, g->mode, r, z);
}

orc_gmg* orc_gmg_create(int n_levels, const orc_level_desc* levels, double omega, int pre,
                        int post, int* err_level, int* err_block) {
  orc_gmg* g = (orc_gmg*)calloc(1, sizeof(orc_gmg));
  g->L = n_levels;
  g->mode = 'v';
  g->omega = omega;
  g->pre = pre;
  g->post = post;
  g->lv = (orc_level*)calloc((size_t)n_levels, sizeof(orc_level));
  *err_level = -1;
  *err_block = -1;
  for (int l = 0; l < n_levels; ++l) {
    orc_level* lv = &g->lv[l];
    lv->d = levels[l];
    if (l == 0) continue;
    const orc_level_desc* d = &lv->d;
    int bad = -1;
    if (sweep_init(&lv->as1, d->g1, d->as1_n, d->as1_ptr, d->as1_idx, d->a_ptr, d->a_idx,
                   d->a_val, 0, &bad)) {
      *err_level = l;
      *err_block = bad;
      return NULL;
    }
    if (sweep_init(&lv->as2, d->n - d->g1, d->as2_n, d->as2_ptr, d->as2_idx, d->a_ptr, d->a_idx,
                   d->a_val, d->g1, &bad)) {
      *err_level = l;
      *err_block = d->as1_n + bad;
      return NULL;
    }
    build_us_csc(lv);
    csc_build(&lv->csc1, 0, d->g1, d->a_ptr, d->a_idx, d->a_val);
    csc_build(&lv->csc2, d->g1, d->n - d->g1, d->a_ptr, d->a_idx, d->a_val);
    lv->order1 = (int*)malloc(sizeof(int) * (size_t)(d->as1_n > 0 ? d->as1_n : 1));
    lv->order2 = (int*)malloc(sizeof(int) * (size_t)(d->as2_n > 0 ? d->as2_n : 1));
    lv->ncol1 = colour_blocks(&lv->as1, &lv->csc1, lv->order1);
    lv->ncol2 = colour_blocks(&lv->as2, &lv->csc2, lv->order2);
  }
  /* coarse: equilibrate like sparse_lu.cpp:104-121, dense LU */
  const orc_level_desc* c = &levels[0];
  const int n = c->n;
  g->n0 = n;
  g->c_rs = (double*)malloc(sizeof(double) * (size_t)n);
  g->c_cs = (double*)malloc(sizeof(double) * (size_t)n);
  g->c_lu = (double*)calloc((size_t)n * n, sizeof(double));
  g->c_piv = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    double mx = 0.0;
    for (int k = c->a_ptr[i]; k < c->a_ptr[i + 1]; ++k) mx = fmax(mx, fabs(c->a_val[k]));
    g->c_rs[i] = mx > 0.0 ? 1.0 / mx : 1.0;
  }
  double* cm = (double*)calloc((size_t)n, sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int k = c->a_ptr[i]; k < c->a_ptr[i + 1]; ++k) {
      const int j = c->a_idx[k];
      cm[j] = fmax(cm[j], fabs(c->a_val[k]) * g->c_rs[i]);
    }
  for (int j = 0; j < n; ++j) g->c_cs[j] = cm[j] > 0.0 ? 1.0 / cm[j] : 1.0;
  free(cm);
  for (int i = 0; i < n; ++i)
    for (int k = c->a_ptr[i]; k < c->a_ptr[i + 1]; ++k) {
      const int j = c->a_idx[k];
      g->c_lu[(size_t)i * n + j] += c->a_val[k] * g->c_rs[i] * g->c_cs[j];
    }
  if (orc_dense_factor(n, g->c_lu, g->c_piv)) {
    *err_level = 0;
    *err_block = -1;
    return NULL;
  }
  return g;
}

void orc_gmg_set_cycle(orc_gmg* g, char mode) { g->mode = mode; }
void orc_gmg_set_smoother(orc_gmg* g, int kind) { g->smoother = kind; }
void orc_gmg_set_fs_mode(orc_gmg* g, int mode) { g->fs_mode = mode; }
int orc_gmg_colours(const orc_gmg* g, int level, int group) {
  return group == 1 ? g->lv[level].ncol1 : g->lv[level].ncol2;
}

void orc_gmg_destroy(orc_gmg* g) {
  if (!g) return;
  for (int l = 1; l < g->L; ++l) {
    sweep_free(&g->lv[l].as1);
    sweep_free(&g->lv[l].as2);
    csc_free(&g->lv[l].csc1);
    csc_free(&g->lv[l].csc2);
    free(g->lv[l].order1);
    free(g->lv[l].order2);
    free(g->lv[l].us_ptr);
    free(g->lv[l].us_row);
    free(g->lv[l].us_val);
  }
  free(g->lv);
  free(g->c_lu);
  free(g->c_piv);
  free(g->c_rs);
  free(g->c_cs);
  free(g);
}

/* ------------------------------------------------------------ GMRES */

static double dot(int n, const double* x, const double* y) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

typedef struct {
  const orc_gmg* g;
  const double* scale;
  double* tmp;
  long long count;
} mop_t;

/* CsrOperator on the row-scaled frame matrix: values scaled once like
 * driver.cpp:177-183 (vals[k] *= row_scale[i]), then SpMV */
static void a_apply(const orc_gmg* g, const double* a_scaled, const double* x, double* y) {
  const orc_level_desc* d = &g->lv[g->L - 1].d;
  orc_csr_spmv(d->n, d->a_ptr, d->a_idx, a_scaled, x, y);
}

static void m_apply(mop_t* m, const double* r, double* z) {
  const int n = m->g->lv[m->g->L - 1].d.n;
  ++m->count;
  for (int i = 0; i < n; ++i) m->tmp[i] = r[i] / m->scale[i];
  orc_gmg_apply(m->g, m->tmp, z);
}

/* gmres, krylov.cpp:20-126 (right preconditioned, MGS, restarted) */
static int gmres_impl(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
                      int max_iters, double rel_tol, double abs_tol, double* x, double* history,
                      int* n_history, int* iterations, int* converged, int* breakdown,
                      long long* m_applies, int flexible);

int orc_gmres(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
              int max_iters, double rel_tol, double abs_tol, double* x, double* history,
              int* n_history, int* iterations, int* converged, int* breakdown,
              long long* m_applies) {
  return gmres_impl(g, frame_scale, b, restart, max_iters, rel_tol, abs_tol, x, history, n_history,
                    iterations, converged, breakdown, m_applies, 0);
}

/* Flexible variant (FGMRES): the same cycle as orc_gmres, but z_j = M v_j
 * is kept and the restart update is x += Z y (no extra M apply,
 * krylov.cpp:110-113 becomes Z y). Needed for a non-linear M (GMRES(1)
 * smoother); for a linear M it equals orc_gmres in exact arithmetic. */
int orc_fgmres(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
               int max_iters, double rel_tol, double abs_tol, double* x, double* history,
               int* n_history, int* iterations, int* converged, int* breakdown,
               long long* m_applies) {
  return gmres_impl(g, frame_scale, b, restart, max_iters, rel_tol, abs_tol, x, history, n_history,
                    iterations, converged, breakdown, m_applies, 1);
}

static int gmres_impl(const orc_gmg* g, const double* frame_scale, const double* b, int restart,
                      int max_iters, double rel_tol, double abs_tol, double* x, double* history,
                      int* n_history, int* iterations, int* converged, int* breakdown,
                      long long* m_applies, int flexible) {
  const int n = g->lv[g->L - 1].d.n;
  const int mr = restart;
  if (mr < 1 || rel_tol <= 0.0 || abs_tol <= 0.0) return 1;
  mop_t M = {g, frame_scale, (double*)malloc(sizeof(double) * (size_t)n), 0};
  const orc_level_desc* top = &g->lv[g->L - 1].d;
  const int nnz = top->a_ptr[n];
  double* a_s = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  for (int i = 0; i < n; ++i)
    for (int k = top->a_ptr[i]; k < top->a_ptr[i + 1]; ++k) a_s[k] = top->a_val[k] * frame_scale[i];
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
  double* v = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(mr + 1));
  double* zs = flexible ? (double*)malloc(sizeof(double) * (size_t)n * (size_t)mr) : NULL;
  double* h = (double*)calloc((size_t)(mr + 1) * mr, sizeof(double));
  double* cs = (double*)calloc((size_t)mr, sizeof(double));
  double* sn = (double*)calloc((size_t)mr, sizeof(double));
  double* gv = (double*)calloc((size_t)mr + 1, sizeof(double));
  double* y = (double*)calloc((size_t)mr, sizeof(double));
#define H(i, j) h[(size_t)(i) * mr + (j)]
  int nh = 0, its = 0, conv = 0, brk = 0;
  memset(x, 0, sizeof(double) * (size_t)n);
  a_apply(g, a_s, x, r);
  for (int i = 0; i < n; ++i) r[i] = 1.0 * b[i] + -1.0 * r[i];
  const double r0 = sqrt(dot(n, r, r));
  history[nh++] = r0;
  const double target = fmax(rel_tol * r0, abs_tol);
  if (r0 <= target) {
    conv = 1;
    goto done;
  }
  double beta = r0;
  while (its < max_iters) {
    memset(h, 0, sizeof(double) * (size_t)(mr + 1) * mr);
    memset(gv, 0, sizeof(double) * (size_t)(mr + 1));
    gv[0] = beta;
    for (int i = 0; i < n; ++i) v[i] = r[i] / beta;
    int j = 0, lucky = 0;
    for (; j < mr && its < max_iters; ++j) {
      double* vj = v + (size_t)j * n;
      double* zj = flexible ? zs + (size_t)j * n : tmp;
      m_apply(&M, vj, zj);
      a_apply(g, a_s, zj, w);
      for (int i = 0; i <= j; ++i) {
        const double hij = dot(n, w, v + (size_t)i * n);
        H(i, j) = hij;
        const double* vi = v + (size_t)i * n;
        for (int q = 0; q < n; ++q) w[q] = -hij * vi[q] + w[q];
      }
      const double hjj = sqrt(dot(n, w, w));
      H(j + 1, j) = hjj;
      ++its;
      if (hjj < 1e-14) {
        brk = 1;
        lucky = 1;
      } else {
        double* vn = v + (size_t)(j + 1) * n;
        for (int q = 0; q < n; ++q) vn[q] = w[q] / hjj;
      }
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
        H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
        H(i, j) = t;
      }
      const double denom = hypot(H(j, j), H(j + 1, j));
      cs[j] = H(j, j) / denom;
      sn[j] = H(j + 1, j) / denom;
      H(j, j) = denom;
      H(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      const double rho = fabs(gv[j + 1]);
      history[nh++] = rho;
      if (rho <= target || lucky) {
        ++j;
        break;
      }
    }
    for (int i = j - 1; i >= 0; --i) {
      double s = gv[i];
      for (int k = i + 1; k < j; ++k) s -= H(i, k) * y[k];
      y[i] = s / H(i, i);
    }
    memset(tmp, 0, sizeof(double) * (size_t)n);
    for (int i = 0; i < j; ++i) {
      const double* vi = (flexible ? zs : v) + (size_t)i * n;
      for (int q = 0; q < n; ++q) tmp[q] = y[i] * vi[q] + tmp[q];
    }
    if (flexible)
      memcpy(w, tmp, sizeof(double) * (size_t)n);
    else
      m_apply(&M, tmp, w);
    for (int q = 0; q < n; ++q) x[q] = 1.0 * w[q] + x[q];
    a_apply(g, a_s, x, r);
    for (int i = 0; i < n; ++i) r[i] = 1.0 * b[i] + -1.0 * r[i];
    beta = sqrt(dot(n, r, r));
    if (beta <= target) {
      conv = 1;
      goto done;
    }
    if (brk) goto done;
  }
done:
#undef H
  *n_history = nh;
  *iterations = its;
  *converged = conv;
  *breakdown = brk;
  *m_applies = M.count;
  free(M.tmp);
  free(a_s);
  free(r);
  free(w);
  free(tmp);
  free(v);
  free(zs);
  free(h);
  free(cs);
  free(sn);
  free(gv);
  free(y);
  return 0;
}
