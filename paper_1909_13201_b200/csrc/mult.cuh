// SPDX-License-Identifier: Apache-2.0
//
// Multiplicative FS smoother (the reference's shipped FsPreconditioner::apply,
// proj/src/precond.cpp:271-303, with SchwarzSweep's multiplicative branch,
// :59-77) in multicolour order.
//
// The reference visits the blocks one after the other; each block solves
// against the residual updated by all previous corrections. Since the
// updates are linear, that residual is r - A_g z with z the corrections so
// far (A_g: the group matrix, group 1 = [d^s, d^f, p^s], group 2 =
// [u^s, u^f, p^f], no coupling between the groups). The blocks are coloured
// so that two blocks of one colour share no dof and the group matrix couples
// them in neither direction (host side, fsigpu.cu colour_blocks); then all
// blocks of a colour can run at once and the result equals the sequential
// sweep over the blocks sorted by colour. One kernel per colour:
//   rhs_i = r[p_i] - (A_g z)[p_i]        (8 lanes per block row)
//   delta  = inv(A_b) rhs                 (explicit inverse, column-major)
//   z[p_i] += delta_i ; x[p_i] += omega delta_i (Richardson update fused)
// The u^s rows of group 2 take the lumped Jacobi step first
// (z = r / lumped, precond.cpp:281-287), in mult_init_kernel.
// CPU restatement: oracle/fsi_oracle.c fs_apply_mult / colour_blocks.
#pragma once

#include "common.cuh"
#include "dense.cuh"

namespace fsigpu {

struct MultArgs {
  const int* col_blocks;  // block ids sorted by (colour, id)
  const int* m;           // block sizes
  const long long* row_off;
  const int* pos;          // block-local row -> frame position
  const double* inv;       // column-major inverses, ld = even_up(m)
  const long long* inv_off;
  const int* ag_ptr;       // group-restricted level matrix (CSR)
  const int* ag_idx;
  const double* ag_val;
  const double* r;         // residual the sweep smooths (b - A x)
  double* z;               // FS(r), accumulated colour by colour
  double* x;               // optional: x += omega * delta
  double omega;
};

constexpr int kMultThreads = 256;

// z = 0 except the u^s rows: z = r / lumped; x = (x_zero ? 0 : x) + omega z
__global__ void mult_init_kernel(int n, int g1, int n_us, const double* __restrict__ r,
                                 const double* __restrict__ lumped, double* __restrict__ z, double* x,
                                 double omega, int x_zero) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool us = i >= g1 && i < g1 + n_us;
    const double zi = us ? r[i] / lumped[i - g1] : 0.0;
    z[i] = zi;
    if (x) {
      double xv = x_zero ? 0.0 : x[i];
      if (us) xv += omega * zi;
      x[i] = xv;
    }
  }
}

// one colour: grid = the colour's block count, blocks col_blocks[first ..]
__global__ void __launch_bounds__(kMultThreads) mult_colour_kernel(MultArgs a, int first) {
  __shared__ double rhs[kLargeMax];
  pdl_trigger();
  pdl_wait();
  const int b = a.col_blocks[first + blockIdx.x];
  const int m = a.m[b];
  const long long ro = a.row_off[b];
  const int t = threadIdx.x;
  constexpr int LPR = 8, U = 8;
  const int lane = t & (LPR - 1);
  for (int i0 = 0; i0 < m; i0 += kMultThreads / LPR) {
    const int i = i0 + t / LPR;
    const bool ok = i < m;
    const int p = ok ? __ldg(a.pos + ro + i) : 0;
    const int k0 = ok ? __ldg(a.ag_ptr + p) : 0, k1 = ok ? __ldg(a.ag_ptr + p + 1) : 0;
    double s = 0.0;
    for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
      int c[U];
      double v[U], zv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + u * LPR;
        c[u] = k < k1 ? __ldg(a.ag_idx + k) : -1;
        v[u] = k < k1 ? __ldg(a.ag_val + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) zv[u] = c[u] >= 0 ? __ldcg(a.z + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) s = fma(v[u], zv[u], s);
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
    if (ok && lane == 0) rhs[i] = __ldg(a.r + p) - s;
  }
  __syncthreads();  // every read of z by this block precedes its writes
  const int ld = even_up(m);
  const double* __restrict__ M = a.inv + a.inv_off[b];
  for (int i = t; i < m; i += kMultThreads) {
    double s = 0.0;
    for (int j0 = 0; j0 < m; j0 += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = j0 + u < m ? __ldg(M + (size_t)(j0 + u) * ld + i) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < m) s = fma(v[u], rhs[j0 + u], s);
    }
    const int p = __ldg(a.pos + ro + i);
    a.z[p] += s;
    if (a.x) a.x[p] += a.omega * s;
  }
}

}  // namespace fsigpu
