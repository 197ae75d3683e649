// SPDX-License-Identifier: Apache-2.0
//
// Batched dense fp64 block kernels: extraction of principal blocks from the
// level CSR matrix, LU with partial pivoting, and the forward/back
// substitutions of the Schwarz block solves.
//
// Reference semantics (proj/src/dense.cpp:31-86):
//   * pivot = first row with strictly larger |a_ik| (ties -> lowest row),
//   * singular when |pivot| <= 1e-14 * max(row_max_original, 1e-300) with
//     row_max swapped along with its row,
//   * l = a_ik * (1/pivot), a_ij -= l * a_kj, non-fused (-ffp-contract=off),
//   * solve: all row swaps first, unit-lower forward, upper back
//     substitution.
// The factorization and the forward sweep here apply exactly the same
// rounded operations in the same order per entry, so LU factors are
// bit-identical to DenseFactorization; the back substitution is tiled
// (order of the subtractions differs) and agrees to rounding.
//
// Layout in HBM: every block's LU is stored column-major (entry (i,j) at
// lu[off + j*m + i]) so the column-oriented sweeps read contiguous 256-B
// rows per warp.  Pivots are folded into one gather map gsrc[s] = source
// position of the pivoted row s.
#pragma once

#include "common.cuh"

namespace fsigpu {

// Work item of the batched solve kernel: either up to 8 small blocks
// (m <= 64, one warp each) or one large block (whole 256-thread CTA).
struct SolveItem {
  int type;   // 0 small, 1 large
  int first;  // first block id
  int count;  // blocks (small items)
  int pad;
};

constexpr int kSolveThreads = 256;
constexpr int kSmallMax = 64;
constexpr int kLargeMax = 1024;

struct SolveArgs {
  const int* m;
  const long long* lu_off;
  const long long* row_off;
  const double* lu;
  const int* gsrc;
  const SolveItem* items;
  // right-hand side source: x[s] = rhs(gsrc[s]); for group-2 positions
  // (p >= g1) the lumped-Jacobi update of precond.cpp:281-287 is applied
  // on the fly: rhs = r[p] - sum_k A_g2[p-g1, k] * (r[g1+k] / lumped[k])
  const double* r;
  int g1;
  const double* lumped;
  const int* aus_ptr;
  const int* aus_col;
  const double* aus_val;
  double* out;  // delta[row_off[b] + i], local order
};

__device__ __forceinline__ double gather_rhs(const SolveArgs& a, int p) {
  double v = __ldg(a.r + p);
  if (p >= a.g1) {
    const int q = p - a.g1;
    const int k0 = __ldg(a.aus_ptr + q), k1 = __ldg(a.aus_ptr + q + 1);
    for (int k = k0; k < k1; ++k) {
      const int c = __ldg(a.aus_col + k);
      const double d = __ldg(a.r + a.g1 + c) / __ldg(a.lumped + c);
      v = sub_rn(v, mul_rn(__ldg(a.aus_val + k), d));
    }
  }
  return v;
}

// Team barrier: one warp (NW==1) or the whole CTA.
template <int NW>
__device__ __forceinline__ void team_sync() {
  if constexpr (NW == 1)
    __syncwarp();
  else
    __syncthreads();
}

// Solve one block with a team of NW warps; xs: shared scratch of m doubles.
template <int NW>
__device__ void solve_block(const SolveArgs& a, int b, double* xs, int t) {
  constexpr int T = NW * 32;
  const int m = a.m[b];
  const long long ro = a.row_off[b];
  const double* __restrict__ LU = a.lu + a.lu_off[b];
  for (int s = t; s < m; s += T) xs[s] = gather_rhs(a, __ldg(a.gsrc + ro + s));
  team_sync<NW>();

  // forward: unit lower, column tiles of 32 (bit-identical order)
  for (int k0 = 0; k0 < m; k0 += 32) {
    const int kb = min(32, m - k0);
    if (t < 32) {
      const int lane = t;
      double v = lane < kb ? xs[k0 + lane] : 0.0;
      double Lr[32];
#pragma unroll
      for (int kk = 0; kk < 32; ++kk)
        Lr[kk] = (kk < lane && lane < kb) ? __ldg(LU + (size_t)(k0 + kk) * m + k0 + lane) : 0.0;
#pragma unroll
      for (int kk = 0; kk < 32; ++kk) {
        if (kk < kb) {
          const double xk = __shfl_sync(kFull, v, kk);
          if (lane > kk && lane < kb) v = sub_rn(v, mul_rn(Lr[kk], xk));
        }
      }
      if (lane < kb) xs[k0 + lane] = v;
    }
    team_sync<NW>();
    for (int i = k0 + kb + t; i < m; i += T) {
      double acc = xs[i];
      const double* col = LU + (size_t)k0 * m + i;
#pragma unroll 8
      for (int kk = 0; kk < kb; ++kk) acc = sub_rn(acc, mul_rn(__ldg(col + (size_t)kk * m), xs[k0 + kk]));
      xs[i] = acc;
    }
    team_sync<NW>();
  }

  // backward: upper with diagonal, column tiles from the bottom
  for (int k1 = ((m - 1) / 32) * 32; k1 >= 0; k1 -= 32) {
    const int kb = min(32, m - k1);
    if (t < 32) {
      const int lane = t;
      double v = lane < kb ? xs[k1 + lane] : 0.0;
      const double d = lane < kb ? __ldg(LU + (size_t)(k1 + lane) * m + k1 + lane) : 1.0;
      double Ur[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        Ur[jj] = (jj > lane && jj < kb) ? __ldg(LU + (size_t)(k1 + jj) * m + k1 + lane) : 0.0;
#pragma unroll
      for (int jj = 31; jj >= 0; --jj) {
        if (jj < kb) {
          if (lane == jj) v = v / d;
          const double xj = __shfl_sync(kFull, v, jj);
          if (lane < jj) v = sub_rn(v, mul_rn(Ur[jj], xj));
        }
      }
      if (lane < kb) xs[k1 + lane] = v;
    }
    team_sync<NW>();
    for (int i = t; i < k1; i += T) {
      double acc = xs[i];
      const double* col = LU + (size_t)k1 * m + i;
#pragma unroll 8
      for (int jj = 0; jj < kb; ++jj) acc = sub_rn(acc, mul_rn(__ldg(col + (size_t)jj * m), xs[k1 + jj]));
      xs[i] = acc;
    }
    team_sync<NW>();
  }
  for (int i = t; i < m; i += T) a.out[ro + i] = xs[i];
}

__global__ void __launch_bounds__(kSolveThreads) block_solve_kernel(SolveArgs a) {
  __shared__ double xs[kLargeMax];
  const SolveItem it = a.items[blockIdx.x];
  const int tid = threadIdx.x;
  if (it.type == 0) {
    const int w = tid >> 5;
    if (w < it.count) solve_block<1>(a, it.first + w, xs + w * kSmallMax, tid & 31);
  } else {
    solve_block<kSolveThreads / 32>(a, it.first, xs, tid);
  }
}

// ---------------------------------------------------------------- LU

// Factor one block per CTA. src/dst column-major (may alias). SMEM: the
// block is staged in dynamic shared memory (m <= 164 at 227 KB); otherwise
// it is factored in place in global memory (dst).
template <int NT, bool SMEM>
__global__ void __launch_bounds__(NT)
    lu_factor_kernel(const int* __restrict__ blist, const int* __restrict__ msz,
                     const long long* __restrict__ lu_off, const long long* __restrict__ row_off,
                     const double* __restrict__ src, double* __restrict__ dst,
                     int* __restrict__ piv_out, int* __restrict__ gsrc_out,
                     const int* __restrict__ src_pos, int pos_base, int* __restrict__ fail) {
  // dynamic smem: [A: m*m doubles, SMEM only][rowmax: m doubles][perm: m ints]
  extern __shared__ double smem[];
  constexpr int NW = NT / 32;
  __shared__ int s_p, s_fail;
  __shared__ double s_inv;
  const int b = blist[blockIdx.x];
  const int m = msz[b];
  const long long off = lu_off[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = SMEM ? smem : dst + off;
  double* rowmax = SMEM ? smem + (size_t)m * m : smem;
  int* perm = reinterpret_cast<int*>(rowmax + m);
  if (SMEM) {
    for (long long e = tid; e < (long long)m * m; e += NT) A[e] = src[off + e];
  } else if (src != dst) {
    for (long long e = tid; e < (long long)m * m; e += NT) A[e] = src[off + e];
  }
  __syncthreads();
  for (int i = tid; i < m; i += NT) {
    double mx = 0.0;
    for (int j = 0; j < m; ++j) mx = fmax(mx, fabs(A[(size_t)j * m + i]));
    rowmax[i] = mx;
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  double inv_prev = 0.0;
  for (int k = 0; k < m; ++k) {
    if (warp == 0) {
      if (k > 0)
        for (int i = k + lane; i < m; i += 32) A[(size_t)(k - 1) * m + i] = mul_rn(A[(size_t)(k - 1) * m + i], inv_prev);
      double best = -1.0;
      int bi = m;
      for (int i = k + lane; i < m; i += 32) {
        const double v = fabs(A[(size_t)k * m + i]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      // first strictly-larger in ascending row order == max value, lowest index
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(kFull, best, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (lane == 0) {
        // sequential scan starts with best = |a_kk| (dense.cpp:42-49); a NaN
        // column keeps p = k
        int p = (bi < m) ? bi : k;
        if (!(fabs(A[(size_t)k * m + k]) < best)) p = k;
        const double pivot = A[(size_t)k * m + p];
        if (fabs(pivot) <= 1e-14 * fmax(rowmax[p], 1e-300)) s_fail = 1;
        s_p = p;
        s_inv = 1.0 / pivot;
      }
    }
    __syncthreads();
    if (s_fail) break;
    const int p = s_p;
    if (p != k) {
      for (int j = tid; j < m; j += NT) {
        const double t0 = A[(size_t)j * m + k];
        A[(size_t)j * m + k] = A[(size_t)j * m + p];
        A[(size_t)j * m + p] = t0;
      }
      if (tid == 0) {
        const double t1 = rowmax[k];
        rowmax[k] = rowmax[p];
        rowmax[p] = t1;
      }
    }
    if (tid == 0) perm[k] = p;  // LAPACK-style pivot for now
    __syncthreads();
    const double inv = s_inv;
    inv_prev = inv;
    for (int j = k + 1 + warp; j < m; j += NW) {
      const double akj = A[(size_t)j * m + k];
      for (int i = k + 1 + lane; i < m; i += 32) {
        const double l = mul_rn(A[(size_t)k * m + i], inv);
        A[(size_t)j * m + i] = sub_rn(A[(size_t)j * m + i], mul_rn(l, akj));
      }
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) atomicMin(fail, b);
    return;
  }
  __syncthreads();
  if (tid == 0) {
    const long long ro = row_off[b];
    for (int k = 0; k < m; ++k) piv_out[ro + k] = perm[k];
    // compose the sequential swaps into a gather map
    for (int k = 0; k < m; ++k) rowmax[k] = (double)k;  // reuse as id array
    for (int k = 0; k < m; ++k) {
      const int p = perm[k];
      const double t2 = rowmax[k];
      rowmax[k] = rowmax[p];
      rowmax[p] = t2;
    }
  }
  __syncthreads();
  const long long ro = row_off[b];
  for (int s = tid; s < m; s += NT) {
    const int loc = (int)rowmax[s];
    gsrc_out[ro + s] = src_pos ? src_pos[ro + loc] + pos_base : (int)(ro + loc);
  }
  if (SMEM)
    for (long long e = tid; e < (long long)m * m; e += NT) dst[off + e] = A[e];
}

// Principal block A[dofs, dofs] of a CSR matrix into column-major dense
// storage (dst pre-zeroed). One warp per block row; columns located by
// binary search in the sorted block index list (extract_submatrix,
// sparse.cpp:171-189).
__global__ void extract_blocks_kernel(int nb, const int* __restrict__ msz,
                                      const long long* __restrict__ lu_off,
                                      const long long* __restrict__ row_off,
                                      const int* __restrict__ pos, int base,
                                      const int* __restrict__ aptr, const int* __restrict__ aidx,
                                      const double* __restrict__ aval, double* __restrict__ dst) {
  const int b = blockIdx.x;
  if (b >= nb) return;
  const int m = msz[b];
  const int* d = pos + row_off[b];
  double* D = dst + lu_off[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < m; i += nw) {
    const int row = d[i] + base;
    for (int k = aptr[row] + lane; k < aptr[row + 1]; k += 32) {
      const int c = aidx[k] - base;
      int lo = 0, hi = m - 1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int v = d[mid];
        if (v == c) {
          D[(size_t)mid * m + i] = aval[k];
          break;
        }
        if (v < c) lo = mid + 1;
        else hi = mid - 1;
      }
    }
  }
}

// Counter-hash uniform[-1,1) for the config-1 generator.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ double hash_uniform(unsigned long long seed, long long b, int i, int j) {
  unsigned long long x = seed * 0x2545F4914F6CDD1Dull ^ ((unsigned long long)b * 0x9E3779B97F4A7C15ull) ^
                         ((unsigned long long)(i + 1) << 40) ^ ((unsigned long long)(j + 1) << 20);
  // two rounds of splitmix
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// One thread per block row: a_ij uniform, a_ii += sum_j |a_ij| (config 1).
__global__ void gen_dominant_kernel(long long nb, const int* __restrict__ msz,
                                    const long long* __restrict__ lu_off,
                                    const long long* __restrict__ row_off, long long total_rows,
                                    unsigned long long seed, double* __restrict__ dst,
                                    const long long* __restrict__ row_block) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= total_rows) return;
  const long long b = row_block[r];
  const int m = msz[b];
  const int i = (int)(r - row_off[b]);
  double* D = dst + lu_off[b];
  double s = 0.0, diag = 0.0;
  for (int j = 0; j < m; ++j) {
    const double v = hash_uniform(seed, b, i, j);
    s += fabs(v);
    if (j == i) diag = v;
    else D[(size_t)j * m + i] = v;
  }
  D[(size_t)i * m + i] = diag + s;
}

__global__ void gen_rhs_kernel(long long total_rows, unsigned long long seed, double* __restrict__ out) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= total_rows) return;
  out[r] = hash_uniform(seed ^ 0x5bd1e995ull, r, -1, 7);
}

}  // namespace fsigpu
