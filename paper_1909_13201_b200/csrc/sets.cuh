// SPDX-License-Identifier: Apache-2.0
//
// Device-side construction of the Schwarz block sets (setup, once per
// hierarchy level), from the mesh-side index maps:
//   * FsPreconditioner's field-split sets (proj/src/precond.cpp:119-269):
//     AS1 solid [d^s, p^s] patches, AS1 fluid d^f patches grown by
//     `overlap_layers` rings of fluid elements sharing a Q2 node, AS2 fluid
//     [u^f, p^f] patches (group-2 local positions); constrained positions
//     dropped (constrained_positions, :90-97) and, in group 1, positions whose
//     A_g1 row is empty (:144-156);
//   * the Vanka sets of the pure-DD smoother (build_vanka_blocks,
//     ordering.cpp:77-115, mapped and filtered as AsPreconditioner does,
//     precond.cpp:99-117).
// One CTA per patch: gather the patch's element list (and its overlap
// rings), collect the dof positions in shared memory, bitonic-sort them and
// drop duplicates (make_index_set, sparse.cpp:27-31). Pass 0 counts, the
// host scans the counts, pass 1 writes. The lumped u^s mass (precond.cpp:
// 231-245) is one thread per row with the reference's sequential sum.
#pragma once

#include <climits>

#include "common.cuh"

namespace fsigpu {

enum SetKind { kSetSolidDp = 0, kSetFluidD = 1, kSetFluidUp = 2, kSetVankaSolid = 3, kSetVankaFluid = 4 };

constexpr int kSetThreads = 256;
constexpr int kSetCap = 4096;      // dof positions (with duplicates) per patch
constexpr int kSetElemCap = 1024;  // elements per patch incl. overlap rings

struct SetArgs {
  int kind, epb, overlap, n_list, npe, dim, ppe, g1;
  const int* list;  // the patch chunks' element list (solid or fluid elements, ascending)
  const int* en;    // element -> Q2 nodes (n_elements x npe)
  const unsigned char* elem_solid;
  const unsigned char* node_solid;
  const int* ne_ptr;  // Q2 node -> elements (CSR)
  const int* ne_idx;
  const int* d_pos;  // frame positions (n_nodes x dim, n_elements x ppe)
  const int* u_pos;
  const int* p_pos;
  const unsigned char* drop;      // constrained frame positions (may be null)
  const unsigned char* g1_empty;  // group-1 rows of A_g1 without a nonzero value
  int* count;                     // pass 0: dofs per patch
  const long long* off;           // pass 1: output offsets
  int* out;
  int* overflow;
};

// ascending bitonic sort of a[0..n2) (n2 a power of two), all threads
__device__ __forceinline__ void set_bitonic(int* a, int n2) {
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int ij = i ^ j;
        if (ij > i) {
          const bool up = (i & k) == 0;
          const int x = a[i], y = a[ij];
          if ((x > y) == up) {
            a[i] = y;
            a[ij] = x;
          }
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(kSetThreads) set_patch_kernel(SetArgs a, int pass) {
  __shared__ int E[kSetElemCap];
  __shared__ int D[kSetCap];
  __shared__ int s_ne, s_nd, s_f0, s_uniq;
  const int t = threadIdx.x;
  const int patch = blockIdx.x;
  const int start = patch * a.epb;
  const int stop = min(start + a.epb, a.n_list);
  if (t == 0) {
    s_ne = stop - start;
    s_f0 = 0;
    s_nd = 0;
  }
  __syncthreads();
  for (int k = t; k < stop - start; k += blockDim.x) E[k] = a.list[start + k];
  __syncthreads();
  // overlap rings (precond.cpp:189-206): fluid elements sharing a Q2 node
  // with the current frontier; the set, not its order, decides the dofs
  const int layers = a.kind == kSetFluidD ? a.overlap : 0;
  for (int layer = 0; layer < layers; ++layer) {
    const int f0 = s_f0, f1 = s_ne;
    for (int q = t; q < (f1 - f0) * a.npe; q += blockDim.x) {
      const int e = E[f0 + q / a.npe];
      const int node = a.en[(size_t)e * a.npe + q % a.npe];
      for (int k = a.ne_ptr[node]; k < a.ne_ptr[node + 1]; ++k) {
        const int nb = a.ne_idx[k];
        if (a.elem_solid[nb]) continue;
        const int slot = atomicAdd(&s_nd, 1);
        if (slot < kSetCap) D[slot] = nb;
      }
    }
    __syncthreads();
    const int nc = s_nd;
    if (nc > kSetCap) {
      if (t == 0) atomicExch(a.overflow, 1);
      return;
    }
    int n2 = 1;
    while (n2 < nc) n2 <<= 1;
    for (int k = nc + t; k < n2; k += blockDim.x) D[k] = INT_MAX;
    __syncthreads();
    set_bitonic(D, n2);
    if (t == 0) {
      int ne = f1;
      for (int k = 0; k < nc; ++k) {
        const int c = D[k];
        if (k > 0 && c == D[k - 1]) continue;
        bool in = false;
        for (int q = 0; q < ne && !in; ++q) in = E[q] == c;
        if (!in) {
          if (ne >= kSetElemCap) {
            atomicExch(a.overflow, 1);
            break;
          }
          E[ne++] = c;
        }
      }
      s_f0 = f1;
      s_ne = ne;
      s_nd = 0;
    }
    __syncthreads();
  }
  // the patch's dof positions
  const int ne = s_ne;
  const bool vanka = a.kind == kSetVankaSolid || a.kind == kSetVankaFluid;
  const bool want_solid = a.kind == kSetSolidDp || a.kind == kSetVankaSolid;
  auto push = [&](int p) {
    const int slot = atomicAdd(&s_nd, 1);
    if (slot < kSetCap) D[slot] = p;
  };
  for (int q = t; q < ne * a.ppe; q += blockDim.x) {
    if (a.kind == kSetFluidD) break;
    const int e = E[q / a.ppe];
    const int p = a.p_pos[(size_t)e * a.ppe + q % a.ppe];
    if (vanka && a.drop && a.drop[p]) continue;  // AsPreconditioner drops every constrained position
    push(a.kind == kSetFluidUp ? p - a.g1 : p);
  }
  for (int q = t; q < ne * a.npe; q += blockDim.x) {
    const int node = a.en[(size_t)E[q / a.npe] * a.npe + q % a.npe];
    if ((bool)a.node_solid[node] != want_solid) continue;
    for (int i = 0; i < a.dim; ++i) {
      if (a.kind != kSetFluidUp) {  // d
        const int p = a.d_pos[(size_t)node * a.dim + i];
        if (!(a.drop && a.drop[p])) push(p);
      }
      if (a.kind == kSetFluidUp || vanka) {  // u
        const int p = a.u_pos[(size_t)node * a.dim + i];
        if (!(a.drop && a.drop[p])) push(a.kind == kSetFluidUp ? p - a.g1 : p);
      }
    }
  }
  __syncthreads();
  const int nd = s_nd;
  if (nd > kSetCap) {
    if (t == 0) atomicExch(a.overflow, 1);
    return;
  }
  int n2 = 1;
  while (n2 < nd) n2 <<= 1;
  for (int k = nd + t; k < n2; k += blockDim.x) D[k] = INT_MAX;
  __syncthreads();
  set_bitonic(D, n2);
  // unique (+ the group-1 empty-row filter of the AS1 sets), in order
  if (t == 0) {
    const bool drop_empty = a.kind == kSetSolidDp || a.kind == kSetFluidD;
    int u = 0;
    for (int k = 0; k < nd; ++k) {
      const int p = D[k];
      if (k > 0 && p == D[k - 1]) continue;
      if (drop_empty && a.g1_empty[p]) continue;
      D[u++] = p;
    }
    s_uniq = u;
  }
  __syncthreads();
  const int u = s_uniq;
  if (pass == 0) {
    if (t == 0) a.count[patch] = u;
  } else {
    int* o = a.out + a.off[patch];
    for (int k = t; k < u; k += blockDim.x) o[k] = D[k];
  }
}

// rows i < g1 of A_g1 = A[0:g1, 0:g1] holding no nonzero value (precond.cpp:144-152)
__global__ void g1_empty_kernel(int g1, const int* __restrict__ ptr, const int* __restrict__ idx,
                                const double* __restrict__ val, unsigned char* __restrict__ empty) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g1) return;
  unsigned char e = 1;
  for (int k = ptr[i]; k < ptr[i + 1] && e; ++k)
    if (idx[k] < g1 && val[k] != 0.0) e = 0;
  empty[i] = e;
}

// lumped u^s mass: row sums of A_g2[0:n_us, :] in column order; an all-zero
// row (a constrained one) -> 1; a non-positive sum -> singular (reported as
// the lowest such row)  (precond.cpp:231-245)
__global__ void lumped_kernel(int g1, int n_us, const int* __restrict__ ptr, const int* __restrict__ idx,
                              const double* __restrict__ val, double* __restrict__ lumped, int* bad_row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_us) return;
  const int row = g1 + i;
  double s = 0.0, amax = 0.0;
  for (int k = ptr[row]; k < ptr[row + 1]; ++k) {
    if (idx[k] < g1) continue;
    s += val[k];
    amax = fmax(amax, fabs(val[k]));
  }
  if (amax == 0.0) {
    lumped[i] = 1.0;
  } else if (s <= 0.0) {
    lumped[i] = s;
    atomicMin(bad_row, i);
  } else {
    lumped[i] = s;
  }
}

}  // namespace fsigpu
