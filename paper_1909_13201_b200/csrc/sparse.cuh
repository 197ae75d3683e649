// SPDX-License-Identifier: Apache-2.0
//
// Sparse level kernels: CSR SpMV with fused epilogues (residual, masked
// restriction, masked prolongation-add, row scaling), the FS combine
// (additive Schwarz gather-reduce + cover average + lumped Jacobi +
// Richardson update), the coarse explicit-inverse GEMV and the setup-time
// Gauss-Jordan inverse.
//
// CSR (int32 row offsets / cols, fp64 values; proj/include/fsi/sparse.hpp:32-74)
// is streamed with LPR lanes per row (vector CSR): values and column
// indices through the read-only path, x gathered through L1/L2 (the level
// vectors are <= 10 MB and stay L2-resident). Per-row sums reduce with a
// fixed xor-shuffle tree, so results are deterministic run to run.
#pragma once

#include "common.cuh"

namespace fsigpu {

// Epilogues: functors applied by lane 0 of each row. pre(i) loads the
// row's own operands (b[i], x[i], mask[i]); kernels call it right after the
// PDL wait, BEFORE the row's dot product, so those loads overlap the
// gathers instead of adding one dependent round trip at the end.
struct EpiPre {
  double a;
  unsigned char m;
};
struct EpiPlain {  // y = A x                       (sparse.cpp:70-76)
  double* y;
  __device__ EpiPre pre(int) const { return {0.0, 0}; }
  __device__ void operator()(int i, double s, EpiPre) const { y[i] = s; }
};
struct EpiResid {  // r = b - A x                   (gmg.cpp:205-206, precond.cpp:312-313)
  const double* b;
  double* r;
  __device__ EpiPre pre(int i) const { return {b[i], 0}; }
  __device__ void operator()(int i, double s, EpiPre p) const { r[i] = p.a - s; }
};
struct EpiScaled {  // w = diag(s) A z              (driver.cpp:177-183,261-262)
  const double* scale;
  double* y;
  __device__ EpiPre pre(int i) const { return {scale[i], 0}; }
  __device__ void operator()(int i, double s, EpiPre p) const { y[i] = p.a * s; }
};
struct EpiResidScaled {  // r = b - diag(s) A x     (krylov.cpp:31-32,116-117)
  const double* b;
  const double* scale;
  double* r;
  __device__ EpiPre pre(int i) const { return {b[i], 0}; }
  __device__ void operator()(int i, double s, EpiPre p) const { r[i] = p.a - scale[i] * s; }
};
struct EpiRestrict {  // rc = R r, rc[constrained_rows below] = 0 (gmg.cpp:208-212)
  const unsigned char* mask;
  double* y;
  __device__ EpiPre pre(int i) const { return {0.0, mask[i]}; }
  __device__ void operator()(int i, double s, EpiPre p) const { y[i] = p.m ? 0.0 : s; }
};
struct EpiProlongAdd {  // x += P ec where !constrained_cols (gmg.cpp:233-236)
  const unsigned char* mask;
  double* x;
  __device__ EpiPre pre(int i) const { return {x[i], mask[i]}; }
  __device__ void operator()(int i, double s, EpiPre p) const {
    if (!p.m) x[i] = p.a + s;
  }
};

struct EpiSetScaled {  // x = 0 + omega * (FS r)   (first Richardson sweep from x = 0)
  double omega;
  double* x;
  __device__ EpiPre pre(int) const { return {0.0, 0}; }
  __device__ void operator()(int i, double s, EpiPre) const { x[i] = add_rn(0.0, mul_rn(omega, s)); }
};
struct EpiAxpy {  // x += omega * (FS r)          (precond.cpp:315)
  double omega;
  double* x;
  __device__ EpiPre pre(int i) const { return {x[i], 0}; }
  __device__ void operator()(int i, double s, EpiPre p) const { x[i] = add_rn(p.a, mul_rn(omega, s)); }
};
// last write of a coarse level's iterate in a V-cycle: the caller masks the
// correction at constrained columns (gmg.cpp:230-231); doing it here lets
// the prolongation gather plain values
struct EpiAxpyMasked {
  double omega;
  double* x;
  const unsigned char* mask;
  __device__ EpiPre pre(int i) const { return {x[i], mask[i]}; }
  __device__ void operator()(int i, double s, EpiPre p) const { x[i] = p.m ? 0.0 : add_rn(p.a, mul_rn(omega, s)); }
};

// x gather, optionally masked (ec[constrained_cols below] = 0, gmg.cpp:230-231)
struct GatherPlain {
  const double* x;
  __device__ double operator()(int c) const { return __ldg(x + c); }
};
struct GatherMasked {
  const double* x;
  const unsigned char* mask;
  __device__ double operator()(int c) const { return __ldg(mask + c) ? 0.0 : __ldg(x + c); }
};

template <int LPR, class Gather, class Epi, int U = 4>
__global__ void __launch_bounds__(256) csr_kernel(int rows, const int* __restrict__ ptr,
                                                  const int* __restrict__ idx,
                                                  const double* __restrict__ val, Gather gx,
                                                  Epi epi, unsigned long long* stamp) {
  stamp_fold(stamp);
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  // idle row groups still run the (empty) loop and the shuffle tree, so no
  // full-mask shuffle waits on an exited lane
  const bool ok = row < rows;
  pdl_trigger();
  // The matrix is setup data (never written by the solve): its row bounds
  // and first batch are fetched before the dependency wait, so under
  // programmatic dependent launch they overlap the predecessor's tail and
  // only the gathers of the vector remain on the critical path.
  const int k0 = ok ? __ldg(ptr + row) : 0, k1 = ok ? __ldg(ptr + row + 1) : 0;
  int c[U];
  double v[U];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + u * LPR;
      const bool in = k < k1;
      c[u] = in ? __ldg(idx + k) : -1;
      v[u] = in ? __ldg(val + k) : 0.0;
    }
  };
  load(k0 + lane);
  pdl_wait();
  stamp_start(stamp);
  EpiPre pe{0.0, 0};
  if (ok && lane == 0) pe = epi.pre(row);
  double s = 0.0;
  // predicated batches of U entries per lane: a batch's index/value loads
  // are in flight before its dependent x gathers, and the next batch's are
  // issued behind those gathers (no early exits)
  for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
    double xv[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = c[u] >= 0 ? gx(c[u]) : 0.0;
      vc[u] = v[u];
    }
    if (kb + U * LPR < k1) load(kb + U * LPR);
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(vc[u], xv[u], s);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  if (ok && lane == 0) epi(row, s, pe);
  stamp_end(stamp);
}

template <int LPR, class Gather, class Epi, int UP = 2>
__global__ void __launch_bounds__(256) csr_pair_kernel(int rows, const int* __restrict__ ptr,
                                                       const int* __restrict__ idx,
                                                       const double* __restrict__ val, Gather gx, Epi epi,
                                                       unsigned long long* stamp) {
  stamp_fold(stamp);
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = row < rows;
  pdl_trigger();
  // setup data (row bounds, first pair batch) before the dependency wait,
  // as in csr_kernel
  const int k0 = ok ? __ldg(ptr + row) : 0, k1 = ok ? __ldg(ptr + row + 1) : 0;
  int2 cn[UP];
  double2 vn[UP];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int k = kb + 2 * u * LPR;
      if (k < k1) {
        cn[u] = __ldg(reinterpret_cast<const int2*>(idx + k));
        vn[u] = __ldg(reinterpret_cast<const double2*>(val + k));
        if (k < k0) cn[u].x = -1;
        if (k + 1 >= k1) cn[u].y = -1;
      } else {
        cn[u] = make_int2(-1, -1);
        vn[u] = make_double2(0.0, 0.0);
      }
    }
  };
  load((k0 & ~1) + 2 * lane);
  pdl_wait();
  stamp_start(stamp);
  EpiPre pe{0.0, 0};
  if (ok && lane == 0) pe = epi.pre(row);
  double s = 0.0;
  for (int kb = (k0 & ~1) + 2 * lane; kb < k1; kb += 2 * UP * LPR) {
    int2 c[UP];
    double2 v[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      c[u] = cn[u];
      v[u] = vn[u];
    }
    if (kb + 2 * UP * LPR < k1) load(kb + 2 * UP * LPR);
    double x0[UP], x1[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      x0[u] = c[u].x >= 0 ? gx(c[u].x) : 0.0;
      x1[u] = c[u].y >= 0 ? gx(c[u].y) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      s = fma(v[u].x, x0[u], s);
      s = fma(v[u].y, x1[u], s);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  if (ok && lane == 0) epi(row, s, pe);
  stamp_end(stamp);
}

// ---- column-pair CSR ("BSR 1 x 2") ---------------------------------------
// The unknowns of the vector fields sit in (x, y) component pairs at
// consecutive frame positions, so the columns of a level-operator or FS-
// operator row come in aligned pairs (2c, 2c + 1): on config 0 every entry of
// the assembled FS operator and 97% of the entries of A. One element stores
// the pair's index c and both values (a missing partner is an explicit 0.0):
// 20 bytes per two entries instead of 24, one 4-B index load, one 16-B value
// load and ONE 16-B gather of x per two entries instead of two of each. The
// vector CSR kernels were L1/TEX-request bound before DRAM (ncu, round 1).
// Needs an even column count (the gathers read x as double2).
struct GatherPlain2 {
  const double* x;
  __device__ double2 operator()(int c2) const { return __ldg(reinterpret_cast<const double2*>(x) + c2); }
};
struct GatherMasked2 {
  const double* x;
  const unsigned char* mask;
  __device__ double2 operator()(int c2) const {
    const uchar2 m = __ldg(reinterpret_cast<const uchar2*>(mask) + c2);
    double2 v = __ldg(reinterpret_cast<const double2*>(x) + c2);
    if (m.x) v.x = 0.0;
    if (m.y) v.y = 0.0;
    return v;
  }
};
__device__ __forceinline__ GatherPlain2 to_pairs(const GatherPlain& g) { return {g.x}; }
__device__ __forceinline__ GatherMasked2 to_pairs(const GatherMasked& g) { return {g.x, g.mask}; }

// csr_kernel on the column-pair format: LPR lanes per row, predicated
// batches of U elements (= 2U entries) per lane, the same epilogues.
template <int LPR, class Gather, class Epi, int U>
__global__ void __launch_bounds__(256) csr2_kernel(int rows, const int* __restrict__ ptr,
                                                   const int* __restrict__ idx,
                                                   const double2* __restrict__ val, Gather gx1, Epi epi,
                                                   unsigned long long* stamp) {
  stamp_fold(stamp);
  const auto gx = to_pairs(gx1);
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = row < rows;
  pdl_trigger();
  const int k0 = ok ? __ldg(ptr + row) : 0, k1 = ok ? __ldg(ptr + row + 1) : 0;
  int c[U];
  double2 v[U];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + u * LPR;
      const bool in = k < k1;
      c[u] = in ? __ldg(idx + k) : -1;
      v[u] = in ? __ldg(val + k) : make_double2(0.0, 0.0);
    }
  };
  load(k0 + lane);
  pdl_wait();
  stamp_start(stamp);
  EpiPre pe{0.0, 0};
  if (ok && lane == 0) pe = epi.pre(row);
  double s = 0.0;
  for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
    double2 xv[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = c[u] >= 0 ? gx(c[u]) : make_double2(0.0, 0.0);
      vc[u] = v[u];
    }
    if (kb + U * LPR < k1) load(kb + U * LPR);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s = fma(vc[u].x, xv[u].x, s);
      s = fma(vc[u].y, xv[u].y, s);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  if (ok && lane == 0) epi(row, s, pe);
  stamp_end(stamp);
}

// ---- 2 x 2 block CSR on top of the column pairs --------------------------
// The two component rows (2R, 2R + 1) of a node share their column pattern
// in the FS operator, so a 2 x 2 block (rows 2R, 2R + 1 x columns 2c, 2c + 1)
// needs ONE 4-byte index for four values: 36 bytes per four entries (9 per
// entry against 10 for the column pairs and 12 for CSR), and one 16-byte
// gather of x serves both rows. val holds {a(2R,2c), a(2R,2c+1)} and
// {a(2R+1,2c), a(2R+1,2c+1)} as two consecutive double2. Patterns that
// differ between the two rows are merged (explicit zeros). LPR lanes per ROW
// PAIR, batches of U blocks per lane.
template <int LPR, class Gather, class Epi, int U>
__global__ void __launch_bounds__(256) bsr22_kernel(int row_pairs, const int* __restrict__ ptr,
                                                    const int* __restrict__ idx,
                                                    const double2* __restrict__ val, Gather gx1, Epi epi,
                                                    unsigned long long* stamp) {
  stamp_fold(stamp);
  const auto gx = to_pairs(gx1);
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int rp = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = rp < row_pairs;
  pdl_trigger();
  const int k0 = ok ? __ldg(ptr + rp) : 0, k1 = ok ? __ldg(ptr + rp + 1) : 0;
  int c[U];
  double2 v0[U], v1[U];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + u * LPR;
      const bool in = k < k1;
      c[u] = in ? __ldg(idx + k) : -1;
      v0[u] = in ? __ldg(val + 2 * (size_t)k) : make_double2(0.0, 0.0);
      v1[u] = in ? __ldg(val + 2 * (size_t)k + 1) : make_double2(0.0, 0.0);
    }
  };
  load(k0 + lane);
  pdl_wait();
  stamp_start(stamp);
  // lane 0 owns row 2 rp, lane 1 row 2 rp + 1 (their epilogue operands)
  EpiPre pe{0.0, 0};
  if (ok && lane < 2) pe = epi.pre(2 * rp + lane);
  double s0 = 0.0, s1 = 0.0;
  for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
    double2 xv[U], a0[U], a1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = c[u] >= 0 ? gx(c[u]) : make_double2(0.0, 0.0);
      a0[u] = v0[u];
      a1[u] = v1[u];
    }
    if (kb + U * LPR < k1) load(kb + U * LPR);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s0 = fma(a0[u].x, xv[u].x, s0);
      s0 = fma(a0[u].y, xv[u].y, s0);
      s1 = fma(a1[u].x, xv[u].x, s1);
      s1 = fma(a1[u].y, xv[u].y, s1);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(kFull, s0, o, LPR);
    s1 += __shfl_xor_sync(kFull, s1, o, LPR);
  }
  if (ok && lane < 2) epi(2 * rp + lane, lane ? s1 : s0, pe);
  stamp_end(stamp);
}

// setup: blocks per row pair (pass 0) / fill (pass 1) from the column-pair
// format (ptr2/idx2/val2 with sorted pair indices): merge of the two rows
__global__ void bsr22_build_kernel(int row_pairs, const int* __restrict__ ptr2, const int* __restrict__ idx2,
                                   const double2* __restrict__ val2, int* __restrict__ ptrb, int* __restrict__ idxb,
                                   double2* __restrict__ valb, int pass) {
  const int rp = blockIdx.x * blockDim.x + threadIdx.x;
  if (rp >= row_pairs) return;
  int a = ptr2[2 * rp], ae = ptr2[2 * rp + 1], b = ae, be = ptr2[2 * rp + 2];
  int n = 0;
  const int o = pass ? ptrb[rp] : 0;
  while (a < ae || b < be) {
    const int ca = a < ae ? idx2[a] : 0x7fffffff, cb = b < be ? idx2[b] : 0x7fffffff;
    const int cmin = ca < cb ? ca : cb;
    if (pass) {
      idxb[o + n] = cmin;
      valb[2 * (size_t)(o + n)] = ca == cmin ? val2[a] : make_double2(0.0, 0.0);
      valb[2 * (size_t)(o + n) + 1] = cb == cmin ? val2[b] : make_double2(0.0, 0.0);
    }
    if (ca == cmin) ++a;
    if (cb == cmin) ++b;
    ++n;
  }
  if (!pass) ptrb[rp + 1] = n;
}

// setup: elements per row (pass 0, out = counts) / fill (pass 1) of the
// column-pair format from a CSR with sorted columns; one thread per row
__global__ void csr2_build_kernel(int rows, const int* __restrict__ ptr, const int* __restrict__ idx,
                                  const double* __restrict__ val, int* __restrict__ ptr2, int* __restrict__ idx2,
                                  double2* __restrict__ val2, int pass) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int k0 = ptr[r], k1 = ptr[r + 1];
  int n = 0, o = pass ? ptr2[r] : 0;
  for (int k = k0; k < k1;) {
    const int c = idx[k], c2 = c >> 1;
    const bool two = k + 1 < k1 && (idx[k + 1] >> 1) == c2;  // sorted: (2 c2, 2 c2 + 1)
    if (pass) {
      double2 v;
      if (two) v = make_double2(val[k], val[k + 1]);
      else v = (c & 1) ? make_double2(0.0, val[k]) : make_double2(val[k], 0.0);
      idx2[o + n] = c2;
      val2[o + n] = v;
    }
    ++n;
    k += two ? 2 : 1;
  }
  if (!pass) ptr2[r + 1] = n;
}

// FS combine on one level (precond.cpp:42-57 additive + 271-287 + 305-317):
//   p <  g1, p >= g1+n_us : z = sum_{(b,i) covering p, block order} delta / cover
//   g1 <= p < g1+n_us     : z = r[p] / lumped[p-g1]
//   x[p] = (x_zero ? 0 : x[p]) + omega * z
// Same rounded operations in the same order as the reference (bit-exact).
__global__ void fs_combine_kernel(int n, int g1, int n_us, const int* __restrict__ inv_ptr,
                                  const int* __restrict__ inv_idx, const double* __restrict__ delta,
                                  const double* __restrict__ r, const double* __restrict__ lumped,
                                  double omega, double* __restrict__ x, int x_zero) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  pdl_trigger();
  pdl_wait();
  if (p >= n) return;
  double z;
  if (p >= g1 && p < g1 + n_us) {
    z = r[p] / lumped[p - g1];
  } else {
    const int k0 = inv_ptr[p], k1 = inv_ptr[p + 1];
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s = add_rn(s, delta[inv_idx[k]]);
    z = (k1 - k0 > 1) ? s / (double)(k1 - k0) : s;
  }
  const double xo = x_zero ? 0.0 : x[p];
  x[p] = add_rn(xo, mul_rn(omega, z));
}

// Coarse solve x0 (+)= Ainv' b0 with the explicit equilibrated inverse
// (row-major n0 x n0): one T-thread CTA per row, U predicated loads per
// thread per batch, so a row of <= T * U columns is ONE batch (latency-bound
// at these sizes); xor tree per warp, warp sums added in warp order.
// <256, 8> is the default; <64, 22> serves coarse levels whose row count
// would otherwise need a second wave of 256-thread CTAs (config 0: 1,348
// rows against 5 x 148 resident CTAs; in-graph 3.2 us).
constexpr int kGemvThreads = 256;
template <int T, int U>
__global__ void __launch_bounds__(T) gemv_kernel(int n, const double* __restrict__ M, const double* __restrict__ b,
                                                 double* __restrict__ x, int accumulate,
                                                 const unsigned char* __restrict__ mask_out,
                                                 unsigned long long* stamp) {
  stamp_fold(stamp);
  __shared__ double red[T / 32];
  const int row = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  pdl_trigger();
  // the inverse and the mask are setup data: the row's first batch is
  // fetched before the dependency wait (see csr_kernel)
  const double* Mr = M + (size_t)row * n;
  double mv[U];
  auto load = [&](int jb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + T * u;
      mv[u] = j < n ? __ldg(Mr + j) : 0.0;
    }
  };
  load(t);
  unsigned char mo = 0;
  if (t == 0 && mask_out) mo = __ldg(mask_out + row);
  pdl_wait();
  stamp_start(stamp);
  double xo = 0.0;
  if (t == 0 && accumulate) xo = x[row];
  double s = 0.0;
  for (int jb = t; jb < n; jb += T * U) {
    double bv[U], mc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + T * u;
      bv[u] = j < n ? __ldg(b + j) : 0.0;
      mc[u] = mv[u];
    }
    if (jb + T * U < n) load(jb + T * U);
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(mc[u], bv[u], s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (t == 0) {
    double z = 0.0;
#pragma unroll
    for (int w = 0; w < T / 32; ++w) z += red[w];
    x[row] = mo ? 0.0 : (accumulate ? xo + z : z);
  }
  stamp_end(stamp);
}

// ---- setup: Gauss-Jordan inverse with partial pivoting on W = [A | I] ----
// Row k's pivot swap moves only the left columns [k, n) and the right
// columns [n, n+k) (the dense part); the unit entries of the not yet
// eliminated rows stay in place, which is the row swap followed by a swap of
// right-half columns n+k <-> n+p. So at step k the live columns are the
// contiguous range [k+1, n+k] (half of [A | I]), and the inverse is the right
// half with its columns unpermuted at the end (gj_extract_kernel, perm from
// the host).
// Step k, single CTA: pivot search in column k, the swap, pivot-row scaling
// of [k+1, n+k], and the elimination factors f = W[:, k] (f[k] = 0).
__global__ void gj_pivot_kernel(int n, double* __restrict__ W, int k, double* __restrict__ f,
                                int* __restrict__ fail, int* __restrict__ piv) {
  __shared__ double sb[32];
  __shared__ int si[32];
  __shared__ int s_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ld = 2 * n;
  double best = -1.0;
  int bi = n;
  for (int i = k + tid; i < n; i += blockDim.x) {
    const double v = fabs(W[(size_t)i * ld + k]);
    if (v > best) {
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, o);
    const int oi = __shfl_xor_sync(kFull, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if (lane == 0) {
    sb[warp] = best;
    si[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < nw; ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < bi)) {
        best = sb[w];
        bi = si[w];
      }
    if (!(best > 1e-14) || bi >= n) *fail = 1;  // equilibrated: entries <= 1
    s_p = bi < n ? bi : k;
    piv[k] = s_p;
  }
  __syncthreads();
  const int p = s_p;
  if (p != k)
    for (int j = k + tid; j < n + k; j += blockDim.x) {
      const double t = W[(size_t)k * ld + j];
      W[(size_t)k * ld + j] = W[(size_t)p * ld + j];
      W[(size_t)p * ld + j] = t;
    }
  __syncthreads();
  const double inv = 1.0 / W[(size_t)k * ld + k];
  for (int j = k + 1 + tid; j <= n + k; j += blockDim.x) W[(size_t)k * ld + j] *= inv;
  for (int i = tid; i < n; i += blockDim.x) f[i] = (i == k) ? 0.0 : W[(size_t)i * ld + k];
}

// rows i != k: W[i, j] -= f_i W[k, j] for the live columns j in [k+1, n+k]
__global__ void gj_eliminate_kernel(int n, double* __restrict__ W, int k,
                                    const double* __restrict__ f) {
  const int ld = 2 * n;
  const int j = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j > n + k) return;
  const double fi = f[i];
  if (fi == 0.0) return;
  W[(size_t)i * ld + j] -= fi * W[(size_t)k * ld + j];
}

// M[i][j] = cs_i * W[i][n + col[j]] * rs_j  (A^{-1} = Dc Ahat^{-1} Dr, right
// half unpermuted by col)
__global__ void gj_extract_kernel(int n, const double* __restrict__ W, const int* __restrict__ col,
                                  const double* __restrict__ rs, const double* __restrict__ cs,
                                  double* __restrict__ M) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e / n), j = (int)(e % n);
  M[e] = cs[i] * W[(size_t)i * 2 * n + n + col[j]] * rs[j];
}

// W = [diag(rs) A diag(cs) | I], W zeroed before
__global__ void gj_init_kernel(int n, const int* __restrict__ ptr, const int* __restrict__ idx,
                               const double* __restrict__ val, const double* __restrict__ rs,
                               const double* __restrict__ cs, double* __restrict__ W) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* Wi = W + (size_t)i * 2 * n;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = idx[k];
    Wi[j] += val[k] * rs[i] * cs[j];
  }
  Wi[n + i] = 1.0;
}

}  // namespace fsigpu

namespace fsigpu {
// ---- fused coarse-grid correction + post-smoothing residual -------------
//   x[i]  += (P ec_m)[i]           if !cmask[i]      (gmg.cpp:233-236)
//   r[i]   = r_pre[i] - (AP_m ec_m)[i]               (= b - A x_new)
// with AP_m = A * diag(!cmask) * P precomputed at setup and ec_m the coarse
// correction masked by the coarse col mask (gmg.cpp:230-231).
template <int LPR, int U = 8>
__device__ __forceinline__ double row_sum(const int* __restrict__ ptr, const int* __restrict__ idx,
                                          const double* __restrict__ val, int row, int lane, const double* x,
                                          const unsigned char* mask /* nullptr: x already masked */) {
  const int k0 = row >= 0 ? __ldg(ptr + row) : 0, k1 = row >= 0 ? __ldg(ptr + row + 1) : 0;
  double s = 0.0;
  for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
    int c[U];
    double v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + u * LPR;
      const bool ok = k < k1;
      c[u] = ok ? __ldg(idx + k) : -1;
      v[u] = ok ? __ldg(val + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      xv[u] = c[u] >= 0 ? ((mask && __ldg(mask + c[u])) ? 0.0 : __ldg(x + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(v[u], xv[u], s);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  return s;
}

// x += P ec ; r = r_pre - (A P) ec for one fine row per LPR lanes. The P
// row (<= 9 entries for Q2 / 3 for P1disc) and the first UA*LPR entries of
// the AP row are fetched in ONE predicated batch, so the two independent
// pointer -> index -> gather chains overlap instead of running back to back.
template <int LPR, int UA>
__global__ void __launch_bounds__(256) prolong_resid_kernel(int rows, const int* __restrict__ pp,
                                                            const int* __restrict__ pi, const double* __restrict__ pv,
                                                            const int* __restrict__ ap, const int* __restrict__ ai,
                                                            const double* __restrict__ av, const double* ec,
                                                            const unsigned char* __restrict__ cmask_coarse,
                                                            const unsigned char* __restrict__ cmask, double* x,
                                                            const double* r_pre, double* r, unsigned long long* stamp) {
  stamp_fold(stamp);
  // P rows hold <= 9 entries (Q2 natural injection, 3 for the P1disc
  // pressure): size the P batch so one batch covers them at any LPR (at
  // least 2 per lane, the config-0 tuning); the tail loop below then only
  // runs for unusual transfer operators
  constexpr int UP = (9 + LPR - 1) / LPR > 2 ? (9 + LPR - 1) / LPR : 2;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = row < rows;
  pdl_trigger();
  // setup data (P, AP, the masks) before the dependency wait (see csr_kernel)
  int p0 = 0, p1 = 0, a0 = 0, a1 = 0;
  if (ok) {
    p0 = __ldg(pp + row);
    p1 = __ldg(pp + row + 1);
    a0 = __ldg(ap + row);
    a1 = __ldg(ap + row + 1);
  }
  unsigned char cm = 1;
  if (ok && lane == 0) cm = __ldg(cmask + row);
  double s1 = 0.0, s2 = 0.0;
  int kp = p0 + lane, ka = a0 + lane;
  int c[UP + UA];
  double v[UP + UA];
#pragma unroll
  for (int u = 0; u < UP; ++u) {
    const int k = kp + u * LPR;
    const bool in = k < p1;
    c[u] = in ? __ldg(pi + k) : -1;
    v[u] = in ? __ldg(pv + k) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < UA; ++u) {
    const int k = ka + u * LPR;
    const bool in = k < a1;
    c[UP + u] = in ? __ldg(ai + k) : -1;
    v[UP + u] = in ? __ldg(av + k) : 0.0;
  }
  pdl_wait();
  stamp_start(stamp);
  // the row's own operands, loaded before the dot products (see EpiPre)
  double xo = 0.0, rp = 0.0;
  if (ok && lane == 0) {
    xo = x[row];
    rp = r_pre[row];
  }
  auto gather = [&](int c) -> double {
    return c >= 0 ? ((cmask_coarse && __ldg(cmask_coarse + c)) ? 0.0 : __ldg(ec + c)) : 0.0;
  };
  {
    double xv[UP + UA];
#pragma unroll
    for (int u = 0; u < UP + UA; ++u) xv[u] = gather(c[u]);
#pragma unroll
    for (int u = 0; u < UP; ++u) s1 = fma(v[u], xv[u], s1);
#pragma unroll
    for (int u = 0; u < UA; ++u) s2 = fma(v[UP + u], xv[UP + u], s2);
  }
  // tails (rows longer than one batch)
  for (kp += UP * LPR; kp < p1; kp += LPR) s1 = fma(__ldg(pv + kp), gather(__ldg(pi + kp)), s1);
  for (ka += UA * LPR; ka < a1; ka += UA * LPR) {
    int c[UA];
    double v[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int k = ka + u * LPR;
      const bool in = k < a1;
      c[u] = in ? __ldg(ai + k) : -1;
      v[u] = in ? __ldg(av + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UA; ++u) s2 = fma(v[u], gather(c[u]), s2);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(kFull, s1, o, LPR);
    s2 += __shfl_xor_sync(kFull, s2, o, LPR);
  }
  if (ok && lane == 0) {
    if (!cm) x[row] = xo + s1;
    r[row] = rp - s2;
  }
  stamp_end(stamp);
}

// prolong_resid_kernel with the A*P half in the column-pair format (one
// element = columns 2c, 2c + 1 of the coarse iterate: 20 bytes and one
// 16-byte gather per two entries; large levels), UA elements per lane per
// batch. The P half stays scalar.
template <int LPR, int UA>
__global__ void __launch_bounds__(256) prolong_resid2_kernel(int rows, const int* __restrict__ pp,
                                                             const int* __restrict__ pi, const double* __restrict__ pv,
                                                             const int* __restrict__ ap, const int* __restrict__ ai,
                                                             const double2* __restrict__ av, const double* ec,
                                                             const unsigned char* __restrict__ cmask_coarse,
                                                             const unsigned char* __restrict__ cmask, double* x,
                                                             const double* r_pre, double* r, unsigned long long* stamp) {
  stamp_fold(stamp);
  constexpr int UP = (9 + LPR - 1) / LPR > 2 ? (9 + LPR - 1) / LPR : 2;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = row < rows;
  pdl_trigger();
  int p0 = 0, p1 = 0, a0 = 0, a1 = 0;
  if (ok) {
    p0 = __ldg(pp + row);
    p1 = __ldg(pp + row + 1);
    a0 = __ldg(ap + row);
    a1 = __ldg(ap + row + 1);
  }
  unsigned char cm = 1;
  if (ok && lane == 0) cm = __ldg(cmask + row);
  double s1 = 0.0, s2 = 0.0;
  int kp = p0 + lane, ka = a0 + lane;
  int c[UP], c2[UA];
  double v[UP];
  double2 v2[UA];
#pragma unroll
  for (int u = 0; u < UP; ++u) {
    const int k = kp + u * LPR;
    const bool in = k < p1;
    c[u] = in ? __ldg(pi + k) : -1;
    v[u] = in ? __ldg(pv + k) : 0.0;
  }
  auto load2 = [&](int kb) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int k = kb + u * LPR;
      const bool in = k < a1;
      c2[u] = in ? __ldg(ai + k) : -1;
      v2[u] = in ? __ldg(av + k) : make_double2(0.0, 0.0);
    }
  };
  load2(ka);
  pdl_wait();
  stamp_start(stamp);
  double xo = 0.0, rp = 0.0;
  if (ok && lane == 0) {
    xo = x[row];
    rp = r_pre[row];
  }
  auto gather = [&](int cc) -> double {
    return cc >= 0 ? ((cmask_coarse && __ldg(cmask_coarse + cc)) ? 0.0 : __ldg(ec + cc)) : 0.0;
  };
  auto gather2 = [&](int cc) -> double2 {
    if (cc < 0) return make_double2(0.0, 0.0);
    double2 e = __ldg(reinterpret_cast<const double2*>(ec) + cc);
    if (cmask_coarse) {
      const uchar2 m = __ldg(reinterpret_cast<const uchar2*>(cmask_coarse) + cc);
      if (m.x) e.x = 0.0;
      if (m.y) e.y = 0.0;
    }
    return e;
  };
  {
    double xv[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) xv[u] = gather(c[u]);
#pragma unroll
    for (int u = 0; u < UP; ++u) s1 = fma(v[u], xv[u], s1);
  }
  for (kp += UP * LPR; kp < p1; kp += LPR) s1 = fma(__ldg(pv + kp), gather(__ldg(pi + kp)), s1);
  for (; ka < a1; ka += UA * LPR) {
    double2 xv[UA], vc[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      xv[u] = gather2(c2[u]);
      vc[u] = v2[u];
    }
    if (ka + UA * LPR < a1) load2(ka + UA * LPR);
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      s2 = fma(vc[u].x, xv[u].x, s2);
      s2 = fma(vc[u].y, xv[u].y, s2);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(kFull, s1, o, LPR);
    s2 += __shfl_xor_sync(kFull, s2, o, LPR);
  }
  if (ok && lane == 0) {
    if (!cm) x[row] = xo + s1;
    r[row] = rp - s2;
  }
  stamp_end(stamp);
}

// The same for a ROW PAIR (2 rp, 2 rp + 1) with A*P as 2 x 2 blocks
// (bsr22_kernel's format): one index and one 16-byte gather of the coarse
// iterate per four entries. LPR lanes per row pair; the two P rows stay
// scalar (lanes 0 / 1 own the two rows' epilogues).
template <int LPR, int UA>
__global__ void __launch_bounds__(256) prolong_resid22_kernel(int row_pairs, const int* __restrict__ pp,
                                                              const int* __restrict__ pi, const double* __restrict__ pv,
                                                              const int* __restrict__ ap, const int* __restrict__ ai,
                                                              const double2* __restrict__ av, const double* ec,
                                                              const unsigned char* __restrict__ cmask_coarse,
                                                              const unsigned char* __restrict__ cmask, double* x,
                                                              const double* r_pre, double* r, unsigned long long* stamp) {
  stamp_fold(stamp);
  constexpr int UP = (9 + LPR - 1) / LPR > 1 ? (9 + LPR - 1) / LPR : 1;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int rp = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = rp < row_pairs;
  pdl_trigger();
  int p0 = 0, p1 = 0, p2 = 0, a0 = 0, a1 = 0;
  if (ok) {
    p0 = __ldg(pp + 2 * rp);
    p1 = __ldg(pp + 2 * rp + 1);
    p2 = __ldg(pp + 2 * rp + 2);
    a0 = __ldg(ap + rp);
    a1 = __ldg(ap + rp + 1);
  }
  unsigned char cm = 1;
  if (ok && lane < 2) cm = __ldg(cmask + 2 * rp + lane);
  int ca[UP], cb[UP], c2[UA];
  double va[UP], vb[UP];
  double2 v0[UA], v1[UA];
#pragma unroll
  for (int u = 0; u < UP; ++u) {
    const int ka = p0 + lane + u * LPR, kb = p1 + lane + u * LPR;
    ca[u] = ka < p1 ? __ldg(pi + ka) : -1;
    va[u] = ka < p1 ? __ldg(pv + ka) : 0.0;
    cb[u] = kb < p2 ? __ldg(pi + kb) : -1;
    vb[u] = kb < p2 ? __ldg(pv + kb) : 0.0;
  }
  int ka2 = a0 + lane;
  auto load2 = [&](int kb) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int k = kb + u * LPR;
      const bool in = k < a1;
      c2[u] = in ? __ldg(ai + k) : -1;
      v0[u] = in ? __ldg(av + 2 * (size_t)k) : make_double2(0.0, 0.0);
      v1[u] = in ? __ldg(av + 2 * (size_t)k + 1) : make_double2(0.0, 0.0);
    }
  };
  load2(ka2);
  pdl_wait();
  stamp_start(stamp);
  double xo = 0.0, rpre = 0.0;
  if (ok && lane < 2) {
    xo = x[2 * rp + lane];
    rpre = r_pre[2 * rp + lane];
  }
  auto gather = [&](int cc) -> double {
    return cc >= 0 ? ((cmask_coarse && __ldg(cmask_coarse + cc)) ? 0.0 : __ldg(ec + cc)) : 0.0;
  };
  auto gather2 = [&](int cc) -> double2 {
    if (cc < 0) return make_double2(0.0, 0.0);
    double2 e = __ldg(reinterpret_cast<const double2*>(ec) + cc);
    if (cmask_coarse) {
      const uchar2 m = __ldg(reinterpret_cast<const uchar2*>(cmask_coarse) + cc);
      if (m.x) e.x = 0.0;
      if (m.y) e.y = 0.0;
    }
    return e;
  };
  double s1a = 0.0, s1b = 0.0, s2a = 0.0, s2b = 0.0;
  {
    double xa[UP], xb[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      xa[u] = gather(ca[u]);
      xb[u] = gather(cb[u]);
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      s1a = fma(va[u], xa[u], s1a);
      s1b = fma(vb[u], xb[u], s1b);
    }
  }
  for (int k = p0 + lane + UP * LPR; k < p1; k += LPR) s1a = fma(__ldg(pv + k), gather(__ldg(pi + k)), s1a);
  for (int k = p1 + lane + UP * LPR; k < p2; k += LPR) s1b = fma(__ldg(pv + k), gather(__ldg(pi + k)), s1b);
  for (; ka2 < a1; ka2 += UA * LPR) {
    double2 xv[UA], w0[UA], w1[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      xv[u] = gather2(c2[u]);
      w0[u] = v0[u];
      w1[u] = v1[u];
    }
    if (ka2 + UA * LPR < a1) load2(ka2 + UA * LPR);
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      s2a = fma(w0[u].x, xv[u].x, s2a);
      s2a = fma(w0[u].y, xv[u].y, s2a);
      s2b = fma(w1[u].x, xv[u].x, s2b);
      s2b = fma(w1[u].y, xv[u].y, s2b);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    s1a += __shfl_xor_sync(kFull, s1a, o, LPR);
    s1b += __shfl_xor_sync(kFull, s1b, o, LPR);
    s2a += __shfl_xor_sync(kFull, s2a, o, LPR);
    s2b += __shfl_xor_sync(kFull, s2b, o, LPR);
  }
  if (ok && lane < 2) {
    const int row = 2 * rp + lane;
    if (!cm) x[row] = xo + (lane ? s1b : s1a);
    r[row] = rpre - (lane ? s2b : s2a);
  }
  stamp_end(stamp);
}

// prolong_resid_kernel with the A*P half streamed as 16-byte pairs (int2
// columns, double2 values; see csr_pair_kernel), UA pairs per lane per
// batch. The P half and the first A*P batch are still fetched together.
template <int LPR, int UA>
__global__ void __launch_bounds__(256) prolong_resid_pair_kernel(
    int rows, const int* __restrict__ pp, const int* __restrict__ pi, const double* __restrict__ pv,
    const int* __restrict__ ap, const int* __restrict__ ai, const double* __restrict__ av, const double* ec,
    const unsigned char* __restrict__ cmask_coarse, const unsigned char* __restrict__ cmask, double* x,
    const double* r_pre, double* r, unsigned long long* stamp) {
  stamp_fold(stamp);
  constexpr int UP = (9 + LPR - 1) / LPR;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / LPR);
  const int lane = threadIdx.x & (LPR - 1);
  const bool ok = row < rows;
  pdl_trigger();
  // setup data (P, AP, the masks) before the dependency wait (see csr_kernel)
  int p0 = 0, p1 = 0, a0 = 0, a1 = 0;
  if (ok) {
    p0 = __ldg(pp + row);
    p1 = __ldg(pp + row + 1);
    a0 = __ldg(ap + row);
    a1 = __ldg(ap + row + 1);
  }
  unsigned char cm = 1;
  if (ok && lane == 0) cm = __ldg(cmask + row);
  auto gather = [&](int c) -> double {
    return c >= 0 ? ((cmask_coarse && __ldg(cmask_coarse + c)) ? 0.0 : __ldg(ec + c)) : 0.0;
  };
  auto load_pairs = [&](int kb, int2 (&c)[UA], double2 (&v)[UA]) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int k = kb + 2 * u * LPR;
      if (k < a1) {
        c[u] = __ldg(reinterpret_cast<const int2*>(ai + k));
        v[u] = __ldg(reinterpret_cast<const double2*>(av + k));
        if (k < a0) c[u].x = -1;
        if (k + 1 >= a1) c[u].y = -1;
      } else {
        c[u] = make_int2(-1, -1);
        v[u] = make_double2(0.0, 0.0);
      }
    }
  };
  double s1 = 0.0, s2 = 0.0, xo = 0.0, rp = 0.0;
  int kp = p0 + lane, ka = (a0 & ~1) + 2 * lane;
  {
    int cp[UP];
    double vp[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int k = kp + u * LPR;
      const bool in = k < p1;
      cp[u] = in ? __ldg(pi + k) : -1;
      vp[u] = in ? __ldg(pv + k) : 0.0;
    }
    int2 c[UA];
    double2 v[UA];
    load_pairs(ka, c, v);
    pdl_wait();
    stamp_start(stamp);
    if (ok && lane == 0) {
      xo = x[row];
      rp = r_pre[row];
    }
    double xp[UP], x0[UA], x1[UA];
#pragma unroll
    for (int u = 0; u < UP; ++u) xp[u] = gather(cp[u]);
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      x0[u] = gather(c[u].x);
      x1[u] = gather(c[u].y);
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) s1 = fma(vp[u], xp[u], s1);
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      s2 = fma(v[u].x, x0[u], s2);
      s2 = fma(v[u].y, x1[u], s2);
    }
  }
  for (kp += UP * LPR; kp < p1; kp += LPR) s1 = fma(__ldg(pv + kp), gather(__ldg(pi + kp)), s1);
  for (ka += 2 * UA * LPR; ka < a1; ka += 2 * UA * LPR) {
    int2 c[UA];
    double2 v[UA];
    load_pairs(ka, c, v);
    double x0[UA], x1[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      x0[u] = gather(c[u].x);
      x1[u] = gather(c[u].y);
    }
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      s2 = fma(v[u].x, x0[u], s2);
      s2 = fma(v[u].y, x1[u], s2);
    }
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(kFull, s1, o, LPR);
    s2 += __shfl_xor_sync(kFull, s2, o, LPR);
  }
  if (ok && lane == 0) {
    if (!cm) x[row] = xo + s1;
    r[row] = rp - s2;
  }
  stamp_end(stamp);
}

// ---- assembled FS operator (setup): COO entries of
//   sum_b R_b^T inv(A_b) R_b / cover  (additive Schwarz, precond.cpp:44-57)
// one CTA per block; key = (row << 32) | col
__global__ void fs_coo_blocks_kernel(int nb, const int* __restrict__ msz, const long long* __restrict__ row_off,
                                     const double* __restrict__ inv, const long long* __restrict__ inv_off,
                                     const int* __restrict__ pos, const int* __restrict__ inv_ptr,
                                     const long long* __restrict__ coo_off, unsigned long long* __restrict__ keys,
                                     double* __restrict__ vals) {
  const int b = blockIdx.x;
  if (b >= nb) return;
  const int m = msz[b];
  const int ld = (m + 1) & ~1;
  const long long ro = row_off[b];
  const double* M = inv + inv_off[b];
  const long long o = coo_off[b];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int j = e / m, i = e % m;  // column-major walk
    const int pi = pos[ro + i], pj = pos[ro + j];
    const int cov = inv_ptr[pi + 1] - inv_ptr[pi];
    double v = M[(size_t)j * ld + i];
    if (cov > 1) v = v / (double)cov;
    keys[o + e] = ((unsigned long long)(unsigned)pi << 32) | (unsigned)pj;
    vals[o + e] = v;
  }
}

// The lumped-Jacobi coupling of the AS2 blocks (precond.cpp:281-287):
// entries (p_i, g1 + c) = -inv(A_b)[i, j] * A_g2[p_j, c] / lumped[c] (/ cover)
// for every row i and coupling (j, c) of block b, emitted in the host
// loop's order (i, then the block's couplings j-major), one CTA per block.
__global__ void fs_coo_coupling_kernel(const int* __restrict__ blk, const int* __restrict__ msz,
                                       const long long* __restrict__ row_off, const double* __restrict__ inv,
                                       const long long* __restrict__ inv_off, const int* __restrict__ pos,
                                       const int* __restrict__ inv_ptr, const long long* __restrict__ cl_off,
                                       const int* __restrict__ cl_j, const int* __restrict__ cl_k,
                                       const int* __restrict__ ac, const double* __restrict__ av,
                                       const double* __restrict__ lumped, int g1, const long long* __restrict__ out_off,
                                       unsigned long long* __restrict__ keys, double* __restrict__ vals) {
  const int q = blockIdx.x;
  const int b = blk[q];
  const int m = msz[b];
  const int ld = (m + 1) & ~1;
  const long long ro = row_off[b];
  const double* M = inv + inv_off[b];
  const long long c0 = cl_off[q];
  const int nc = (int)(cl_off[q + 1] - c0);
  const long long o = out_off[q];
  for (long long e = threadIdx.x; e < (long long)m * nc; e += blockDim.x) {
    const int i = (int)(e / nc), t = (int)(e % nc);
    const int j = cl_j[c0 + t], k = cl_k[c0 + t];
    const int pi = pos[ro + i];
    const int cov = inv_ptr[pi + 1] - inv_ptr[pi];
    const int c = ac[k];
    double v = -M[(size_t)j * ld + i] * av[k] / lumped[c];
    if (cov > 1) v = v / (double)cov;
    keys[o + e] = ((unsigned long long)(unsigned)pi << 32) | (unsigned)(g1 + c);
    vals[o + e] = v;
  }
}

__global__ void coo_row_count_kernel(long long nnz, const unsigned long long* __restrict__ keys,
                                     int* __restrict__ cnt) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  atomicAdd(cnt + (int)(keys[e] >> 32) + 1, 1);
}

__global__ void coo_cols_kernel(long long nnz, const unsigned long long* __restrict__ keys, int* __restrict__ cols) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  cols[e] = (int)(keys[e] & 0xffffffffull);
}
}  // namespace fsigpu

namespace fsigpu {
// ---- setup: A*P on the device ---------------------------------------------
// AP_m = A * diag(!col_mask) * P, one CTA per row: the row's products
// (c, a_ik * p_kc) are collected in traversal order (k ascending, then the P
// row), sorted by (column, traversal index) and summed per column in
// traversal order with separate rounded mul/add: the host Gustavson loop's
// exact arithmetic (acc += a * p from 0), so AP is bit-identical to it.
constexpr int kApThreads = 128;
constexpr int kApCap = 2048;  // products per row (Q2: <= 65 x 9)

// exclusive scan of v[0..n) in shared memory (any n), block-wide; returns the total
__device__ __forceinline__ int ap_block_scan(int* v, int n, int* part) {
  const int t = threadIdx.x;
  const int per = (n + kApThreads - 1) / kApThreads;
  const int b = t * per, e = min(n, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += v[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int q = 0; q < kApThreads; ++q) {
      const int x = part[q];
      part[q] = acc;
      acc += x;
    }
    part[kApThreads] = acc;
  }
  __syncthreads();
  int acc = part[t];
  for (int i = b; i < e; ++i) {
    const int x = v[i];
    v[i] = acc;
    acc += x;
  }
  __syncthreads();
  return part[kApThreads];
}

__global__ void __launch_bounds__(kApThreads) ap_row_kernel(int n, const int* __restrict__ ap, const int* __restrict__ ai,
                                                            const double* __restrict__ av,
                                                            const unsigned char* __restrict__ cmask,
                                                            const int* __restrict__ pp, const int* __restrict__ pi,
                                                            const double* __restrict__ pv, int pass,
                                                            int* __restrict__ count, const long long* __restrict__ off,
                                                            int* __restrict__ oi, double* __restrict__ ov,
                                                            int* overflow) {
  __shared__ unsigned long long key[kApCap];
  __shared__ double val[kApCap];
  __shared__ int len[kApCap];
  __shared__ int part[kApThreads + 1];
  const int row = blockIdx.x;
  const int t = threadIdx.x;
  const int k0 = ap[row], k1 = ap[row + 1];
  const int na = k1 - k0;
  if (na > kApCap) {
    if (t == 0) atomicExch(overflow, 1);
    return;
  }
  // products in traversal order (k ascending, then the P row): slot base of
  // A entry k = exclusive prefix of the P row lengths of the unmasked columns
  for (int q = t; q < na; q += kApThreads) {
    const int c = ai[k0 + q];
    len[q] = cmask[c] ? 0 : pp[c + 1] - pp[c];
  }
  __syncthreads();
  const int np = ap_block_scan(len, na, part);
  if (np > kApCap) {
    if (t == 0) atomicExch(overflow, 1);
    return;
  }
  for (int q = t; q < na; q += kApThreads) {
    const int c = ai[k0 + q];
    if (cmask[c]) continue;
    const double a = av[k0 + q];
    int slot = len[q];
    for (int r = pp[c]; r < pp[c + 1]; ++r, ++slot) {
      key[slot] = ((unsigned long long)(unsigned)pi[r] << 32) | (unsigned)slot;
      val[slot] = __dmul_rn(a, pv[r]);
    }
  }
  int n2 = 1;
  while (n2 < np) n2 <<= 1;
  for (int i = np + t; i < n2; i += kApThreads) key[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < n2; i += kApThreads) {
        const int ij = i ^ j;
        if (ij > i) {
          const bool up = (i & k) == 0;
          const unsigned long long x = key[i], y = key[ij];
          if ((x > y) == up) {  // values stay put: the slot is the key's low word
            key[i] = y;
            key[ij] = x;
          }
        }
      }
      __syncthreads();
    }
  // column runs: head flags -> their output index (exclusive scan), then
  // each head sums its run in traversal order
  for (int i = t; i < np; i += kApThreads)
    len[i] = (i == 0 || (key[i] >> 32) != (key[i - 1] >> 32)) ? 1 : 0;
  __syncthreads();
  const int nu = ap_block_scan(len, np, part);
  if (!pass) {
    if (t == 0) count[row] = nu;
    return;
  }
  const long long o = off[row];
  for (int i = t; i < np; i += kApThreads) {
    const unsigned col = (unsigned)(key[i] >> 32);
    const bool head = i == 0 || (unsigned)(key[i - 1] >> 32) != col;
    if (!head) continue;
    double acc = 0.0;
    for (int j = i; j < np && (unsigned)(key[j] >> 32) == col; ++j) acc = __dadd_rn(acc, val[(unsigned)key[j]]);
    oi[o + len[i]] = (int)col;
    ov[o + len[i]] = acc;
  }
}

// CSR sanity on the device (the host loops over ~1e8 entries took seconds):
// offsets nondecreasing from 0, columns in [0, cols)
__global__ void csr_check_kernel(int rows, int cols, long long nnz, const int* __restrict__ ptr,
                                 const int* __restrict__ idx, int* bad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) {
    const int a = ptr[i], b = ptr[i + 1];
    if (a > b || (i == 0 && a != 0) || a < 0 || b > nnz) atomicOr(bad, 1);
    for (int k = max(a, 0); k < b && k < nnz; ++k)
      if (idx[k] < 0 || idx[k] >= cols) {
        atomicOr(bad, 2);
        break;
      }
  }
}
}  // namespace fsigpu
