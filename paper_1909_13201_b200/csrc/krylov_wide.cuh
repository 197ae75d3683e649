// SPDX-License-Identifier: Apache-2.0
//
// Arnoldi step for restarts above 32 (the reference's KrylovConfig default
// is restart = 60, include/fsi/krylov.hpp:43, config.hpp:61). Same CGS2
// orthogonalisation as the register path of krylov.cuh (w -= V h1, w -= V h2,
// h_{j+1,j} = sqrt(||w||^2 - ||h2||^2), Givens on device), but the basis is
// walked in chunks of 32 vectors so any nv <= kMaxRestart fits the per-thread
// registers: five kernels per step instead of three.
//   W1 k_wide_spmv     : w = diag(scale) A z_j, Z[j] = z_j
//   W2 k_wide_dots<0>  : per-(chunk, CTA) partials of V^T w
//   W3 k_wide_update   : h1 = fixed-order sum of W2's partials (every CTA);
//                        w -= V h1
//   W4 k_wide_dots<1>  : partials of V^T w and ||w||^2
//   W5 k_wide_normalize: h2, ||w||^2 from W4 (every CTA); hn; row CTAs
//                        w -= V h2, v_{j+1} = w / hn, u = v_{j+1} / scale; the
//                        extra last CTA runs the Givens step (+ WHILE flag)
// Partials: partialw[(chunk * parts_w + cta) * kPartLd + v % 32]; W4's norm
// sits at slot min(32, nv) of chunk 0. Every sum runs in CTA order, so the
// history is bit-reproducible run to run.
#pragma once

#include "krylov.cuh"

namespace fsigpu {

constexpr int kWideThreads = 256;

__global__ void __launch_bounds__(kWideThreads) k_wide_spmv(KBufs k) {
  pdl_trigger();
  pdl_wait();
  const int j = k.st->j;
  constexpr int LPR = 8, RPC = kWideThreads / LPR;
  const int t = threadIdx.x;
  for (int r0 = blockIdx.x * RPC; r0 < k.n; r0 += gridDim.x * RPC) {
    const int row = r0 + t / LPR;
    const bool ok = row < k.n;
    const bool head = ok && (t & (LPR - 1)) == 0;
    const double sc = head ? k.scale[row] : 0.0;
    const double s = fused_row<LPR>(k, ok ? row : -1, t & (LPR - 1));
    if (head) k.w[row] = sc * s;
  }
  double* __restrict__ zj = k.Z + (size_t)j * k.n;
  for (int r = blockIdx.x * blockDim.x + t; r < k.n; r += gridDim.x * blockDim.x) zj[r] = k.zbuf[r];
}

// grid = (parts_w, ceil(mr / 32)); CTAs of chunks past nv exit.
template <bool NORM>
__global__ void __launch_bounds__(kWideThreads) k_wide_dots(KBufs k) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sm[kPartLd * (kWideThreads / 32)];
  const int nv = k.st->j + 1;
  const int c0 = blockIdx.y * kRegRestart;
  if (c0 >= nv) return;
  const int cn = min(kRegRestart, nv - c0);
  const bool with_norm = NORM && blockIdx.y == 0;
  double acc[kRegRestart];
#pragma unroll
  for (int v = 0; v < kRegRestart; ++v) acc[v] = 0.0;
  double n2 = 0.0;
  const double* __restrict__ V = k.V + (size_t)c0 * k.n;
  const double* __restrict__ W = k.w;
  const size_t n = (size_t)k.n;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k.n; r += gridDim.x * blockDim.x) {
    double vr[kRegRestart];
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v) vr[v] = v < cn ? __ldg(V + (size_t)v * n + r) : 0.0;
    const double wr = W[r];
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v)
      if (v < cn) acc[v] = fma(vr[v], wr, acc[v]);
    if (with_norm) n2 = fma(wr, wr, n2);
  }
  cta_reduce_t32<kWideThreads>(acc, n2, cn, sm,
                               k.partialw + ((size_t)blockIdx.y * k.parts_w + blockIdx.x) * kPartLd);
}

// hs[v] = sum over the parts_w CTAs (in CTA order) of value v, v < nv
__device__ __forceinline__ void wide_sum(const KBufs& k, int nv, double* hs) {
  const int P = k.parts_w;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    const double* p = k.partialw + (size_t)(v / kRegRestart) * P * kPartLd + (v % kRegRestart);
    double s = 0.0;
    constexpr int U = 8;
    for (int b0 = 0; b0 < P; b0 += U) {
      double pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) pv[u] = b0 + u < P ? __ldcg(p + (size_t)(b0 + u) * kPartLd) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) s += pv[u];
    }
    hs[v] = s;
  }
}

// w -= V h over all nv basis vectors, chunk by chunk (row r, value wr)
__device__ __forceinline__ double wide_sub(const KBufs& k, const double* hs, int nv, int r, double wr) {
  const size_t n = (size_t)k.n;
  for (int c0 = 0; c0 < nv; c0 += kRegRestart) {
    double vr[kRegRestart];
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v) vr[v] = c0 + v < nv ? __ldg(k.V + (size_t)(c0 + v) * n + r) : 0.0;
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v)
      if (c0 + v < nv) wr = fma(-hs[c0 + v], vr[v], wr);
  }
  return wr;
}

__global__ void __launch_bounds__(kWideThreads) k_wide_update(KBufs k) {
  pdl_trigger();
  pdl_wait();
  __shared__ double hs[kMaxRestart + 1];
  const int j = k.st->j;
  const int nv = j + 1;
  wide_sum(k, nv, hs);
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int v = threadIdx.x; v < nv; v += blockDim.x) k.st->h1[v] = hs[v];
    if (threadIdx.x == 0) k.st->jc = j + 1;
  }
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k.n; r += gridDim.x * blockDim.x)
    k.w[r] = wide_sub(k, hs, nv, r, k.w[r]);
}

// grid = parts_w + 1 (the last CTA runs the Givens step)
__global__ void __launch_bounds__(kWideThreads) k_wide_normalize(KBufs k) {
  pdl_trigger();
  pdl_wait();
  __shared__ double hs[kMaxRestart + 1];
  __shared__ double g_col[kMaxRestart + 2], g_cs[kMaxRestart + 1], g_sn[kMaxRestart + 1];
  __shared__ double s_hn, s_gj;
  const int jn = k.st->jc;  // = j + 1; st->j itself is advanced by the Givens CTA
  const int nv = jn;
  const int nb = gridDim.x - 1;
  const bool rows_cta = blockIdx.x < nb;
  const int t = threadIdx.x;
  wide_sum(k, nv, hs);
  if (t == 0) {
    // ||w||^2: chunk 0, slot min(32, nv), CTA order
    const double* p = k.partialw + min(kRegRestart, nv);
    double s = 0.0;
    for (int b = 0; b < k.parts_w; ++b) s += __ldcg(p + (size_t)b * kPartLd);
    hs[kMaxRestart] = s;
  }
  __syncthreads();
  if (t < 32) {
    double q = 0.0;
    for (int v = t; v < nv; v += 32) q = fma(hs[v], hs[v], q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(kFull, q, o);
    if (t == 0) s_hn = sqrt(fmax(hs[kMaxRestart] - q, 0.0));
  }
  __syncthreads();
  const double hn = s_hn;
  if (!rows_cta) {
    for (int v = t; v < nv; v += blockDim.x) {
      k.st->h2[v] = hs[v];
      g_col[v] = __ldcg(k.st->h1 + v) + hs[v];
    }
    for (int v = t; v < nv - 1; v += blockDim.x) {
      g_cs[v] = __ldcg(k.cs + v);
      g_sn[v] = __ldcg(k.sn + v);
    }
    if (t == 0) s_gj = __ldcg(k.g + nv - 1);
    __syncthreads();
    givens_core(k, nv - 1, hn, g_col, g_cs, g_sn, s_gj, givens_prefetch(k));
    return;
  }
  const bool lucky = hn < 1e-14;
  double* __restrict__ VJ = k.V + (size_t)jn * k.n;
  for (int r = blockIdx.x * blockDim.x + t; r < k.n; r += nb * blockDim.x) {
    const double wr = wide_sub(k, hs, nv, r, k.w[r]);
    if (!lucky) {
      const double vv = wr / hn;
      VJ[r] = vv;
      k.ubuf[r] = vv / k.scale[r];
    }
  }
}

}  // namespace fsigpu
