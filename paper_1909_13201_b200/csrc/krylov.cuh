// SPDX-License-Identifier: Apache-2.0
//
// Device-resident FGMRES(m) Arnoldi kernels (reference: gmres,
// proj/src/krylov.cpp:20-126).
//
// One Arnoldi step after the V-cycle (z_j = M v_j) and the scaled SpMV
// (w = A_s z_j) is three row-parallel passes plus a normalisation:
//   k_dots        : h1 = V_{0..j}^T w           (+ copy z_j into Z[j])
//   k_update_dots : w -= V h1 ; h2 = V^T w      (classical Gram-Schmidt, 2nd pass)
//   k_update_norm : w -= V h2 ; ||w||, then on device: H(:,j) = h1+h2,
//                   Givens rotations, rho = |g_{j+1}|, stop flags
//   k_normalize   : v_{j+1} = w / h_{j+1,j} ; u = v_{j+1} / frame_scale
// Each reduction is two-stage with a fixed order (per-CTA partials, the
// last CTA to arrive sums them in CTA order), so the iteration history is
// bit-reproducible run to run. All step parameters (j, its) live in device
// memory so one captured graph serves every step.
#pragma once

#include "common.cuh"

namespace fsigpu {

constexpr int kRegRestart = 32;   // restart <= 32: the V_{0..j} dots of a row held in registers
constexpr int kMaxRestart = 128;  // larger restarts (the reference default is 60) take the
                                  // chunked path of krylov_wide.cuh
constexpr int kPartLd = kRegRestart + 1;  // row stride of the per-CTA partial-dot buffers
constexpr int kKThreads = 128;

struct KState {
  int j;          // columns done in this cycle
  int its;        // Arnoldi steps done in total
  int stop;       // inner loop must stop (rho <= target or lucky)
  int breakdown;  // lucky breakdown seen (krylov.cpp:74-77)
  int max_iters;
  int restart;
  int first;      // next norm is ||r0||
  int converged;
  int keep_going; // cycle-level continue flag (host side)
  int jc;         // Krylov column k_update_normalize writes (set by k_update_dots_norm)
  double target;
  double beta;
  double rho;
  double hn;
  double rel_tol, abs_tol;
  double h1[kMaxRestart + 1];
  double h2[kMaxRestart + 1];
  double y[kMaxRestart + 1];
};

struct KBufs {
  int n;
  int mr;
  const double* scale;  // frame_scale
  double* V;            // (mr+1) x n
  double* Z;            // mr x n
  double* w;            // n
  double* zbuf;         // V-cycle output
  double* ubuf;         // V-cycle input (v_j / scale)
  double* r;            // residual
  double* x;            // iterate
  const double* b;      // rhs
  double* H;            // (mr+1) x mr, row-major H(i,j) = H[i*mr+j]
  double* cs;
  double* sn;
  double* g;
  double* history;      // max_iters + 2
  double* partial;      // grid x (kRegRestart+1)
  double* partial2;     // second partial buffer of the fused Arnoldi step
  int parts_a;          // CTAs of k_spmv_dots (rows of partial it writes)
  int fuse_small;       // large n: (A) runs as SpMV + k_dots_copy
  int parts_b;          // CTAs of k_update_dots_norm (rows of partial2)
  int parts_c;          // row CTAs of k_update_normalize (+1 Givens CTA)
  double* partialw;     // restart > 32 (krylov_wide.cuh): chunks x parts_w x kPartLd
  int parts_w;          // row CTAs of the wide-path kernels
  unsigned int* ticket;
  KState* st;
  // fused Arnoldi (3 kernels per step)
  const int* a_ptr;            // top-level CSR (outer operator A_s = diag(scale) A)
  const int* a_idx;
  const double* a_val;
  int a_lpr;
  cudaGraphConditionalHandle cond;  // WHILE handle of the restart-cycle graph
  unsigned long long* stamp;        // device-clock stamps of (A), (B), (C): 3 slots of 4 u64, or null
  int use_cond;
};

// Block-level sums of NV per-thread accumulators -> out[v] (v < nv): the
// accumulators are transposed through shared memory (sm: NV * kKThreads
// doubles) and warp w sums vectors v = w, w + NW, ... (lanes stride the
// threads, fixed xor tree): one shuffle tree per vector instead of one per
// vector per warp.
template <int NV>
__device__ __forceinline__ void block_reduce_vec(double (&acc)[NV], int nv, double* sm, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kKThreads / 32;
#pragma unroll
  for (int v = 0; v < NV; ++v)
    if (v < nv) sm[v * kKThreads + threadIdx.x] = acc[v];
  __syncthreads();
  for (int v = warp; v < nv; v += NW) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kKThreads / 32; ++q) s += sm[v * kKThreads + q * 32 + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) out[v] = s;
  }
}

// Last-CTA detection; returns true in every thread of the last CTA.
// bar.sync orders the CTA's partial writes before thread 0's gpu-scope
// fence + arrival (cumulativity), so one fenced thread suffices (a fence in
// every thread showed up as the top ERRBAR stall in ncu).
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const bool last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    if (last) __threadfence();
    s_last = last;
  }
  __syncthreads();
  return s_last;
}

// Sum of the per-CTA partials, fixed order: warp w reduces vectors
// v = w, w+NW, ...; lanes stride over CTAs, then a fixed xor tree.
__device__ __forceinline__ void finish_sum(const KBufs& k, int nv, double* dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kKThreads / 32;
  for (int v = warp; v < nv; v += NW) {
    double s = 0.0;
    constexpr int U = 8;  // predicated load batches (no per-load exits)
    for (unsigned int b0 = lane; b0 < gridDim.x; b0 += 32 * U) {
      double pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned int b = b0 + 32 * u;
        pv[u] = b < gridDim.x ? __ldcg(k.partial + (size_t)b * kPartLd + v) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) s += pv[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) dst[v] = s;
  }
  if (threadIdx.x == 0) *k.ticket = 0;
}

// Givens update of column j on device (krylov.cpp:79-100), staged in
// shared memory by the whole CTA; one thread runs the recurrence. With
// use_cond, also sets the restart-cycle WHILE condition. Core: col[0..j]
// already holds H(:,j) = h1 + h2, cs/sn[0..j) the previous rotations and
// gj = g[j]; all in shared memory / registers (loaded by the caller).
// pre: the solve state's scalars (its, max_iters, target), loaded by the
// caller before its reduction so their L2 round trip is off the chain.
struct GivensPre {
  int its, max_iters;
  double target;
};
__device__ __forceinline__ GivensPre givens_prefetch(const KBufs& k) {
  GivensPre p;
  p.its = __ldcg(&k.st->its);
  p.max_iters = __ldcg(&k.st->max_iters);
  p.target = __ldcg(&k.st->target);
  return p;
}
__device__ void givens_core(const KBufs& k, int j, double hn, double* col, double* cs, double* sn, double gj,
                            GivensPre pre) {
  KState* st = k.st;
  const int mr = k.mr;
  const int t = threadIdx.x;
  int stop = 0;
  if (t == 0) {
    col[j + 1] = hn;
    int lucky = 0;
    if (hn < 1e-14) {
      st->breakdown = 1;
      lucky = 1;
    }
    // the running element stays in a register: the dependent chain is two
    // flops per rotation, the shared-memory traffic is off it
    double carry = col[0];
#pragma unroll 4
    for (int i = 0; i < j; ++i) {
      const double nxt = col[i + 1], c = cs[i], sg = sn[i];
      col[i] = c * carry + sg * nxt;
      carry = -sg * carry + c * nxt;
    }
    const double denom = hypot(carry, hn);
    const double c = carry / denom, sj = hn / denom;
    col[j] = denom;
    col[j + 1] = 0.0;
    k.g[j + 1] = -sj * gj;
    k.g[j] = c * gj;
    const double rho = fabs(-sj * gj);
    st->its = pre.its + 1;
    st->rho = rho;
    st->hn = hn;
    k.history[pre.its + 1] = rho;
    stop = (rho <= pre.target || lucky) ? 1 : 0;
    st->stop = stop;
    k.cs[j] = c;
    k.sn[j] = sj;
  }
  __syncthreads();
  for (int i = t; i <= j + 1; i += blockDim.x) k.H[i * mr + j] = col[i];
  if (t == 0) {
    st->j = j + 1;
    if (k.use_cond) {
      const int go = (!stop && j + 1 < mr && pre.its + 1 < pre.max_iters) ? 1 : 0;
      cudaGraphSetConditional(k.cond, go);
    }
  }
}

// ||r|| -> beta; on the first call also r0, history[0] and target.
__global__ void __launch_bounds__(kKThreads) k_norm_r(KBufs k) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sm[kKThreads];
  double acc[1] = {0.0};
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k.n; r += gridDim.x * blockDim.x)
    acc[0] = fma(k.r[r], k.r[r], acc[0]);
  block_reduce_vec<1>(acc, 1, sm, k.partial + (size_t)blockIdx.x * kPartLd);
  if (last_block(k.ticket)) {
    __shared__ double s_n2;
    finish_sum(k, 1, &s_n2);
    __syncthreads();
    if (threadIdx.x == 0) {
      KState* st = k.st;
      const double beta = sqrt(s_n2);
      st->beta = beta;
      if (st->first) {
        st->first = 0;
        k.history[0] = beta;
        st->target = fmax(st->rel_tol * beta, st->abs_tol);
      }
      st->converged = beta <= st->target ? 1 : 0;
      // start of a cycle: g = (beta, 0, ...), j = 0 (krylov.cpp:55-58)
      for (int i = 0; i <= k.mr; ++i) k.g[i] = 0.0;
      k.g[0] = beta;
      st->j = 0;
      st->stop = 0;
    }
  }
}

// v_0 = r / beta ; u = v_0 / scale
__global__ void k_cycle_start(KBufs k) {
  pdl_trigger();
  pdl_wait();
  const double beta = k.st->beta;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k.n; r += gridDim.x * blockDim.x) {
    const double v = k.r[r] / beta;
    k.V[r] = v;
    k.ubuf[r] = v / k.scale[r];
  }
}

// y = H^{-1} g (back substitution, krylov.cpp:103-109): H (j <= 32) staged
// in shared memory, one thread runs the recurrence; wider restarts read H
// from global memory (once per restart cycle, off the per-step path).
__global__ void k_solve_y(KBufs k) {
  pdl_trigger();
  pdl_wait();
  __shared__ double Hs[kRegRestart * kRegRestart];
  __shared__ double gs[kMaxRestart + 1];
  __shared__ double y[kMaxRestart];
  KState* st = k.st;
  const int j = st->j;
  const int mr = k.mr;
  const bool staged = j <= kRegRestart;
  if (staged)
    for (int e = threadIdx.x; e < j * j; e += blockDim.x) Hs[e] = k.H[(e / j) * mr + (e % j)];
  for (int i = threadIdx.x; i < j; i += blockDim.x) gs[i] = k.g[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = j - 1; i >= 0; --i) {
      double s = gs[i];
      if (staged) {
        for (int q = i + 1; q < j; ++q) s -= Hs[i * j + q] * y[q];
        y[i] = s / Hs[i * j + i];
      } else {
        const double* Hi = k.H + (size_t)i * mr;
        for (int q = i + 1; q < j; ++q) s -= __ldcg(Hi + q) * y[q];
        y[i] = s / __ldcg(Hi + i);
      }
    }
    for (int i = 0; i < j; ++i) st->y[i] = y[i];
  }
}

// x += Z y  (FGMRES: M(V y) = Z y for the fixed linear V-cycle)
__global__ void k_update_x(KBufs k) {
  pdl_trigger();
  pdl_wait();
  const KState* st = k.st;
  const int j = st->j;
  __shared__ double ys[kMaxRestart];
  for (int i = threadIdx.x; i < j; i += blockDim.x) ys[i] = st->y[i];
  __syncthreads();
  // all loads of a row's 32-column chunk issued before its FMA chain
  // (predicated batch; a runtime-bound loop left one DRAM latency per term)
  const double* __restrict__ Z = k.Z;
  double* __restrict__ X = k.x;
  const size_t n = (size_t)k.n;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k.n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c0 = 0; c0 < j; c0 += kRegRestart) {
      double z[kRegRestart];
#pragma unroll
      for (int i = 0; i < kRegRestart; ++i) z[i] = c0 + i < j ? __ldg(Z + (size_t)(c0 + i) * n + r) : 0.0;
#pragma unroll
      for (int i = 0; i < kRegRestart; ++i)
        if (c0 + i < j) s = fma(ys[c0 + i], z[i], s);
    }
    X[r] += s;
  }
}

}  // namespace fsigpu

namespace fsigpu {
// ---- fused Arnoldi step (3 kernels): -----------------------------------
// (A) w = diag(scale) A z_j and h1 = V^T w in one pass: a CTA owns 64 rows,
//     computes them with LPR-lane CSR rows, keeps w in shared memory and
//     forms its partial dots (Z[j] = zbuf copied on the way).
constexpr int kFuseThreads = 1024;
constexpr int kFuseRows = 128;  // rows per CTA of k_spmv_dots (one pass at LPR = 8)
constexpr int kArnThreads = 128;  // CTA size of the fused update kernels
template <int LPR>
__device__ __forceinline__ double fused_row(const KBufs& k, int row, int lane) {
  const int k0 = row >= 0 ? __ldg(k.a_ptr + row) : 0, k1 = row >= 0 ? __ldg(k.a_ptr + row + 1) : 0;
  double s = 0.0;
  constexpr int U = 8;
  for (int kb = k0 + lane; kb < k1; kb += U * LPR) {
    int c[U];
    double v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * LPR;
      const bool ok = kk < k1;
      c[u] = ok ? __ldg(k.a_idx + kk) : -1;
      v[u] = ok ? __ldg(k.a_val + kk) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? k.zbuf[c[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(v[u], xv[u], s);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  return s;
}

// Small systems: one 128-row tile per CTA (no tile loop), as first tuned
// on config 0.
template <int LPR>
__global__ void __launch_bounds__(kFuseThreads) k_spmv_dots_1(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 0 : nullptr);
  static_assert(kFuseThreads / LPR >= kFuseRows, "one row pass per CTA");
  pdl_trigger();
  __shared__ double ws[kFuseRows];
  const int r0 = blockIdx.x * kFuseRows;
  const int t = threadIdx.x;
  // setup data first (the outer operator's row and its first batch, the
  // frame scale: never written by the solve), so under programmatic
  // dependent launch it overlaps the V-cycle's last kernel
  const int rl = t / LPR, ln = t & (LPR - 1);
  const int row = r0 + rl;
  const bool ok = rl < kFuseRows && row < k.n;
  const bool head = ok && ln == 0;
  const double sc = head ? __ldg(k.scale + row) : 0.0;
  constexpr int U = 8;
  const int k0 = ok ? __ldg(k.a_ptr + row) : 0, k1 = ok ? __ldg(k.a_ptr + row + 1) : 0;
  int c[U];
  double av[U];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = kb + u * LPR;
      c[u] = kk < k1 ? __ldg(k.a_idx + kk) : -1;
      av[u] = kk < k1 ? __ldg(k.a_val + kk) : 0.0;
    }
  };
  load(k0 + ln);
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 0 : nullptr);
  const int j = k.st->j;
  const int nv = j + 1;
  // operands that do not depend on w are loaded before the SpMV so their
  // latency overlaps it: the V entries of the partial dots (warp v, lanes
  // over the CTA's 128 rows, 4 each) and z_j for the copy into Z[j]
  const int v = t >> 5, lane = t & 31;
  double vv[kFuseRows / 32];
#pragma unroll
  for (int q = 0; q < kFuseRows / 32; ++q) {
    const int rr = r0 + lane + 32 * q;
    vv[q] = (v < nv && rr < k.n) ? k.V[(size_t)v * k.n + rr] : 0.0;
  }
  const bool zc = t < kFuseRows && r0 + t < k.n;
  const double zj = zc ? k.zbuf[r0 + t] : 0.0;
  {
    double s = 0.0;
    for (int kb = k0 + ln; kb < k1; kb += U * LPR) {
      double xv[U], vc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xv[u] = c[u] >= 0 ? k.zbuf[c[u]] : 0.0;
        vc[u] = av[u];
      }
      if (kb + U * LPR < k1) load(kb + U * LPR);
#pragma unroll
      for (int u = 0; u < U; ++u) s = fma(vc[u], xv[u], s);
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
    if (head) {
      const double w = sc * s;
      k.w[row] = w;
      ws[rl] = w;
    }
  }
  if (zc) k.Z[(size_t)j * k.n + r0 + t] = zj;
  if (t < kFuseRows && r0 + t >= k.n) ws[t] = 0.0;
  __syncthreads();
  double s = 0.0;
  if (v < nv) {
#pragma unroll
    for (int q = 0; q < kFuseRows / 32; ++q) s = fma(vv[q], ws[lane + 32 * q], s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0 && v < nv) k.partial[(size_t)blockIdx.x * kPartLd + v] = s;
  stamp_end(k.stamp ? k.stamp + 0 : nullptr);
}

// Grid-stride over 128-row tiles with the grid capped at the resident CTA
// count (k.parts_a): the partial-dot rows the consumers sum stay <= 2 per
// SM however large n is (on the 1.25M-dof config-2 fine level a CTA per
// tile left 9,761 partials that every CTA of (B) summed, ~1 MB each).
template <int LPR>
__global__ void __launch_bounds__(kFuseThreads) k_spmv_dots(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 0 : nullptr);
  pdl_trigger();
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 0 : nullptr);
  __shared__ double ws[kFuseRows];
  const int j = k.st->j;
  const int nv = j + 1;
  const int t = threadIdx.x;
  const int v = t >> 5, lane = t & 31;
  const int ntiles = (k.n + kFuseRows - 1) / kFuseRows;
  double s = 0.0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int r0 = tile * kFuseRows;
    // operands that do not depend on w are loaded before the SpMV so their
    // latency overlaps it: the V entries of the partial dots (warp v, lanes
    // over the tile's 128 rows, 4 each) and z_j for the copy into Z[j]
    double vv[kFuseRows / 32];
#pragma unroll
    for (int q = 0; q < kFuseRows / 32; ++q) {
      const int row = r0 + lane + 32 * q;
      vv[q] = (v < nv && row < k.n) ? k.V[(size_t)v * k.n + row] : 0.0;
    }
    const bool zc = t < kFuseRows && r0 + t < k.n;
    const double zj = zc ? k.zbuf[r0 + t] : 0.0;
    constexpr int RPP = kFuseThreads / LPR;  // rows per pass
    for (int p = 0; p < kFuseRows; p += RPP) {
      const int rl = p + t / LPR;
      const int row = r0 + rl;
      const bool ok = rl < kFuseRows && row < k.n;
      const bool head = ok && (t & (LPR - 1)) == 0;
      const double sc = head ? k.scale[row] : 0.0;
      const double sr = fused_row<LPR>(k, ok ? row : -1, t & (LPR - 1));
      if (head) {
        const double w = sc * sr;
        k.w[row] = w;
        ws[rl] = w;
      }
    }
    if (zc) k.Z[(size_t)j * k.n + r0 + t] = zj;
    if (t < kFuseRows && r0 + t >= k.n) ws[t] = 0.0;
    __syncthreads();
    if (v < nv) {
#pragma unroll
      for (int q = 0; q < kFuseRows / 32; ++q) s = fma(vv[q], ws[lane + 32 * q], s);
    }
    __syncthreads();  // ws is rewritten by the next tile
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0 && v < nv) k.partial[(size_t)blockIdx.x * kPartLd + v] = s;
  stamp_end(k.stamp ? k.stamp + 0 : nullptr);
}

// Per-CTA sums of 32 per-thread values plus one extra: a butterfly
// transpose-reduction gives lane L of every warp its warp's total of value
// L in 31 shuffles (16+8+4+2+1) instead of 32 separate 5-level trees; warp
// totals are then added in warp order. out[0..nv) = sums, out[nv] = extra.
template <int T>
__device__ __forceinline__ void cta_reduce_t32(double (&a)[32], double extra, int nv, double* sm, double* out) {
  constexpr int NW = T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const bool up = lane & w;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const double send = up ? a[i] : a[i + w];
      const double keep = up ? a[i + w] : a[i];
      a[i] = keep + __shfl_xor_sync(kFull, send, w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) extra += __shfl_xor_sync(kFull, extra, o);
  sm[warp * 33 + lane] = a[0];
  if (lane == 0) sm[warp * 33 + 32] = extra;
  __syncthreads();
  if (threadIdx.x <= nv) {
    const int v = threadIdx.x < nv ? threadIdx.x : 32;
    double s = 0.0;
    for (int i = 0; i < NW; ++i) s += sm[i * 33 + v];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Fixed-order sum of `nparts` per-CTA partial rows (row stride
// kRegRestart+1) for values 0..nv-1 (nv <= kRegRestart+1) into dst[]:
// lanes own values, warps own CTA slices, slices added in order. Every CTA
// of the consumer kernel runs it on the producer's partials, so no CTA of
// the producer has to finish the reduction (no last-CTA tail).
// U: loads per thread per round. Small systems (one row per thread, ~160
// partial rows, 4 slices at nv = 31) take U = 40 so the whole sum is ONE L2
// round trip: with U = 10 its four dependent rounds were ~3 us of the 4 us
// of (B) and of the 8 us of (C) on config 0 (device-clock stamps).
constexpr int kSumSlices = 16;
template <int T, int U = 10>
__device__ __forceinline__ void sum_partials(const double* __restrict__ part, int nparts, int nv, double* dst,
                                             double* red /* kSumSlices x (kRegRestart+1) */) {
  constexpr int LD = kRegRestart + 1;
  // thread t -> value t % nv of CTA slice t / nv (ns slices, fixed for a
  // given nv, so the summation order is deterministic)
  const int ns = min(kSumSlices, T / nv);
  const int v = threadIdx.x % nv, q = threadIdx.x / nv;
  if (q < ns) {
    double s = 0.0;
    for (int b0 = q; b0 < nparts; b0 += ns * U) {
      double pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + ns * u;
        pv[u] = b < nparts ? __ldcg(part + (size_t)b * LD + v) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) s += pv[u];
    }
    red[q * LD + v] = s;
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nv; w += T) {
    double z = 0.0;
    for (int i = 0; i < ns; ++i) z += red[i * LD + w];
    dst[w] = z;
  }
  __syncthreads();
}

// Large systems run (A) as two launches: the outer SpMV through the level
// operator's own kernel (bsr22_kernel when A is held as 2 x 2 blocks, else the
// CSR kernels) with the w = diag(s) A z epilogue, then this kernel: the
// partials of h1 = V^T w in (A)'s layout, and Z[j] = z_j. The fused large-n
// kernel it replaced (256-thread CTAs on 32-row tiles with the row loop inside)
// ran at 246 us on config 2 against 145 + 43 us, and at 115 us on the 3D
// system against 88 + 12 us. Rows grid-stride.
constexpr int kDotsThreads = 256;
// NV: compile-time bound on the vectors; RP rows per thread per pass, so a
// thread keeps NV x RP loads in flight whatever the Krylov column (with one
// row per thread the first columns of a cycle move a few bytes per thread
// and the kernel ran at 3.1 TB/s on config 2).
template <int NV, int RP>
__device__ __forceinline__ void dots_copy_rows(const KBufs& k, int nv, int j, double (&acc)[kRegRestart]) {
  const double* __restrict__ V = k.V;
  const double* __restrict__ W = k.w;
  const double* __restrict__ Zb = k.zbuf;
  double* __restrict__ zj = k.Z + (size_t)j * k.n;
  const size_t n = (size_t)k.n;
  const int stride = gridDim.x * blockDim.x;
  for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < k.n; r0 += RP * stride) {
    double vr[RP][NV], wr[RP], zr[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      const bool in = r < k.n;
#pragma unroll
      for (int v = 0; v < NV; ++v) vr[q][v] = (in && v < nv) ? __ldg(V + (size_t)v * n + r) : 0.0;
      wr[q] = in ? W[r] : 0.0;
      zr[q] = in ? Zb[r] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      if (r < k.n) zj[r] = zr[q];
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = fma(vr[q][v], wr[q], acc[v]);
    }
  }
}
__global__ void __launch_bounds__(kDotsThreads) k_dots_copy(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 0 : nullptr);
  pdl_trigger();
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 0 : nullptr);
  __shared__ double sm[kPartLd * (kDotsThreads / 32)];
  const int j = k.st->j;
  const int nv = j + 1;
  double acc[kRegRestart];
#pragma unroll
  for (int v = 0; v < kRegRestart; ++v) acc[v] = 0.0;
  if (nv <= 4) dots_copy_rows<4, 8>(k, nv, j, acc);
  else if (nv <= 8) dots_copy_rows<8, 4>(k, nv, j, acc);
  else if (nv <= 16) dots_copy_rows<16, 2>(k, nv, j, acc);
  else dots_copy_rows<kRegRestart, 1>(k, nv, j, acc);
  cta_reduce_t32<kDotsThreads>(acc, 0.0, nv, sm, k.partial + (size_t)blockIdx.x * kPartLd);
  stamp_end(k.stamp ? k.stamp + 0 : nullptr);
}

// (B) h1 = sum of (A)'s partials (every CTA); w -= V h1 ; partial2 <- V^T w
//     and ||w||^2 (h2 and the norm are finished by the CTAs of (C)).
// PF: the first row's operands are loaded before the h1 reduction (small
// systems, one row per thread); large systems skip it: the row loop alone
// streams every row, and the 64 freed registers double the resident warps.
template <bool PF>
__global__ void __launch_bounds__(kArnThreads) k_update_dots_norm(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 4 : nullptr);
  pdl_trigger();
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 4 : nullptr);
  __shared__ double sm[kPartLd * (kArnThreads / 32)];
  __shared__ double hs[kRegRestart + 1];
  __shared__ double red[kPartLd * kSumSlices];
  const int j = k.st->j;
  const int nv = j + 1;
  // this thread's first row is loaded before the h1 reduction (independent
  // of it), so the two latencies overlap
  const int r0 = blockIdx.x * blockDim.x + threadIdx.x;
  double w0 = 0.0, v0[PF ? kRegRestart : 1];
  if constexpr (PF) {
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v) v0[v] = (r0 < k.n && v < nv) ? k.V[(size_t)v * k.n + r0] : 0.0;
    if (r0 < k.n) w0 = k.w[r0];
  }
  sum_partials<kArnThreads, PF ? 40 : 10>(k.partial, k.parts_a, nv, hs, red);
  if (blockIdx.x == 0) {
    if (threadIdx.x < nv) k.st->h1[threadIdx.x] = hs[threadIdx.x];
    if (threadIdx.x == 0) k.st->jc = j + 1;
  }
  double acc[kRegRestart];
#pragma unroll
  for (int v = 0; v < kRegRestart; ++v) acc[v] = 0.0;
  double n2 = 0.0;
  if (PF && r0 < k.n) {
    double wr = w0;
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v)
      if (v < nv) wr = fma(-hs[v], v0[PF ? v : 0], wr);
    k.w[r0] = wr;
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v)
      if (v < nv) acc[v] = fma(v0[PF ? v : 0], wr, acc[v]);
    n2 = fma(wr, wr, n2);
  }
  if constexpr (PF) {
    for (int r = r0 + gridDim.x * blockDim.x; r < k.n; r += gridDim.x * blockDim.x) {
      double wr = k.w[r];
  #pragma unroll
      for (int v = 0; v < kRegRestart; ++v)
        if (v < nv) wr = fma(-hs[v], k.V[(size_t)v * k.n + r], wr);
      k.w[r] = wr;
  #pragma unroll
      for (int v = 0; v < kRegRestart; ++v)
        if (v < nv) acc[v] = fma(k.V[(size_t)v * k.n + r], wr, acc[v]);  // L1 hits
      n2 = fma(wr, wr, n2);
    }
  } else {
    // restrict-qualified views: w's store does not alias V, so the next
    // row's loads may be issued before this row's store
    const double* __restrict__ V = k.V;
    double* __restrict__ W = k.w;
    const size_t n = (size_t)k.n;
    for (int r = PF ? r0 + gridDim.x * blockDim.x : r0; r < k.n; r += gridDim.x * blockDim.x) {
      double vr[kRegRestart];
#pragma unroll
      for (int v = 0; v < kRegRestart; ++v) vr[v] = v < nv ? __ldg(V + (size_t)v * n + r) : 0.0;
      double wr = W[r];
#pragma unroll
      for (int v = 0; v < kRegRestart; ++v)
        if (v < nv) wr = fma(-hs[v], vr[v], wr);
      W[r] = wr;
#pragma unroll
      for (int v = 0; v < kRegRestart; ++v)
        if (v < nv) acc[v] = fma(vr[v], wr, acc[v]);
      n2 = fma(wr, wr, n2);
    }
  }
  // partial2[cta][0..nv) = h2 dots, partial2[cta][nv] = ||w||^2
  static_assert(kRegRestart == 32, "cta_reduce_t32 holds one slot per Krylov vector");
  cta_reduce_t32<kArnThreads>(acc, n2, nv, sm, k.partial2 + (size_t)blockIdx.x * kPartLd);
  stamp_end(k.stamp ? k.stamp + 4 : nullptr);
}

// Large-n (B) with NV x RP loads in flight per thread (see dots_copy_rows):
// RP rows per thread per pass, each row's operands in registers. It replaced a
// cp.async-staged variant with one row in flight ahead (config 2 in-graph: 62 ->
// 41 us = 4.3 TB/s; (C) with the same row loop 62 -> 44 us).
template <int NV, int RP>
__device__ __forceinline__ void update_dots_rows(const KBufs& k, int nv, const double* hs,
                                                 double (&acc)[kRegRestart], double& n2) {
  const double* __restrict__ V = k.V;
  double* __restrict__ W = k.w;
  const size_t n = (size_t)k.n;
  const int stride = gridDim.x * blockDim.x;
  for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < k.n; r0 += RP * stride) {
    double vr[RP][NV], wr[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      const bool in = r < k.n;
#pragma unroll
      for (int v = 0; v < NV; ++v) vr[q][v] = (in && v < nv) ? __ldg(V + (size_t)v * n + r) : 0.0;
      wr[q] = in ? W[r] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      double w1 = wr[q];
#pragma unroll
      for (int v = 0; v < NV; ++v) w1 = fma(-hs[v], vr[q][v], w1);  // hs[v] = 0 beyond nv
      if (r < k.n) W[r] = w1;
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = fma(vr[q][v], w1, acc[v]);
      n2 = fma(w1, w1, n2);
    }
  }
}
__global__ void __launch_bounds__(kArnThreads) k_update_dots_norm_mr(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 4 : nullptr);
  pdl_trigger();
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 4 : nullptr);
  __shared__ double sm[kPartLd * (kArnThreads / 32)];
  __shared__ double hs[kRegRestart + 1];
  __shared__ double red[kPartLd * kSumSlices];
  const int j = k.st->j;
  const int nv = j + 1;
  if (threadIdx.x <= kRegRestart) hs[threadIdx.x] = 0.0;
  __syncthreads();
  sum_partials<kArnThreads>(k.partial, k.parts_a, nv, hs, red);
  if (blockIdx.x == 0) {
    if (threadIdx.x < nv) k.st->h1[threadIdx.x] = hs[threadIdx.x];
    if (threadIdx.x == 0) k.st->jc = j + 1;
  }
  double acc[kRegRestart];
#pragma unroll
  for (int v = 0; v < kRegRestart; ++v) acc[v] = 0.0;
  double n2 = 0.0;
  if (nv <= 4) update_dots_rows<4, 8>(k, nv, hs, acc, n2);
  else if (nv <= 8) update_dots_rows<8, 4>(k, nv, hs, acc, n2);
  else if (nv <= 16) update_dots_rows<16, 2>(k, nv, hs, acc, n2);
  else update_dots_rows<kRegRestart, 1>(k, nv, hs, acc, n2);
  cta_reduce_t32<kArnThreads>(acc, n2, nv, sm, k.partial2 + (size_t)blockIdx.x * kPartLd);
  stamp_end(k.stamp ? k.stamp + 4 : nullptr);
}

// Row loop of the large-n (C) with NV x RP loads in flight per thread.
template <int NV, int RP>
__device__ __forceinline__ void normalize_rows(const KBufs& k, int nv, int nb, const double* hs, double hn,
                                               bool lucky, double* __restrict__ VJ) {
  const double* __restrict__ V = k.V;
  const double* __restrict__ W = k.w;
  const double* __restrict__ S = k.scale;
  double* __restrict__ UB = k.ubuf;
  const size_t n = (size_t)k.n;
  const int stride = nb * blockDim.x;
  for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < k.n; r0 += RP * stride) {
    double vr[RP][NV], wr[RP], sc[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      const bool in = r < k.n;
#pragma unroll
      for (int v = 0; v < NV; ++v) vr[q][v] = (in && v < nv) ? __ldg(V + (size_t)v * n + r) : 0.0;
      wr[q] = in ? W[r] : 0.0;
      sc[q] = in ? S[r] : 1.0;
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
      const int r = r0 + q * stride;
      double w1 = wr[q];
#pragma unroll
      for (int v = 0; v < NV; ++v) w1 = fma(-hs[v], vr[q][v], w1);
      if (r < k.n && !lucky) {
        const double vv = w1 / hn;
        VJ[r] = vv;
        UB[r] = vv / sc[q];
      }
    }
  }
}

// (C) every CTA sums (B)'s partials into h2 and ||w||^2 and forms
//     h_{j+1,j} = sqrt(||w||^2 - ||h2||^2) (the norm of w - V h2 for an
//     orthonormal V; h2 is the small second CGS correction). The LAST CTA
//     only runs the Givens step (and sets the CUDA-graph WHILE condition),
//     overlapping the others, which do w -= V h2 ; v_{j+1} = w / h_{j+1,j} ;
//     u = v_{j+1} / scale over the rows. Launched with one extra CTA.
template <bool PF>
__global__ void __launch_bounds__(kArnThreads) k_update_normalize(KBufs k) {
  stamp_fold(k.stamp ? k.stamp + 8 : nullptr);
  pdl_trigger();
  pdl_wait();
  stamp_start(k.stamp ? k.stamp + 8 : nullptr);
  __shared__ double hs[kRegRestart + 1];
  __shared__ double red[kPartLd * kSumSlices];
  __shared__ double s_hn;
  const int jn = k.st->jc;  // = j + 1; st->j itself is advanced by the Givens CTA
  const int nv = jn;
  const int nb = gridDim.x - 1;
  const bool rows_cta = blockIdx.x < nb;
  // Givens CTA: its inputs other than h2 are loaded before the reduction
  __shared__ double g_col[kRegRestart + 2], g_cs[kRegRestart + 1], g_sn[kRegRestart + 1];
  double h1t = 0.0, gj = 0.0;
  GivensPre gpre{};
  if (!rows_cta) {
    const int t = threadIdx.x;
    if (t < nv) h1t = __ldcg(k.st->h1 + t);
    if (t < nv - 1) {
      g_cs[t] = __ldcg(k.cs + t);
      g_sn[t] = __ldcg(k.sn + t);
    }
    if (t == 0) gj = __ldcg(k.g + nv - 1);
    if (t == 0) gpre = givens_prefetch(k);
  }
  // first row prefetched before the reduction (see k_update_dots_norm)
  const int r0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool has0 = rows_cta && r0 < k.n;
  double w0 = 0.0, sc0 = 1.0, v0[PF ? kRegRestart : 1];
  if constexpr (PF) {
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v) v0[v] = (has0 && v < nv) ? k.V[(size_t)v * k.n + r0] : 0.0;
    if (has0) {
      w0 = k.w[r0];
      sc0 = k.scale[r0];
    }
  }
  sum_partials<kArnThreads, PF ? 40 : 10>(k.partial2, k.parts_b, nv + 1, hs, red);
  if (threadIdx.x < 32) {
    double q = 0.0;
    for (int v = threadIdx.x; v < nv; v += 32) q = fma(hs[v], hs[v], q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(kFull, q, o);
    if (threadIdx.x == 0) s_hn = sqrt(fmax(hs[nv] - q, 0.0));
  }
  __syncthreads();
  const double hn = s_hn;
  if (!rows_cta) {
    if (threadIdx.x < nv) {
      k.st->h2[threadIdx.x] = hs[threadIdx.x];
      g_col[threadIdx.x] = h1t + hs[threadIdx.x];
    }
    __syncthreads();
    givens_core(k, nv - 1, hn, g_col, g_cs, g_sn, gj, gpre);
    stamp_end(k.stamp ? k.stamp + 8 : nullptr);
    return;
  }
  const bool lucky = hn < 1e-14;
  double* vj = k.V + (size_t)jn * k.n;
  if (PF && has0) {
    double wr = w0;
#pragma unroll
    for (int v = 0; v < kRegRestart; ++v)
      if (v < nv) wr = fma(-hs[v], v0[PF ? v : 0], wr);
    if (!lucky) {
      const double vv = wr / hn;
      vj[r0] = vv;
      k.ubuf[r0] = vv / sc0;
    }
  }
  if constexpr (PF) {
    for (int r = r0 + nb * blockDim.x; r < k.n; r += nb * blockDim.x) {
      double wr = k.w[r];
  #pragma unroll
      for (int v = 0; v < kRegRestart; ++v)
        if (v < nv) wr = fma(-hs[v], k.V[(size_t)v * k.n + r], wr);
      if (!lucky) {
        const double vv = wr / hn;
        vj[r] = vv;
        k.ubuf[r] = vv / k.scale[r];
      }
    }
  } else {
    // large systems: NV x RP loads in flight per thread (normalize_rows);
    // hs[] beyond nv must read as 0 for the fixed-length FMA chains
    if (rows_cta) {
      __syncthreads();
      if (threadIdx.x + nv <= kRegRestart) hs[nv + threadIdx.x] = 0.0;
      __syncthreads();
      if (nv <= 4) normalize_rows<4, 8>(k, nv, nb, hs, hn, lucky, vj);
      else if (nv <= 8) normalize_rows<8, 4>(k, nv, nb, hs, hn, lucky, vj);
      else if (nv <= 16) normalize_rows<16, 2>(k, nv, nb, hs, hn, lucky, vj);
      else normalize_rows<kRegRestart, 1>(k, nv, nb, hs, hn, lucky, vj);
    }
  }
  stamp_end(k.stamp ? k.stamp + 8 : nullptr);
}

}  // namespace fsigpu
