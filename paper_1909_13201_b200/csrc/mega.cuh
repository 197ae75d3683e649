// SPDX-License-Identifier: Apache-2.0
//
// Persistent cooperative FGMRES restart cycle ("megakernel").
//
// One launch runs a whole restart cycle of the reference's gmres
// (proj/src/krylov.cpp:52-113): per Arnoldi step the V-cycle
// (gmg.cpp:188-239, inverse-mode FS smoothers), the row-scaled outer SpMV,
// CGS2 orthogonalisation with on-device Givens, and the normalisation;
// then the back substitution, x += Z y and the true residual
// (krylov.cpp:103-118). Phases are separated by a software grid barrier
// (all CTAs are co-resident: cooperative launch, grid = SMs x occupancy),
// which replaces ~23 dependent kernel launches per Arnoldi step.
//
// Data produced inside the kernel (level vectors, Krylov basis, partials)
// is read with L2-coherent loads (__ldcg); only setup-time matrices
// (CSR values/indices, block inverses, masks) use the read-only path.
// Per-element arithmetic and summation order match the multi-kernel path
// (same LPR lane split, same 8-column-group tile reduction, same combine),
// except the Arnoldi reductions, which reduce over this grid's CTAs.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "dense.cuh"
#include "krylov.cuh"

namespace fsigpu {

constexpr int kMegaThreads = 256;
constexpr int kMegaMaxLevels = 8;

struct GridBar {
  unsigned int count;
  unsigned int gen;
  unsigned int error;   // watchdog tripped (deadlock guard)
  unsigned int phase;   // barrier sequence number, for diagnostics
  unsigned int limit;   // debug: every thread exits after `limit` barriers (0 = off)
  unsigned int ntrace;  // debug: phase timestamps recorded by CTA 0
  unsigned long long trace[256];
};

__device__ __forceinline__ void trace_point(GridBar* gb) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned int i = gb->ntrace;
    if (i < 256) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      gb->trace[i] = t;
      gb->ntrace = i + 1;
    }
  }
}

__shared__ unsigned int s_phase_count;  // zeroed at kernel entry (mg_init_cta)

__device__ __forceinline__ void mg_init_cta() {
  if (threadIdx.x == 0) s_phase_count = 0;
  __syncthreads();
}

__device__ __forceinline__ void phase_limit_check(GridBar* gb) {
  const unsigned int lim = *((volatile unsigned int*)&gb->limit);
  if (lim) {
    if (threadIdx.x == 0) s_phase_count += 1;
    __syncthreads();
    if (s_phase_count >= lim) asm volatile("exit;");
  }
}

// Spin with a ~2 s watchdog (globaltimer): a broken barrier reports an
// error instead of hanging the device.
__device__ __forceinline__ bool spin_until_changed(GridBar* gb, volatile unsigned int* vgen, unsigned int g) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*vgen == g) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) {
      atomicExch(&gb->error, 1u);
      return false;
    }
    if (*((volatile unsigned int*)&gb->error)) return false;
  }
  return true;
}

struct MLevel {
  int n, nc;
  const int* a_ptr;
  const int* a_idx;
  const double* a_val;
  int a_lpr;
  const int* p_ptr;
  const int* p_idx;
  const double* p_val;
  int p_lpr;
  const int* r_ptr;
  const int* r_idx;
  const double* r_val;
  int r_lpr;
  const unsigned char* rmask;
  const unsigned char* cmask;
  int g1, n_us;
  const double* lumped;
  const int* aus_ptr;
  const int* aus_col;
  const double* aus_val;
  const int* bm;
  const long long* row_off;
  const double* inv;
  const long long* inv_off;
  const int* pos;
  const SolveItem* tiles;
  int n_tiles;
  const int* inv_ptr;
  const int* inv_idx;
  double* b;
  double* x;
  double* r;
  double* delta;
};

struct MegaArgs {
  int L;
  MLevel lv[kMegaMaxLevels];
  const double* cinv;  // coarse explicit inverse, row-major n0 x n0
  double omega;
  int pre, post;
  KBufs kb;
  GridBar* bar;
  int first_cycle;  // compute r0 / beta / target before the cycle
};

// ---------------------------------------------------------------- barrier
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense/generation barrier with acquire-release atomics (no full fences):
// arrive = atom.add.acq_rel; the last arriver resets the counter and
// publishes gen+1 with st.release; waiters poll gen with ld.acquire.
__device__ __forceinline__ void grid_sync_ar(GridBar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = ld_acquire(&gb->gen);
    if (atom_add_acqrel(&gb->count, 1u) == gridDim.x - 1) {
      gb->count = 0;
      st_release(&gb->gen, g + 1);
    } else {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (ld_acquire(&gb->gen) == g) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 2000000000ull) {
          atomicExch(&gb->error, 1u);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Plain phase barrier: cooperative_groups grid sync (measured 1.2 us on
// 148-296 CTAs, vs 2.0 us for an acquire/release counter and 4 us for a
// fence-based one; tools/debug_mega.py).
__device__ __forceinline__ void grid_sync(GridBar* gb) {
  cooperative_groups::this_grid().sync();
  trace_point(gb);
  phase_limit_check(gb);
}

// Fence-based generation barrier (reference implementation for the
// barrier microbenchmark only).
__device__ __forceinline__ void grid_sync_fence(GridBar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &gb->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&gb->count, 1u) == gridDim.x - 1) {
      gb->count = 0;
      gb->phase += 1;
      __threadfence();
      atomicExch(&gb->gen, g + 1);
    } else {
      spin_until_changed(gb, vgen, g);
    }
    __threadfence();
  }
  __syncthreads();
}

// Barrier whose last arriving CTA runs `fn` (a fixed-order reduction of
// the per-CTA partials) before releasing the others.
template <class F>
__device__ __forceinline__ void grid_sync_reduce(GridBar* gb, F fn) {
  __shared__ int s_last;
  __shared__ unsigned int s_gen;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_gen = ld_acquire(&gb->gen);
    __threadfence();  // publish this CTA's partials (written by all its threads)
    s_last = (atom_add_acqrel(&gb->count, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    fn();
    __syncthreads();
    if (threadIdx.x == 0) {
      gb->count = 0;
      gb->phase += 1;
      __threadfence();
      st_release(&gb->gen, s_gen + 1);
    }
  } else if (threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire(&gb->gen) == s_gen) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 2000000000ull) {
        atomicExch(&gb->error, 1u);
        break;
      }
    }
  }
  __syncthreads();
  trace_point(gb);
  phase_limit_check(gb);
}

__device__ __forceinline__ long long gtid() { return (long long)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ long long gthreads() { return (long long)gridDim.x * blockDim.x; }

// ---------------------------------------------------------------- level ops
// rhs of the block solve at frame position p (lumped-Jacobi update for
// group-2 rows, precond.cpp:281-287), coherent loads of the in-kernel r
__device__ __forceinline__ double mg_gather(const MLevel& L, const double* r, int p) {
  double v = __ldcg(r + p);
  if (p >= L.g1) {
    const int q = p - L.g1;
    const int k0 = __ldg(L.aus_ptr + q), k1 = __ldg(L.aus_ptr + q + 1);
    for (int k = k0; k < k1; ++k) {
      const int c = __ldg(L.aus_col + k);
      const double d = __ldcg(r + L.g1 + c) / __ldg(L.lumped + c);
      v = sub_rn(v, mul_rn(__ldg(L.aus_val + k), d));
    }
  }
  return v;
}

// inverse-mode block solve: CTA-stride over 64-row tiles (inv_gemv_kernel)
__device__ void mg_block_solve(const MLevel& L, const double* rhs, double* xs, double (*red)[kInvTileRows]) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int item = blockIdx.x; item < L.n_tiles; item += gridDim.x) {
    const SolveItem it = L.tiles[item];
    const int b = it.first, row0 = it.pad;
    const int m = __ldg(L.bm + b);
    const int RP = even_up(m) / 2;
    const long long ro = __ldg(L.row_off + b);
    for (int s = tid; s < m; s += kMegaThreads) xs[s] = mg_gather(L, rhs, __ldg(L.pos + ro + s));
    __syncthreads();
    const int rp = row0 / 2 + lane;
    double s0 = 0.0, s1 = 0.0;
    if (rp < RP)
      inv_rowpair_dot(reinterpret_cast<const double2*>(L.inv + __ldg(L.inv_off + b)), RP, rp, m, w, 8, xs, s0, s1);
    red[w][2 * lane] = s0;
    red[w][2 * lane + 1] = s1;
    __syncthreads();
    if (tid < kInvTileRows) {
      const int i = row0 + tid;
      if (i < m) {
        double z = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) z += red[c][tid];
        L.delta[ro + i] = z;
      }
    }
    __syncthreads();
  }
}

// fs_combine_kernel, grid-stride
__device__ void mg_combine(const MLevel& L, const double* r, double omega, int x_zero) {
  for (long long p = gtid(); p < L.n; p += gthreads()) {
    double z;
    if (p >= L.g1 && p < L.g1 + L.n_us) {
      z = __ldcg(r + p) / __ldg(L.lumped + (p - L.g1));
    } else {
      const int k0 = __ldg(L.inv_ptr + p), k1 = __ldg(L.inv_ptr + p + 1);
      double s = 0.0;
      for (int k = k0; k < k1; ++k) s = add_rn(s, __ldcg(L.delta + __ldg(L.inv_idx + k)));
      z = (k1 - k0 > 1) ? s / (double)(k1 - k0) : s;
    }
    const double xo = x_zero ? 0.0 : __ldcg(L.x + p);
    L.x[p] = add_rn(xo, mul_rn(omega, z));
  }
}

// One CSR row sum with LPR lanes (same batching/reduction as csr_kernel).
// row < 0: an idle row group (all LPR lanes still run the shuffle tree, so
// full-mask shuffles never wait on lanes that skipped the row).
template <int LPR, class G>
__device__ __forceinline__ double mg_row(const int* __restrict__ ptr, const int* __restrict__ idx,
                                         const double* __restrict__ val, int row, int lane, G gx) {
  const int k0 = row >= 0 ? __ldg(ptr + row) : 0, k1 = row >= 0 ? __ldg(ptr + row + 1) : 0;
  double s = 0.0;
  constexpr int U = 4;
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
    for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? gx(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(v[u], xv[u], s);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
  return s;
}

struct MgGather {
  const double* x;
  __device__ double operator()(int c) const { return __ldcg(x + c); }
};
struct MgGatherMasked {
  const double* x;
  const unsigned char* mask;
  __device__ double operator()(int c) const { return __ldg(mask + c) ? 0.0 : __ldcg(x + c); }
};

// grid-stride CSR sweep; the epilogue runs in lane 0 of each row
template <int LPR, class G, class E>
__device__ void mg_csr_t(int rows, const int* ptr, const int* idx, const double* val, G gx, E epi) {
  const long long groups = gthreads() / LPR;
  const int lane = threadIdx.x & (LPR - 1);
  const long long rounds = (rows + groups - 1) / groups;
  for (long long rd = 0; rd < rounds; ++rd) {
    const long long row = rd * groups + gtid() / LPR;
    const bool ok = row < rows;
    const double s = mg_row<LPR>(ptr, idx, val, ok ? (int)row : -1, lane, gx);
    if (ok && lane == 0) epi((int)row, s);
  }
}
template <class G, class E>
__device__ void mg_csr(int lpr, int rows, const int* ptr, const int* idx, const double* val, G gx, E epi) {
  switch (lpr) {
    case 2: mg_csr_t<2>(rows, ptr, idx, val, gx, epi); break;
    case 4: mg_csr_t<4>(rows, ptr, idx, val, gx, epi); break;
    case 8: mg_csr_t<8>(rows, ptr, idx, val, gx, epi); break;
    case 16: mg_csr_t<16>(rows, ptr, idx, val, gx, epi); break;
    default: mg_csr_t<32>(rows, ptr, idx, val, gx, epi); break;
  }
}

struct MgEpiResid {
  const double* b;
  double* r;
  __device__ void operator()(int i, double s) const { r[i] = __ldcg(b + i) - s; }
};
struct MgEpiRestrict {
  const unsigned char* mask;
  double* y;
  __device__ void operator()(int i, double s) const { y[i] = __ldg(mask + i) ? 0.0 : s; }
};
struct MgEpiProlongAdd {
  const unsigned char* mask;
  double* x;
  __device__ void operator()(int i, double s) const {
    if (!__ldg(mask + i)) x[i] = __ldcg(x + i) + s;
  }
};
struct MgEpiScaled {
  const double* scale;
  double* y;
  __device__ void operator()(int i, double s) const { y[i] = __ldg(scale + i) * s; }
};
struct MgEpiResidScaled {
  const double* b;
  const double* scale;
  double* r;
  __device__ void operator()(int i, double s) const { r[i] = __ldcg(b + i) - __ldg(scale + i) * s; }
};

// coarse: x0 (+)= Cinv b0, warp per row (gemv_kernel)
__device__ void mg_coarse(const double* __restrict__ M, int n, const double* b, double* x, int acc) {
  const long long warps = gthreads() / 32;
  const int lane = threadIdx.x & 31;
  const long long rounds = (n + warps - 1) / warps;
  for (long long rd = 0; rd < rounds; ++rd) {
    const long long row = rd * warps + gtid() / 32;
    if (row >= n) continue;
    const double* Mr = M + (size_t)row * n;
    double s = 0.0;
    constexpr int U = 8;
    for (int jb = lane; jb < n; jb += 32 * U) {
      double mv[U], bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = jb + 32 * u;
        mv[u] = j < n ? __ldg(Mr + j) : 0.0;
        bv[u] = j < n ? __ldcg(b + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) s = fma(mv[u], bv[u], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) x[row] = acc ? __ldcg(x + row) + s : s;
  }
}

// ---------------------------------------------------------------- V-cycle
struct MegaSmem {
  double xs[kLargeMax];
  double red[8][kInvTileRows];
  double sm[kMaxRestart * kMegaThreads / 8];  // Arnoldi transposes (per warp slot)
};

__device__ void mg_sweep(const MegaArgs& A, int l, int x_zero, double* xs, double (*red)[kInvTileRows]) {
  const MLevel& L = A.lv[l];
  const double* rhs = L.b;
  if (!x_zero) {
    mg_csr(L.a_lpr, L.n, L.a_ptr, L.a_idx, L.a_val, MgGather{L.x}, MgEpiResid{L.b, L.r});
    grid_sync(A.bar);
    rhs = L.r;
  }
  mg_block_solve(L, rhs, xs, red);
  grid_sync(A.bar);
  mg_combine(L, rhs, A.omega, x_zero);
  grid_sync(A.bar);
}

__device__ void mg_vcycle(const MegaArgs& A, double* xs, double (*red)[kInvTileRows]) {
  const int top = A.L - 1;
  for (int l = top; l >= 1; --l) {
    const MLevel& L = A.lv[l];
    const MLevel& B = A.lv[l - 1];
    if (A.pre == 0) {
      for (long long p = gtid(); p < L.n; p += gthreads()) L.x[p] = 0.0;
      grid_sync(A.bar);
    }
    for (int k = 0; k < A.pre; ++k) mg_sweep(A, l, k == 0, xs, red);
    mg_csr(L.a_lpr, L.n, L.a_ptr, L.a_idx, L.a_val, MgGather{L.x}, MgEpiResid{L.b, L.r});
    grid_sync(A.bar);
    mg_csr(L.r_lpr, L.nc, L.r_ptr, L.r_idx, L.r_val, MgGather{L.r}, MgEpiRestrict{B.rmask, B.b});
    grid_sync(A.bar);
  }
  mg_coarse(A.cinv, A.lv[0].n, A.lv[0].b, A.lv[0].x, 0);
  grid_sync(A.bar);
  for (int l = 1; l <= top; ++l) {
    const MLevel& L = A.lv[l];
    const MLevel& B = A.lv[l - 1];
    mg_csr(L.p_lpr, L.n, L.p_ptr, L.p_idx, L.p_val, MgGatherMasked{B.x, B.cmask}, MgEpiProlongAdd{L.cmask, L.x});
    grid_sync(A.bar);
    for (int k = 0; k < A.post; ++k) mg_sweep(A, l, 0, xs, red);
  }
}

// ---------------------------------------------------------------- Arnoldi
// per-thread partial dots of nv vectors over grid-stride rows, reduced per
// CTA through shared memory and written to partial[blockIdx][v]
__device__ void mg_cta_partials(const KBufs& k, double (&acc)[kMaxRestart], int nv, double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kMegaThreads / 32;
  // first reduce within the warp (tree), then across warps via smem
#pragma unroll
  for (int v = 0; v < kMaxRestart; ++v) {
    if (v < nv) {
      double s = acc[v];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
      if (lane == 0) sm[warp * kMaxRestart + v] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += sm[w * kMaxRestart + threadIdx.x];
    k.partial[(size_t)blockIdx.x * (kMaxRestart + 1) + threadIdx.x] = s;
  }
}

__device__ void mg_finish(const KBufs& k, int nv, double* dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kMegaThreads / 32;
  for (int v = warp; v < nv; v += NW) {
    double s = 0.0;
    for (unsigned int b = lane; b < gridDim.x; b += 32) s += __ldcg(k.partial + (size_t)b * (kMaxRestart + 1) + v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) dst[v] = s;
  }
}

// ||r|| -> beta (and r0/history/target on the first call); cycle start
__device__ void mg_norm_r(const MegaArgs& A, double* sm) {
  const KBufs& k = A.kb;
  double acc[kMaxRestart] = {0.0};
  for (long long r = gtid(); r < k.n; r += gthreads()) {
    const double v = __ldcg(k.r + r);
    acc[0] = fma(v, v, acc[0]);
  }
  mg_cta_partials(k, acc, 1, sm);
  __shared__ double s_n2;
  grid_sync_reduce(A.bar, [&]() {
    mg_finish(k, 1, &s_n2);
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
      for (int i = 0; i <= k.mr; ++i) k.g[i] = 0.0;
      k.g[0] = beta;
      st->j = 0;
      st->stop = 0;
    }
  });
}

__device__ void mg_arnoldi(const MegaArgs& A, double* sm) {
  const KBufs& k = A.kb;
  KState* st = k.st;
  const int j = *((volatile int*)&st->j);
  const int nv = j + 1;
  // ---- h1 = V^T w, Z[j] = zbuf
  {
    double acc[kMaxRestart];
#pragma unroll
    for (int v = 0; v < kMaxRestart; ++v) acc[v] = 0.0;
    double* zj = k.Z + (size_t)j * k.n;
    for (long long r = gtid(); r < k.n; r += gthreads()) {
      const double wr = __ldcg(k.w + r);
      zj[r] = __ldcg(k.zbuf + r);
#pragma unroll
      for (int v = 0; v < kMaxRestart; ++v)
        if (v < nv) acc[v] = fma(__ldcg(k.V + (size_t)v * k.n + r), wr, acc[v]);
    }
    mg_cta_partials(k, acc, nv, sm);
    grid_sync_reduce(A.bar, [&]() { mg_finish(k, nv, st->h1); });
  }
  // ---- w -= V h1 ; h2 = V^T w
  {
    __shared__ double hs[kMaxRestart];
    if (threadIdx.x < nv) hs[threadIdx.x] = __ldcg(st->h1 + threadIdx.x);
    __syncthreads();
    double acc[kMaxRestart];
#pragma unroll
    for (int v = 0; v < kMaxRestart; ++v) acc[v] = 0.0;
    for (long long r = gtid(); r < k.n; r += gthreads()) {
      double wr = __ldcg(k.w + r);
#pragma unroll
      for (int v = 0; v < kMaxRestart; ++v)
        if (v < nv) wr = fma(-hs[v], __ldcg(k.V + (size_t)v * k.n + r), wr);
      k.w[r] = wr;
#pragma unroll
      for (int v = 0; v < kMaxRestart; ++v)
        if (v < nv) acc[v] = fma(__ldcg(k.V + (size_t)v * k.n + r), wr, acc[v]);
    }
    mg_cta_partials(k, acc, nv, sm);
    grid_sync_reduce(A.bar, [&]() { mg_finish(k, nv, st->h2); });
  }
  // ---- w -= V h2 ; ||w|| ; Givens (krylov.cpp:79-100)
  {
    __shared__ double hs[kMaxRestart];
    if (threadIdx.x < nv) hs[threadIdx.x] = __ldcg(st->h2 + threadIdx.x);
    __syncthreads();
    double acc[kMaxRestart] = {0.0};
    for (long long r = gtid(); r < k.n; r += gthreads()) {
      double wr = __ldcg(k.w + r);
#pragma unroll
      for (int v = 0; v < kMaxRestart; ++v)
        if (v < nv) wr = fma(-hs[v], __ldcg(k.V + (size_t)v * k.n + r), wr);
      k.w[r] = wr;
      acc[0] = fma(wr, wr, acc[0]);
    }
    mg_cta_partials(k, acc, 1, sm);
    __shared__ double s_w2;
    grid_sync_reduce(A.bar, [&]() {
      mg_finish(k, 1, &s_w2);
      __syncthreads();
      givens_step(k, sqrt(s_w2));
    });
  }
  // ---- v_{j+1} = w / hn ; u = v_{j+1} / scale
  {
    const double hn = *((volatile double*)&st->hn);
    if (hn >= 1e-14) {
      double* vj = k.V + (size_t)(j + 1) * k.n;
      for (long long r = gtid(); r < k.n; r += gthreads()) {
        const double v = __ldcg(k.w + r) / hn;
        vj[r] = v;
        k.ubuf[r] = v / __ldg(k.scale + r);
      }
    }
    grid_sync(A.bar);
  }
}

// One restart cycle (or, with first_cycle, the initial residual too).
__global__ void barrier_test_kernel(GridBar* gb, int iters, int kind) {
  mg_init_cta();
  if (kind == 0) {
    for (int i = 0; i < iters; ++i) grid_sync_fence(gb);
  } else if (kind == 1) {
    for (int i = 0; i < iters; ++i) grid_sync_ar(gb);
  } else {
    cooperative_groups::grid_group gg = cooperative_groups::this_grid();
    for (int i = 0; i < iters; ++i) gg.sync();
  }
}

__global__ void __launch_bounds__(kMegaThreads, 2) fgmres_cycle_kernel(MegaArgs A) {
  __shared__ double xs[kLargeMax];
  __shared__ double red[8][kInvTileRows];
  __shared__ double sm[(kMegaThreads / 32) * kMaxRestart];
  const KBufs& k = A.kb;
  KState* st = k.st;
  mg_init_cta();
  if (A.first_cycle) {
    mg_csr(A.lv[A.L - 1].a_lpr, k.n, A.lv[A.L - 1].a_ptr, A.lv[A.L - 1].a_idx, A.lv[A.L - 1].a_val, MgGather{k.x},
           MgEpiResidScaled{k.b, k.scale, k.r});
    grid_sync(A.bar);
    mg_norm_r(A, sm);
  }
  if (*((volatile int*)&st->converged) || *((volatile int*)&st->its) >= *((volatile int*)&st->max_iters)) return;
  // v0 = r / beta ; u = v0 / scale
  {
    const double beta = *((volatile double*)&st->beta);
    for (long long r = gtid(); r < k.n; r += gthreads()) {
      const double v = __ldcg(k.r + r) / beta;
      k.V[r] = v;
      k.ubuf[r] = v / __ldg(k.scale + r);
    }
    grid_sync(A.bar);
  }
  const int mr = k.mr;
  for (int guard = 0; guard < mr; ++guard) {
    if (*((volatile unsigned int*)&A.bar->error)) return;
    mg_vcycle(A, xs, red);  // zbuf = M u   (top level: b = ubuf, x = zbuf)
    mg_csr(A.lv[A.L - 1].a_lpr, k.n, A.lv[A.L - 1].a_ptr, A.lv[A.L - 1].a_idx, A.lv[A.L - 1].a_val, MgGather{k.zbuf},
           MgEpiScaled{k.scale, k.w});
    grid_sync(A.bar);
    mg_arnoldi(A, sm);
    const int stop = *((volatile int*)&st->stop);
    const int jj = *((volatile int*)&st->j);
    const int its = *((volatile int*)&st->its);
    if (stop || jj >= mr || its >= *((volatile int*)&st->max_iters)) break;
  }
  // y = H^{-1} g (one CTA), x += Z y, r = b - A_s x, beta
  if (blockIdx.x == 0) {
    __shared__ double Hs[kMaxRestart * kMaxRestart];
    __shared__ double gs[kMaxRestart + 1];
    __shared__ double y[kMaxRestart];
    const int j = st->j;
    for (int e = threadIdx.x; e < j * j; e += blockDim.x) Hs[e] = __ldcg(k.H + (e / j) * mr + (e % j));
    if (threadIdx.x < j) gs[threadIdx.x] = __ldcg(k.g + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = j - 1; i >= 0; --i) {
        double s = gs[i];
        for (int q = i + 1; q < j; ++q) s -= Hs[i * j + q] * y[q];
        y[i] = s / Hs[i * j + i];
      }
      for (int i = 0; i < j; ++i) st->y[i] = y[i];
    }
  }
  grid_sync(A.bar);
  {
    const int j = *((volatile int*)&st->j);
    __shared__ double ys[kMaxRestart];
    if (threadIdx.x < j) ys[threadIdx.x] = __ldcg(st->y + threadIdx.x);
    __syncthreads();
    for (long long r = gtid(); r < k.n; r += gthreads()) {
      double s = 0.0;
      for (int i = 0; i < j; ++i) s = fma(ys[i], __ldcg(k.Z + (size_t)i * k.n + r), s);
      k.x[r] = __ldcg(k.x + r) + s;
    }
    grid_sync(A.bar);
  }
  mg_csr(A.lv[A.L - 1].a_lpr, k.n, A.lv[A.L - 1].a_ptr, A.lv[A.L - 1].a_idx, A.lv[A.L - 1].a_val, MgGather{k.x},
         MgEpiResidScaled{k.b, k.scale, k.r});
  grid_sync(A.bar);
  mg_norm_r(A, sm);
}

}  // namespace fsigpu
