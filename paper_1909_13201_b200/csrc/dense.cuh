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
// (m <= 64, one warp each, factor streamed with LDG) or one large block
// (whole 256-thread CTA, factor panels double-buffered in shared memory by
// TMA bulk copies).
struct SolveItem {
  int type;   // 0 small, 1 large
  int first;  // first block id
  int count;  // blocks (small items)
  int pad;
};

constexpr int kSolveThreads = 256;
constexpr int kSmallMax = 64;
constexpr int kLargeMax = 1024;
constexpr int kTmaMax = 256;  // largest m whose panels are TMA-staged

// ---- solve format -------------------------------------------------------
// Per block, per 32-column panel p (k0 = 32p, kb = min(32, m-k0)):
//   fwd chunk: Ltri  = strictly-lower part of inv(L_pp), column-packed (lte)
//              Lpan  = L[k0+kb:m, k0:k0+kb], column-major, ld = hLe (even)
//   bwd chunk: Utri  = upper part of inv(U_pp) incl. diagonal, column-packed (ute)
//              Upan  = U[0:k0, k0:k0+kb], column-major, ld = k0
// Each chunk is contiguous and a multiple of 16 bytes, so one
// cp.async.bulk moves it. Bytes per block ~= 8 m^2 (the two triangular
// tile inverses replace the diagonal tiles, so nothing is read twice).
__host__ __device__ __forceinline__ int even_up(int x) { return (x + 1) & ~1; }

struct PanelGeom {
  int k0, kb, lt, lte, hL, hLe, ut, ute;
  __host__ __device__ PanelGeom(int m, int p) {
    k0 = 32 * p;
    kb = m - k0 < 32 ? m - k0 : 32;
    lt = kb * (kb - 1) / 2;
    lte = even_up(lt);
    hL = m - k0 - kb;
    hLe = even_up(hL);
    ut = kb * (kb + 1) / 2;
    ute = even_up(ut);
  }
  __host__ __device__ long long fwd_size() const { return (long long)lte + (long long)hLe * kb; }
  __host__ __device__ long long bwd_size() const { return (long long)ute + (long long)k0 * kb; }
  __host__ __device__ long long size() const { return fwd_size() + bwd_size(); }
};

__host__ __device__ __forceinline__ long long panel_offset(int m, int p) {
  long long o = 0;
  for (int q = 0; q < p; ++q) o += PanelGeom(m, q).size();
  return o;
}
__host__ __device__ __forceinline__ long long solve_format_size(int m) {
  return panel_offset(m, (m + 31) / 32);
}
// column-packed strictly-lower triangle: column kk holds rows kk+1..kb-1
__host__ __device__ __forceinline__ int ltri_col(int kb, int kk) { return kk * (kb - 1) - kk * (kk - 1) / 2; }
// column-packed upper triangle incl. diagonal: column jj holds rows 0..jj
__host__ __device__ __forceinline__ int utri_col(int jj) { return jj * (jj + 1) / 2; }

struct SolveArgs {
  const int* m;
  const long long* sf_off;
  const long long* row_off;
  const double* sf;
  const int* gsrc;
  const SolveItem* items;
  int smem_cap;  // doubles per panel buffer (TMA path)
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
  // explicit-inverse mode
  const int* lperm;         // pivoted row -> block-local row
  double* inv;              // column-major inverses, ld = even_up(m)
  const long long* inv_off;
  const int* pos;           // block-local row -> rhs source position
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

// ---- TMA bulk copy + mbarrier (sm_90+ PTX; SASS UBLKCP / SYNCS) ----------

template <int NW>
__device__ __forceinline__ void team_sync() {
  if constexpr (NW == 1)
    __syncwarp();
  else
    __syncthreads();
}

// Issue the q-th chunk load (q < P: forward chunk of panel q, else backward
// chunk of panel 2P-1-q) into buffer q&1.
__device__ __forceinline__ void issue_chunk(const double* blk, int m, int P, int q, double* buf, int cap,
                                           unsigned long long* bars) {
  const bool fwd = q < P;
  const int p = fwd ? q : 2 * P - 1 - q;
  const PanelGeom g(m, p);
  const long long off = panel_offset(m, p) + (fwd ? 0 : g.fwd_size());
  const unsigned bytes = (unsigned)(8 * (fwd ? g.fwd_size() : g.bwd_size()));
  double* dst = buf + (size_t)(q & 1) * cap;
  mbar_arrive_expect_tx(&bars[q & 1], bytes);
  if (bytes) tma_bulk_g2s(dst, blk + off, bytes, &bars[q & 1]);
}

// Solve one block with a team of NW warps (NW == 1: warp path, factor read
// with LDG; NW > 1 with TMA: panel chunks staged through `buf`).
// xs: shared scratch of m doubles (the pivoted, then solved, vector).
template <int NW, bool TMA>
__device__ void solve_block(const SolveArgs& a, int b, double* xs, double* buf, unsigned long long* bars, int t,
                            int ucol = -1) {
  constexpr int T = NW * 32;
  const int m = a.m[b];
  const int P = (m + 31) / 32;
  const long long ro = a.row_off[b];
  const double* __restrict__ blk = a.sf + a.sf_off[b];
  if constexpr (TMA) {
    if (t == 0) {
      issue_chunk(blk, m, P, 0, buf, a.smem_cap, bars);
      if (2 * P > 1) issue_chunk(blk, m, P, 1, buf, a.smem_cap, bars);
    }
  }
  if (ucol < 0) {
    for (int s = t; s < m; s += T) xs[s] = gather_rhs(a, __ldg(a.gsrc + ro + s));
  } else {  // e_ucol (block-local order) through the pivots: inverse columns
    for (int s = t; s < m; s += T) xs[s] = (__ldg(a.lperm + ro + s) == ucol) ? 1.0 : 0.0;
  }
  team_sync<NW>();

  // rows of the diagonal tile handled as (row, sub) pairs
  constexpr int DS = (NW == 1) ? 1 : 8;  // threads per diagonal row
  for (int q = 0; q < 2 * P; ++q) {
    const bool fwd = q < P;
    const int p = fwd ? q : 2 * P - 1 - q;
    const PanelGeom g(m, p);
    const double* src;
    if constexpr (TMA) {
      mbar_wait(&bars[q & 1], (q >> 1) & 1);
      src = buf + (size_t)(q & 1) * a.smem_cap;
    } else {
      src = blk + panel_offset(m, p) + (fwd ? 0 : g.fwd_size());
    }
    const int k0 = g.k0, kb = g.kb;
    // --- diagonal tile: x_p <- inv(L_pp) x_p  or  inv(U_pp) x_p
    double y = 0.0;
    const int i = t / DS, sub = t % DS;
    if (i < 32) {
      double s = 0.0;
      constexpr int U = 32 / DS;  // whole row in one predicated batch
      double v[U];
      if (fwd) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = sub + u * DS;
          v[u] = (kk < kb && kk < i && i < kb) ? src[ltri_col(kb, kk) + i - kk - 1] : 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int jj = sub + u * DS;
          v[u] = (jj < kb && jj >= i && i < kb) ? src[utri_col(jj) + i] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = sub + u * DS;
        s = fma(v[u], kk < kb ? xs[k0 + kk] : 0.0, s);
      }
      if constexpr (DS > 1) {
#pragma unroll
        for (int o = DS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, DS);
      }
      if (i < kb) y = fwd ? xs[k0 + i] + s : s;
    }
    team_sync<NW>();
    if (i < kb && sub == 0) xs[k0 + i] = y;
    team_sync<NW>();
    // --- off-diagonal panel: rows below (fwd) or above (bwd)
    const int h = fwd ? g.hL : k0;
    const int ld = fwd ? g.hLe : k0;
    const double* pan = fwd ? src + g.lte : src + g.ute;
    const int rbase = fwd ? k0 + kb : 0;
    if (h > 0) {
      const int tpr = (NW == 1) ? 1 : (h <= 32 ? 8 : h <= 64 ? 4 : h <= 128 ? 2 : 1);
      const int rows_per_pass = T / tpr;
      for (int r0 = 0; r0 < h; r0 += rows_per_pass) {
        const int r = r0 + t / tpr, sb = t % tpr;
        double s = 0.0;
        if (r < h) {
          constexpr int U = 8;
          for (int kq = sb; kq < kb; kq += U * tpr) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int kk = kq + u * tpr;
              v[u] = kk < kb ? pan[(size_t)kk * ld + r] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int kk = kq + u * tpr;
              s = fma(v[u], kk < kb ? xs[k0 + kk] : 0.0, s);
            }
          }
        }
        if (tpr > 1) {
          for (int o = tpr / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, tpr);
        }
        if (r < h && sb == 0) xs[rbase + r] -= s;
      }
    }
    team_sync<NW>();
    if constexpr (TMA) {
      if (t == 0 && q + 2 < 2 * P) {
        fence_proxy_async();
        issue_chunk(blk, m, P, q + 2, buf, a.smem_cap, bars);
      }
    }
  }
  if (ucol < 0) {
    for (int k = t; k < m; k += T) a.out[ro + k] = xs[k];
  } else {  // column ucol of inv(A_b), column-major with even leading dimension
    const int ld = even_up(m);
    double* col = a.inv + a.inv_off[b] + (size_t)ucol * ld;
    for (int k = t; k < ld; k += T) col[k] = k < m ? xs[k] : 0.0;
  }
}

// Items: type 0 = up to 8 small blocks (warp each); type 1 = one large
// block; type 2 = (block first, columns pad..pad+count-1) of a small block,
// one column per warp; type 3 = (block first, column pad) of a large block.
// Types 2/3 compute inverse columns (setup of the explicit-inverse mode).
// Three CTAs per SM (<= 80 registers): 24 warps keep more blocks' phases in
// flight; config-1 solve 2.51 -> 2.33 ms (4.07 -> 4.37 TB/s). Four CTAs
// (64 registers) spill and lose it again.
__global__ void __launch_bounds__(kSolveThreads, 3) block_solve_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double xs[kLargeMax];
  __shared__ unsigned long long bars[2];
  pdl_trigger();
  const SolveItem it = a.items[blockIdx.x];
  pdl_wait();
  const int tid = threadIdx.x;
  if (it.type == 0 || it.type == 2) {
    const int w = tid >> 5;
    if (w < it.count) {
      if (it.type == 0)
        solve_block<1, false>(a, it.first + w, xs + w * kSmallMax, nullptr, nullptr, tid & 31);
      else
        solve_block<1, false>(a, it.first, xs + w * kSmallMax, nullptr, nullptr, tid & 31, it.pad + w);
    }
  } else if (it.type == 3) {
    solve_block<kSolveThreads / 32, false>(a, it.first, xs, nullptr, nullptr, tid, it.pad);
  } else {
    const int m = a.m[it.first];
    if (m <= kTmaMax && a.smem_cap > 0) {
      if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
      }
      __syncthreads();
      solve_block<kSolveThreads / 32, true>(a, it.first, xs, dsm, bars, tid);
    } else {
      solve_block<kSolveThreads / 32, false>(a, it.first, xs, nullptr, nullptr, tid);
    }
  }
}

// ---------------------------------------------------------------- pipelined small-block solve
// Batched LU solve of blocks with m <= 64 and a plain gathered right-hand
// side (config 1: no lumped-Jacobi rows). Each warp streams its own blocks
// (block = gw, gw + G, ...) through two shared-memory buffers: one
// cp.async.bulk moves a block's whole solve format (contiguous, 16-B
// aligned, ~8 m^2 bytes) while the warp solves the previous block out of
// shared memory, so the HBM stream never waits on the dependent phases of
// a solve. The gathered right-hand side runs two blocks ahead in
// registers (index loads for block i+2, value loads for block i+1).
// dynamic smem: [NW][2][cap] doubles, then xs[NW][64]; static: mbarriers.
struct SmallPipeArgs {
  const int* m;
  const long long* sf_off;
  const long long* row_off;
  const double* sf;
  const int* gsrc;
  const double* r;
  double* out;
  long long nb;
  int cap;     // doubles per buffer
  int single;  // one buffer per warp + L2 prefetch of the next block (else two buffers)
};

// solve one block (m <= 64) whose solve format is at blk (shared memory);
// xs holds the pivoted right-hand side on entry and the solution on exit
__device__ __forceinline__ void small_solve_smem(const double* blk, int m, double* xs, int lane) {
  const int P = (m + 31) / 32;
  const long long po1 = PanelGeom(m, 0).size();
  for (int q = 0; q < 2 * P; ++q) {
    const bool fwd = q < P;
    const int p = fwd ? q : 2 * P - 1 - q;
    const PanelGeom g(m, p);
    const double* src = blk + (p ? po1 : 0) + (fwd ? 0 : g.fwd_size());
    const int k0 = g.k0, kb = g.kb;
    const int i = lane;
    // diagonal tile: two interleaved partial sums halve the FMA chain
    double s0 = 0.0, s1 = 0.0;
    if (fwd) {
#pragma unroll
      for (int kk = 0; kk < 32; kk += 2) {
        const double v0 = (kk < i && i < kb) ? src[ltri_col(kb, kk) + i - kk - 1] : 0.0;
        const double v1 = (kk + 1 < i && i < kb) ? src[ltri_col(kb, kk + 1) + i - kk - 2] : 0.0;
        s0 = fma(v0, xs[k0 + kk], s0);
        s1 = fma(v1, xs[k0 + kk + 1], s1);
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 32; jj += 2) {
        const double v0 = (jj < kb && jj >= i) ? src[utri_col(jj) + i] : 0.0;
        const double v1 = (jj + 1 < kb && jj + 1 >= i) ? src[utri_col(jj + 1) + i] : 0.0;
        s0 = fma(v0, jj < kb ? xs[k0 + jj] : 0.0, s0);
        s1 = fma(v1, jj + 1 < kb ? xs[k0 + jj + 1] : 0.0, s1);
      }
    }
    const double y = fwd ? xs[k0 + i] + (s0 + s1) : s0 + s1;
    __syncwarp();
    if (i < kb) xs[k0 + i] = y;
    __syncwarp();
    // off-diagonal panel: rows below (fwd, h = hL <= 32) or above (bwd, h = k0 <= 32)
    const int h = fwd ? g.hL : k0;
    if (h > 0) {
      const int ld = fwd ? g.hLe : k0;
      const double* pan = fwd ? src + g.lte : src + g.ute;
      const int rbase = fwd ? k0 + kb : 0;
      double t0 = 0.0, t1 = 0.0;
      if (lane < h) {
#pragma unroll
        for (int kk = 0; kk < 32; kk += 2) {
          if (kk < kb) t0 = fma(pan[(size_t)kk * ld + lane], xs[k0 + kk], t0);
          if (kk + 1 < kb) t1 = fma(pan[(size_t)(kk + 1) * ld + lane], xs[k0 + kk + 1], t1);
        }
        xs[rbase + lane] -= t0 + t1;
      }
      __syncwarp();
    }
  }
}

constexpr int kPipeMaxWarps = 8;
__global__ void __launch_bounds__(kPipeMaxWarps * 32) small_pipe_solve_kernel(SmallPipeArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) double dsm[];
  __shared__ unsigned long long bars[kPipeMaxWarps][2];
  const int NW = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long G = (long long)gridDim.x * NW;
  const long long b0 = (long long)blockIdx.x * NW + warp;  // iteration j handles block b0 + j*G
  const int nbuf = a.single ? 1 : 2;
  double* buf = dsm + (size_t)warp * nbuf * a.cap;
  double* xs = dsm + (size_t)NW * nbuf * a.cap + warp * 64;
  unsigned long long* bar = bars[warp];
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (b0 >= a.nb) return;
  // block metadata for 32 iterations at a time: lane l holds iteration
  // 32*batch + l; two batches in registers so lookups up to 2 ahead never
  // wait on a dependent global load
  long long c_ro = 0, c_o0 = 0, n_ro = 0, n_o0 = 0;
  int c_m = -1, c_sz = 0, n_m = -1, n_sz = 0;
  auto load_batch = [&](int j0, long long& ro, long long& o0, int& m, int& sz) {
    const long long bb = b0 + (long long)(j0 + lane) * G;
    m = -1;
    if (bb < a.nb) {
      ro = a.row_off[bb];
      m = (int)(a.row_off[bb + 1] - ro);
      o0 = a.sf_off[bb];
      sz = (int)(a.sf_off[bb + 1] - o0);
    }
  };
  load_batch(0, c_ro, c_o0, c_m, c_sz);
  load_batch(32, n_ro, n_o0, n_m, n_sz);
  int it = 0;
  auto meta = [&](int j, long long& ro, long long& o0, int& m, int& sz) {
    const bool cur = (j >> 5) == (it >> 5);
    const int l = j & 31;
    ro = __shfl_sync(kFull, cur ? c_ro : n_ro, l);
    o0 = __shfl_sync(kFull, cur ? c_o0 : n_o0, l);
    m = __shfl_sync(kFull, cur ? c_m : n_m, l);
    sz = __shfl_sync(kFull, cur ? c_sz : n_sz, l);
  };
  auto issue = [&](long long o0, int sz, int slot) {
    mbar_arrive_expect_tx(&bar[slot], (unsigned)(8 * sz));
    tma_bulk_g2s(buf + (size_t)slot * a.cap, a.sf + o0, (unsigned)(8 * sz), &bar[slot]);
  };
  auto load_idx = [&](long long ro, int mm, int& i0, int& i1) {
    i0 = (lane < mm) ? __ldg(a.gsrc + ro + lane) : -1;
    i1 = (lane + 32 < mm) ? __ldg(a.gsrc + ro + lane + 32) : -1;
  };
  long long ro, o0;
  int m, sz;
  meta(0, ro, o0, m, sz);
  if (lane == 0) issue(o0, sz, 0);
  // right-hand side two blocks ahead: values of iteration it + 1, indices of it + 2
  int c0, c1, n0, n1;
  load_idx(ro, m, c0, c1);
  double v0 = c0 >= 0 ? __ldg(a.r + c0) : 0.0, v1 = c1 >= 0 ? __ldg(a.r + c1) : 0.0;
  {
    long long r1, q1;
    int m1, s1;
    meta(1, r1, q1, m1, s1);
    load_idx(r1, m1, n0, n1);
  }
  for (;; ++it) {
    if ((it & 31) == 0 && it > 0) {
      c_ro = n_ro, c_o0 = n_o0, c_m = n_m, c_sz = n_sz;
      load_batch(it + 32, n_ro, n_o0, n_m, n_sz);
    }
    meta(it, ro, o0, m, sz);
    if (m < 0) break;
    long long r1, q1;
    int m1, s1;
    meta(it + 1, r1, q1, m1, s1);
    if (m1 >= 0 && lane == 0) {
      if (a.single) {
        l2_prefetch_bulk(a.sf + q1, (unsigned)(8 * s1));  // lands in L2 during this solve
      } else {
        fence_proxy_async();  // the buffer's last generic reads precede the async write
        issue(q1, s1, (it + 1) & 1);
      }
    }
    // next block's values (its indices arrived during the last solve) and
    // the indices of the block after it
    const double w0 = n0 >= 0 ? __ldg(a.r + n0) : 0.0, w1 = n1 >= 0 ? __ldg(a.r + n1) : 0.0;
    {
      long long r2, q2;
      int m2, s2;
      meta(it + 2, r2, q2, m2, s2);
      load_idx(r2, m2, n0, n1);
    }
    xs[lane] = v0;
    xs[lane + 32] = v1;
    if (a.single)
      mbar_wait(&bar[0], it & 1);
    else
      mbar_wait(&bar[it & 1], (it >> 1) & 1);
    __syncwarp();
    small_solve_smem(buf + (size_t)(a.single ? 0 : (it & 1)) * a.cap, m, xs, lane);
    if (lane < m) a.out[ro + lane] = xs[lane];
    if (lane + 32 < m) a.out[ro + lane + 32] = xs[lane + 32];
    __syncwarp();
    if (a.single && m1 >= 0 && lane == 0) {  // the next block, now mostly an L2 hit
      fence_proxy_async();
      issue(q1, s1, 0);
    }
    v0 = w0;
    v1 = w1;
  }
}

// ---------------------------------------------------------------- inverse mode
// delta_b = inv(A_b) * rhs_b  (rhs gathered in block-local order). inv(A_b)
// is column-major with even leading dimension ld. Small blocks (m <= 64):
// one warp per block, a lane owns a row pair. Large blocks: one CTA per
// 64-row tile; thread (rp, cg) owns row pair rp of the tile and columns
// j = cg (mod 8); the 8 column-group partial sums are added in a fixed
// order (deterministic). Loads are issued in predicated batches of 8
// 16-byte vectors per thread.
constexpr int kInvTileRows = 64;

__device__ __forceinline__ void inv_rowpair_dot(const double2* __restrict__ M, int RP, int rp, int m, int cg,
                                                int CG, const double* xs, double& s0, double& s1) {
  constexpr int U = 8;
  for (int jb = cg; jb < m; jb += U * CG) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u * CG;
      v[u] = j < m ? __ldg(M + (size_t)j * RP + rp) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u * CG;
      const double xj = j < m ? xs[j] : 0.0;
      s0 = fma(v[u].x, xj, s0);
      s1 = fma(v[u].y, xj, s1);
    }
  }
}

__global__ void __launch_bounds__(kSolveThreads) inv_gemv_kernel(SolveArgs a) {
  __shared__ double xs[kLargeMax];
  __shared__ double red[8][kInvTileRows];
  pdl_trigger();
  const SolveItem it = a.items[blockIdx.x];
  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (it.type == 0) {  // small blocks: warp per block
    if (w >= it.count) return;
    const int b = it.first + w;
    const int m = a.m[b];
    const int RP = even_up(m) / 2;
    const long long ro = a.row_off[b];
    double* x = xs + w * kSmallMax;
    for (int s = lane; s < m; s += 32) x[s] = gather_rhs(a, a.pos ? __ldg(a.pos + ro + s) : (int)(ro + s));
    __syncwarp();
    double s0 = 0.0, s1 = 0.0;
    if (lane < RP)
      inv_rowpair_dot(reinterpret_cast<const double2*>(a.inv + a.inv_off[b]), RP, lane, m, 0, 1, x, s0, s1);
    if (2 * lane < m) a.out[ro + 2 * lane] = s0;
    if (2 * lane + 1 < m) a.out[ro + 2 * lane + 1] = s1;
    return;
  }
  // large block tile: rows [row0, row0 + 64)
  const int b = it.first;
  const int row0 = it.pad;
  const int m = a.m[b];
  const int RP = even_up(m) / 2;
  const long long ro = a.row_off[b];
  for (int s = tid; s < m; s += kSolveThreads) xs[s] = gather_rhs(a, a.pos ? __ldg(a.pos + ro + s) : (int)(ro + s));
  __syncthreads();
  const int rp = row0 / 2 + lane;
  double s0 = 0.0, s1 = 0.0;
  if (rp < RP)
    inv_rowpair_dot(reinterpret_cast<const double2*>(a.inv + a.inv_off[b]), RP, rp, m, w, 8, xs, s0, s1);
  red[w][2 * lane] = s0;
  red[w][2 * lane + 1] = s1;
  __syncthreads();
  if (tid < kInvTileRows) {
    const int i = row0 + tid;
    if (i < m) {
      double z = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) z += red[c][tid];
      a.out[ro + i] = z;
    }
  }
}

// ---------------------------------------------------------------- LU
// inv(L_pp) (unit lower, strict part) and inv(U_pp) (upper) of the kb x kb
// diagonal tile at k0 of a column-major m x m factor A, written to S
// (column c at S[c*33 ..], stride 33 keeps the 32 threads on distinct
// banks). Thread c < kb inverts column c by column-oriented substitution:
// within a step the updates are independent, so shared-memory accesses
// pipeline instead of forming dependent chains.
constexpr int kTileLd = 33;
__device__ __forceinline__ void tile_inverses(const double* A, int m, int k0, int kb, double* S, int t) {
  if (t >= kb) return;
  const int c = t;
  double* x = S + c * kTileLd;
  for (int i = 0; i < kb; ++i) x[i] = (i == c) ? 1.0 : 0.0;
  for (int k = c; k < kb; ++k) {  // lower: L x = e_c
    const double xk = x[k];
    const double* Lk = A + (size_t)(k0 + k) * m + k0;
    for (int i = k + 1; i < kb; ++i) x[i] = fma(-Lk[i], xk, x[i]);
  }
  // the upper solve touches only x[0..c]: the strict-lower result at
  // x[c+1..kb) stays in place
  for (int i = 0; i <= c; ++i) x[i] = (i == c) ? 1.0 : 0.0;
  for (int k = c; k >= 0; --k) {  // upper: U x = e_c
    const double* Uk = A + (size_t)(k0 + k) * m + k0;
    const double xk = x[k] / Uk[k];
    x[k] = xk;
    for (int i = 0; i < k; ++i) x[i] = fma(-Uk[i], xk, x[i]);
  }
}

// Register version of tile_inverses for one warp, lane c = column c:
// which == 0 writes the strict lower part of inv(L_pp), which == 1 the upper
// part of inv(U_pp) (incl. the diagonal), into the same S layout. The loops
// run over all 32 steps (x[k] = 0 for the steps before column c, so those
// updates leave x unchanged) and index x at compile time; the diagonal
// reciprocals are formed once per lane and broadcast by shuffle, which
// takes the divisions off the back-substitution chain.
__device__ __forceinline__ void tile_inverse_warp(const double* A, int m, int k0, int kb, double* S, int c,
                                                  int which) {
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == c) ? 1.0 : 0.0;
  if (which == 0) {
#pragma unroll
    for (int k = 0; k < 31; ++k) {
      if (k < kb - 1) {
        const double xk = x[k];
        const double* Lk = A + (size_t)(k0 + k) * m + k0;
        // rows i >= kb read past the tile (still inside the staged block
        // and its scratch); they never feed back into x[k < kb]
#pragma unroll
        for (int i = k + 1; i < 32; ++i) x[i] = fma(-Lk[i], xk, x[i]);
      }
    }
    if (c < kb) {
#pragma unroll
      for (int i = 1; i < 32; ++i)
        if (i > c && i < kb) S[c * kTileLd + i] = x[i];
    }
  } else {
    const double rinv = (c < kb) ? 1.0 / A[(size_t)(k0 + c) * m + k0 + c] : 0.0;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k < kb) {
        const double xk = x[k] * __shfl_sync(kFull, rinv, k);
        x[k] = xk;
        const double* Uk = A + (size_t)(k0 + k) * m + k0;
#pragma unroll
        for (int i = 0; i < k; ++i) x[i] = fma(-Uk[i], xk, x[i]);
      }
    }
    if (c < kb) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i <= c) S[c * kTileLd + i] = x[i];
    }
  }
}

// Outputs of a finished factorization held column-major in A (shared or
// global): pivots, the composed gather map, the optional bit-exact LU and
// the solve format (tile inverses + packed panels, see PanelGeom).
// perm[k] = pivot row of step k; scratch: m doubles; S: 32 x kTileLd doubles.
template <int NT, bool REG_TILE>
__device__ __forceinline__ void lu_write_outputs(const double* A, int m, int b, const int* perm, double* scratch,
                                                 double* S, const long long* __restrict__ row_off,
                                                 const long long* __restrict__ lu_off,
                                                 const long long* __restrict__ sf_off, double* __restrict__ lu_out,
                                                 bool write_lu, double* __restrict__ sf_out, int* __restrict__ piv_out,
                                                 int* __restrict__ gsrc_out, int* __restrict__ lperm_out,
                                                 const int* __restrict__ src_pos, int pos_base,
                                                 bool maps_done = false) {
  const int tid = threadIdx.x;
  const long long ro = row_off[b];
  const long long off = lu_off[b];
  if (!maps_done && tid == 0) {
    for (int k = 0; k < m; ++k) piv_out[ro + k] = perm[k];
    // compose the sequential swaps (dense.cpp:74-75) into one gather map
    for (int k = 0; k < m; ++k) scratch[k] = (double)k;
    for (int k = 0; k < m; ++k) {
      const int p = perm[k];
      const double t2 = scratch[k];
      scratch[k] = scratch[p];
      scratch[p] = t2;
    }
  }
  __syncthreads();
  for (int s2 = tid; s2 < m && !maps_done; s2 += NT) {
    const int loc = (int)scratch[s2];
    gsrc_out[ro + s2] = src_pos ? src_pos[ro + loc] + pos_base : (int)(ro + loc);
    lperm_out[ro + s2] = loc;
  }
  if (lu_out && write_lu)
    for (long long e = tid; e < (long long)m * m; e += NT) lu_out[off + e] = A[e];

  // ---- solve format: tile inverses + packed panels
  double* dst = sf_out + sf_off[b];
  const int P = (m + 31) / 32;
  long long po = 0;
  for (int p = 0; p < P; ++p) {
    const PanelGeom g(m, p);
    const int k0 = g.k0, kb = g.kb;
    if (!REG_TILE) {
      tile_inverses(A, m, k0, kb, S, tid);
    } else if (NT >= 64) {
      if (tid < 64) tile_inverse_warp(A, m, k0, kb, S, tid & 31, tid >> 5);
    } else {
      tile_inverse_warp(A, m, k0, kb, S, tid, 0);
      tile_inverse_warp(A, m, k0, kb, S, tid, 1);
    }
    __syncthreads();
    double* fw = dst + po;
    for (int e = tid; e < 32 * 32; e += NT) {
      const int kk = e >> 5, i = e & 31;
      if (kk < kb && i < kb && i > kk) fw[ltri_col(kb, kk) + i - kk - 1] = S[kk * kTileLd + i];
    }
    if (tid == 0 && g.lte > g.lt) fw[g.lt] = 0.0;
    double* lp = fw + g.lte;
    for (int e = tid; e < g.hLe * kb; e += NT) {
      const int kk = e / g.hLe, r = e % g.hLe;
      lp[e] = r < g.hL ? A[(size_t)(k0 + kk) * m + k0 + kb + r] : 0.0;
    }
    double* bw = fw + g.fwd_size();
    for (int e = tid; e < 32 * 32; e += NT) {
      const int jj = e >> 5, i = e & 31;
      if (jj < kb && i <= jj) bw[utri_col(jj) + i] = S[jj * kTileLd + i];
    }
    if (tid == 0 && g.ute > g.ut) bw[g.ut] = 0.0;
    double* up = bw + g.ute;
    for (int e = tid; e < k0 * kb; e += NT) {
      const int jj = e / k0, r = e % k0;
      up[e] = A[(size_t)(k0 + jj) * m + r];
    }
    po += g.size();
    __syncthreads();
  }
}

// Factor one block per CTA (DenseFactorization ctor, dense.cpp:31-67), then
// write the solve format (tile inverses + packed panels, see PanelGeom).
// src: column-major input (same offsets as lu_off). The block is staged in
// dynamic shared memory (m <= 164 fits 227 KB).
// lu_out (optional) receives the bit-exact LU in column-major order.
// dynamic smem (doubles): [A: m*m][rowmax: m][perm: m ints][scratch: 32*32]
template <int NT>
__global__ void __launch_bounds__(NT)
    lu_factor_kernel(const int* __restrict__ blist, const int* __restrict__ msz,
                     const long long* __restrict__ lu_off, const long long* __restrict__ row_off,
                     const long long* __restrict__ sf_off, const double* __restrict__ src,
                     double* __restrict__ lu_out, double* __restrict__ sf_out,
                     int* __restrict__ piv_out, int* __restrict__ gsrc_out, int* __restrict__ lperm_out,
                     const int* __restrict__ src_pos, int pos_base, int* __restrict__ fail) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NW = NT / 32;
  __shared__ int s_p, s_fail;
  __shared__ double s_inv;
  const int b = blist[blockIdx.x];
  const int m = msz[b];
  const long long off = lu_off[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = smem;
  double* rowmax = smem + (size_t)m * m;
  int* perm = reinterpret_cast<int*>(rowmax + m);
  double* S = rowmax + m + (m + 1) / 2;
  for (long long e = tid; e < (long long)m * m; e += NT) A[e] = src[off + e];
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
      // multipliers of column k-1 (l = a_ik * inv, dense.cpp:58-61)
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
        // the sequential scan starts from best = |a_kk| (dense.cpp:42-49)
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
    if (tid == 0) perm[k] = p;
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
  lu_write_outputs<NT, false>(A, m, b, perm, rowmax, S, row_off, lu_off, sf_off, lu_out, true, sf_out,
                       piv_out, gsrc_out, lperm_out, src_pos, pos_base);
}

// One elimination step k = K of lu_reg_kernel, recursing to K + 1: the
// step index is a template parameter so every register index is a
// compile-time constant (a rolled loop would put the row array in local
// memory). m is uniform per CTA. One CTA barrier per step: each warp's
// best candidate row publishes itself in a per-warp slot (double-buffered
// by step parity) before the barrier; after it every thread picks the
// winning slot. Slot layout (16-B aligned doubles): [0] |pivot| bits + 1
// (0 = no candidate), [1] logical row | singular flag << 30, then the row
// with the pivot's reciprocal at index K. Returns true on a singular pivot.
template <int MM>
struct LuSlot {
  static constexpr int kStride = MM + 2;  // even: keeps every slot 16-B aligned
};
__device__ __forceinline__ unsigned long long lu_vkey(double v) {
  return (unsigned long long)__double_as_longlong(v) + (1ull << 32);
}
template <int K, int MM, int NW>
struct LuRegStep {
  static __device__ __forceinline__ bool run(double (&a)[MM], double rmax, int& pos, int m, int t, double* slots,
                                             int* perm) {
    constexpr int kNone = 1 << 20;
    constexpr int kStride = LuSlot<MM>::kStride;
    if (K >= m) return false;
    const int lane = t & 31, warp = t >> 5;
    constexpr int buf = K & 1;
    // candidate of this row; its reciprocal is formed off the critical path
    const bool cand = pos >= K && pos < m;
    const double my_inv = 1.0 / a[K];
    // warp argmax of (|a_k|, -row): |a| >= 0 orders like its bit pattern,
    // so three redux steps (high word, low word, lowest row) replace the
    // shuffle tree
    const unsigned long long vb = cand ? lu_vkey(fabs(a[K])) : 0ull;
    const unsigned hi = (unsigned)(vb >> 32), lo = (unsigned)vb;
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    const unsigned key = __reduce_min_sync(kFull, (cand && hi == mh && lo == ml) ? (unsigned)pos : (unsigned)kNone);
    double* slot = slots + (size_t)(buf * NW + warp) * kStride;
    if (mh == 0) {  // no candidate row in this warp: an empty slot
      if (lane == 0) slot[0] = __longlong_as_double(0);
    } else if ((unsigned)pos == key) {  // this warp's best row publishes itself
      const int bad = fabs(a[K]) <= 1e-14 * fmax(rmax, 1e-300);
      reinterpret_cast<double2*>(slot)[0] =
          make_double2(__longlong_as_double((long long)vb), __longlong_as_double((long long)(key | (bad << 30))));
      // the row (reciprocal at K) in 16-B pairs; slot + 2 is 16-B aligned
      double2* r2 = reinterpret_cast<double2*>(slot + 2);
#pragma unroll
      for (int j = K & ~1; j < MM; j += 2)
        r2[j >> 1] = make_double2(j == K ? my_inv : a[j], j + 1 == K ? my_inv : a[j + 1]);
    }
    if (NW > 1) __syncthreads();
    else __syncwarp();
    // the reference scan starts from |a_kk| and keeps the first strictly
    // larger value: the maximum at the lowest logical row
    int ws = buf * NW;
    unsigned long long bv = (unsigned long long)__double_as_longlong(slots[(size_t)ws * kStride]);
    int bk = (int)__double_as_longlong(slots[(size_t)ws * kStride + 1]);
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const double2 o = reinterpret_cast<const double2*>(slots + (size_t)(buf * NW + w) * kStride)[0];
      const unsigned long long ov = (unsigned long long)__double_as_longlong(o.x);
      const int ok = (int)__double_as_longlong(o.y);
      if (ov > bv || (ov == bv && (ok & 0x3fffffff) < (bk & 0x3fffffff))) {
        bv = ov;
        bk = ok;
        ws = buf * NW + w;
      }
    }
    if (NW == 1) bk = (int)__double_as_longlong(slots[(size_t)ws * kStride + 1]);
    const int p = bk & 0x3fffffff;
    if (t == 0) perm[K] = p;
    pos = (pos == p) ? K : (pos == K ? p : pos);
    if (bk >> 30) return true;
    if (pos > K && pos < m) {
      const double2* r2 = reinterpret_cast<const double2*>(slots + (size_t)ws * kStride + 2);
      const double2 first = r2[K >> 1];
      const double l = mul_rn(a[K], (K & 1) ? first.y : first.x);
      a[K] = l;
      if (!(K & 1) && K + 1 < MM) a[K + 1] = sub_rn(a[K + 1], mul_rn(l, first.y));
#pragma unroll
      for (int j = (K + 2) & ~1; j < MM; j += 2) {
        const double2 u = r2[j >> 1];
        a[j] = sub_rn(a[j], mul_rn(l, u.x));
        a[j + 1] = sub_rn(a[j + 1], mul_rn(l, u.y));
      }
    }
    if constexpr (K + 1 < MM) return LuRegStep<K + 1, MM, NW>::run(a, rmax, pos, m, t, slots, perm);
    return false;
  }
};

// Register-resident LU for small blocks (m <= MM <= 64): one thread per
// block row, the row held in registers (a[MM], compile-time indexed: the
// elimination loop is fully unrolled). Row interchanges are not data moves:
// each thread tracks the logical position `pos` of its physical row, and a
// swap (k, p) only exchanges two positions. This is the same sequence of
// rounded operations per entry as DenseFactorization (dense.cpp:31-67):
//   * pivot = largest |a_ik| over logical rows i >= k, ties to the lowest
//     logical row (the reference's first-strictly-larger scan),
//   * row_max travels with its row (it is per thread), singular test
//     |pivot| <= 1e-14 * max(row_max, 1e-300),
//   * l = a_ik * (1/pivot), then a_ij = a_ij - l * a_kj, non-fused, k ascending.
// Per step: a shuffle argmax per warp + one cross-warp combine, the pivot
// thread publishes its row in shared memory, every active row updates its
// registers. Two CTA barriers per step and no shared-memory traffic for the
// trailing matrix. The finished rows are placed at their logical positions
// in shared memory and the common writer produces the solve format.
// dynamic smem (doubles): [A: m*m][scratch: m][perm: m ints][S: 32*kTileLd]
template <int MM>
__global__ void __launch_bounds__(MM <= 32 ? 32 : 64)
    lu_reg_kernel(const int* __restrict__ blist, const int* __restrict__ msz, const long long* __restrict__ lu_off,
                  const long long* __restrict__ row_off, const long long* __restrict__ sf_off,
                  const double* __restrict__ src, double* __restrict__ lu_out, double* __restrict__ sf_out,
                  int* __restrict__ piv_out, int* __restrict__ gsrc_out, int* __restrict__ lperm_out,
                  const int* __restrict__ src_pos, int pos_base, int* __restrict__ fail) {
  constexpr int NT = MM <= 32 ? 32 : 64;
  constexpr int NW = NT / 32;
  constexpr int kNone = 1 << 20;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(16) double s_slots[2 * NW * LuSlot<MM>::kStride];
  const int b = blist[blockIdx.x];
  const int m = msz[b];
  const long long off = lu_off[b];
  const int t = threadIdx.x;
  double* A = smem;
  double* scratch = smem + (size_t)m * m;
  int* perm = reinterpret_cast<int*>(scratch + m);
  double* S = scratch + m + (m + 1) / 2;

  double a[MM];
  const bool valid = t < m;
#pragma unroll
  for (int j = 0; j < MM; ++j) a[j] = (valid && j < m) ? __ldg(src + off + (size_t)j * m + t) : 0.0;
  double rmax = 0.0;
#pragma unroll
  for (int j = 0; j < MM; ++j) rmax = fmax(rmax, fabs(a[j]));
  int pos = valid ? t : kNone;
  if (LuRegStep<0, MM, NW>::run(a, rmax, pos, m, t, s_slots, perm)) {
    if (t == 0) atomicMin(fail, b);
    return;
  }
  // rows to their logical positions, column-major. The swaps applied to the
  // right-hand side (dense.cpp:74-75) move entry t to the final position of
  // row t, so each thread writes its own gather-map entry.
  const long long ro = row_off[b];
  if (valid) {
#pragma unroll
    for (int j = 0; j < MM; ++j)
      if (j < m) A[(size_t)j * m + pos] = a[j];
    gsrc_out[ro + pos] = src_pos ? src_pos[ro + t] + pos_base : (int)(ro + t);
    lperm_out[ro + pos] = t;
    piv_out[ro + t] = perm[t];
  }
  __syncthreads();
  lu_write_outputs<NT, true>(A, m, b, perm, scratch, S, row_off, lu_off, sf_off, lu_out, true, sf_out, piv_out,
                             gsrc_out, lperm_out, src_pos, pos_base, /*maps_done=*/true);
}

// ---------------------------------------------------------------- blocked LU (m > 164)
// Right-looking LU in panels of kBigNB columns for the large blocks (the
// pure-DD Vanka patches of config 4, m ~ 500-780), factored in place in
// global memory (column-major), one launch pair per panel for the whole
// batch:
//   lu_big_panel_smem_kernel (one CTA per block): for each panel column k
//     the pivot search (largest |a_ik|, lowest row on ties), the swap of
//     rows k and p (and of their original row maxima), the singular test,
//     l = a_ik * (1/pivot), the rank-1 update of the remaining panel
//     columns; then the panel rows of the trailing columns (U12): per
//     column, a_ij -= l_ik * a_kj for k = k0..i-1 in order;
//   lu_big_update_r4_kernel (a CTA per 64-row strip of A22): a_ij -= l_ik *
//     u_kj for the panel's k in order, non-fused, from register tiles.
// Every entry therefore receives the reference's rounded updates in the
// reference's k order (DenseFactorization, dense.cpp:31-67): the factors
// are bit-identical. Row swaps move whole rows immediately, as the
// reference does.
constexpr int kBigNB = 32;
constexpr int kBigTile = 64;

__global__ void __launch_bounds__(256) lu_big_init_kernel(const int* __restrict__ blist, const int* __restrict__ msz,
                                                          const long long* __restrict__ lu_off,
                                                          const long long* __restrict__ row_off,
                                                          const double* __restrict__ src, double* __restrict__ work,
                                                          double* __restrict__ rowmax, int* __restrict__ bad) {
  const int bi = blockIdx.x;
  const int b = blist[bi];
  const int m = msz[b];
  const long long off = lu_off[b], ro = row_off[b];
  // one pass over the block: a warp takes 32 consecutive rows (coalesced
  // columns) over one of 8 column slices, copies them and folds |a_ij| into
  // the row maximum; the slices combine by an integer max on the bit
  // patterns (non-negative doubles order as unsigned), exact and
  // order-independent like fmax
  unsigned long long* rmu = reinterpret_cast<unsigned long long*>(rowmax + ro);
  for (int i = threadIdx.x; i < m; i += blockDim.x) rmu[i] = 0ull;
  __syncthreads();
  constexpr int S = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int chunks = (m + 31) / 32;
  for (int it = warp; it < chunks * S; it += nw) {
    const int i = (it / S) * 32 + lane, s = it % S;
    if (i >= m) continue;
    const int j0 = s * m / S, j1 = (s + 1) * m / S;
    double mx = 0.0;
    const double* sp = src + off + i;
    double* wp = work + off + i;
    // 8 loads in flight before their stores (src may alias work, so the
    // compiler cannot hoist loads over the stores by itself)
    constexpr int U = 8;
    int j = j0;
    for (; j + U <= j1; j += U) {
      double v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) v[q] = sp[(size_t)(j + q) * m];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if (src != work) wp[(size_t)(j + q) * m] = v[q];
        mx = fmax(mx, fabs(v[q]));
      }
    }
    for (; j < j1; ++j) {
      const double v = sp[(size_t)j * m];
      if (src != work) wp[(size_t)j * m] = v;
      mx = fmax(mx, fabs(v));
    }
    atomicMax(rmu + i, (unsigned long long)__double_as_longlong(mx));
  }
  if (threadIdx.x == 0) bad[bi] = 0;
}

// (column-major, ld = m - k0; 200 KB at m = 780), so the 32 pivot steps
// (search, swap, scale, rank-1 update of the panel) run out of shared memory
// instead of making L2 round trips per column. The row swaps of the columns
// outside the panel are deferred to the end of the panel and applied in k
// order (no other column is read or written in between, so the result is
// the same as swapping whole rows immediately); U12 then reads L11 from
// shared memory. Same rounded operations in the same order: bit-identical.
constexpr int kBigPanelMaxM = 850;  // panel (m * 32 doubles) + row maxima (m) <= 227 KB
// 256 threads (measured: 512 threads slow the panel launch from 289 to 355 us,
// the longer barriers outweigh the shorter per-thread row loops)
constexpr int kPanelThreads = 256;
__global__ void __launch_bounds__(kPanelThreads, 1)
    lu_big_panel_smem_kernel(const int* __restrict__ blist, const int* __restrict__ msz,
                             const long long* __restrict__ lu_off, const long long* __restrict__ row_off,
                             double* work, double* rowmax, int* __restrict__ piv, int* bad, int* __restrict__ fail,
                             int k0) {
  extern __shared__ __align__(16) double P[];
  const int bi = blockIdx.x;
  const int b = blist[bi];
  const int m = msz[b];
  if (k0 >= m || bad[bi]) return;
  const long long off = lu_off[b], ro = row_off[b];
  double* A = work + off;
  double* rm = rowmax + ro;
  const int kb = min(kBigNB, m - k0);
  const int ld = m - k0;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __shared__ double s_v[kPanelThreads / 32];
  __shared__ int s_i[kPanelThreads / 32];
  __shared__ int s_p, s_bad;
  __shared__ int s_perm[kBigNB];
  // (loops are column-outer / row-inner: no per-element integer division)
  // the remaining rows' original maxima (singular test) follow the panel, so
  // the per-step test and swap never wait on a global load
  double* R = P + (size_t)ld * kb;
  // panel columns arrive by TMA bulk copies (one per column, one mbarrier)
  // when every column start is 16-byte aligned (even m and block offset);
  // ncu showed the per-thread loads of the panel as the top stall at one
  // CTA per SM. Otherwise plain loads.
  __shared__ __align__(8) unsigned long long s_bar;
  const bool bulk = ((off | m) & 1) == 0;
  if (bulk) {
    if (t == 0) {
      mbar_init(&s_bar, 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (t == 0) {
      mbar_arrive_expect_tx(&s_bar, (unsigned)(ld * kb * 8));
      for (int q = 0; q < kb; ++q)
        tma_bulk_g2s(P + (size_t)q * ld, A + (size_t)(k0 + q) * m + k0, (unsigned)(ld * 8), &s_bar);
    }
  } else {
    for (int q = 0; q < kb; ++q)
      for (int i = t; i < ld; i += blockDim.x) P[(size_t)q * ld + i] = A[(size_t)(k0 + q) * m + k0 + i];
  }
  for (int i = t; i < ld; i += blockDim.x) R[i] = rm[k0 + i];
  if (bulk) mbar_wait(&s_bar, 0);
  __syncthreads();
  for (int k = k0; k < k0 + kb; ++k) {
    const int kq = k - k0;
    double* Pk = P + (size_t)kq * ld;  // column k; local row i - k0
    double best = -1.0;
    int bidx = m;
    for (int i = k + t; i < m; i += blockDim.x) {
      const double v = fabs(Pk[i - k0]);
      if (v > best) {
        best = v;
        bidx = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(kFull, best, o);
      const int oi = __shfl_xor_sync(kFull, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    if (lane == 0) {
      s_v[warp] = best;
      s_i[warp] = bidx;
    }
    __syncthreads();
    if (t == 0) {
      double bv = s_v[0];
      int bx = s_i[0];
      for (int w = 1; w < kPanelThreads / 32; ++w)
        if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bx)) {
          bv = s_v[w];
          bx = s_i[w];
        }
      int p = bx < m ? bx : k;
      if (!(fabs(Pk[kq]) < bv)) p = k;
      s_p = p;
      const double pivot = Pk[p - k0];
      const int bd = fabs(pivot) <= 1e-14 * fmax(R[p - k0], 1e-300);
      s_bad = bd;
      piv[ro + k] = p;
      s_perm[kq] = p;
      if (!bd && p != k) {
        const double r0 = R[kq];
        R[kq] = R[p - k0];
        R[p - k0] = r0;
      }
    }
    __syncthreads();
    if (s_bad) {
      if (t == 0) {
        bad[bi] = 1;
        atomicMin(fail, b);
      }
      return;
    }
    const int p = s_p;
    if (p != k && t < kb) {
      double* c = P + (size_t)t * ld;
      const double a0 = c[kq];
      c[kq] = c[p - k0];
      c[p - k0] = a0;
    }
    __syncthreads();
    const double inv = 1.0 / Pk[kq];
    for (int i = k + 1 + t; i < m; i += blockDim.x) Pk[i - k0] = mul_rn(Pk[i - k0], inv);
    __syncthreads();
    // rank-1 update of the panel columns right of k: each thread keeps the
    // multipliers of its rows in registers across the columns
    constexpr int kRows = (kBigPanelMaxM + kPanelThreads - 1) / kPanelThreads;
    double lr[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int i = kq + 1 + t + r * kPanelThreads;
      lr[r] = i < ld ? Pk[i] : 0.0;
    }
    for (int jq = kq + 1; jq < kb; ++jq) {
      double* c = P + (size_t)jq * ld;
      const double u = c[kq];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int i = kq + 1 + t + r * kPanelThreads;
        if (i < ld) c[i] = sub_rn(c[i], mul_rn(lr[r], u));
      }
    }
    __syncthreads();
  }
  for (int q = 0; q < kb; ++q)
    for (int i = t; i < ld; i += blockDim.x) A[(size_t)(k0 + q) * m + k0 + i] = P[(size_t)q * ld + i];
  for (int i = t; i < ld; i += blockDim.x) rm[k0 + i] = R[i];
  // deferred row swaps of the columns left and right of the panel, in k order
  for (int j = t; j < m - kb; j += blockDim.x) {
    const int jc = j < k0 ? j : j + kb;
    double* col = A + (size_t)jc * m;
    for (int q = 0; q < kb; ++q) {
      const int p = s_perm[q];
      if (p != k0 + q) {
        const double a0 = col[k0 + q];
        col[k0 + q] = col[p];
        col[p] = a0;
      }
    }
  }
  __syncthreads();
  // U12: panel rows of the trailing columns, L11 from shared memory
  for (int j = k0 + kb + t; j < m; j += blockDim.x) {
    double u[kBigNB];
#pragma unroll
    for (int q = 0; q < kBigNB; ++q) u[q] = q < kb ? A[(size_t)j * m + k0 + q] : 0.0;
#pragma unroll
    for (int i = 1; i < kBigNB; ++i)
#pragma unroll
      for (int q = 0; q < i; ++q)
        if (i < kb) u[i] = sub_rn(u[i], mul_rn(P[(size_t)q * ld + i], u[q]));
#pragma unroll
    for (int q = 1; q < kBigNB; ++q)
      if (q < kb) A[(size_t)j * m + k0 + q] = u[q];
  }
}

// A 1 x 16 strip tile was shared-memory bound (ncu: L1/TEX 86%, 10
// wavefronts per k for 16 mul/sub pairs per lane); here a warp is 16
// row lanes x 2 column groups, so per k it reads 4 L21 values (16 distinct
// doubles each, one wavefront) and 4 double2 U12 broadcasts (two addresses
// in disjoint banks, one wavefront): 8 wavefronts for 32 pairs per lane.
// Same per-entry operations in the same k order: bit-identical.
// grid = (tiles_r, blocks), 256 threads, RT = 2 rows x 8 columns per thread
// (124 registers, 16 warps per SM; measured 1% faster than 4 x 8 tiles at
// 242 registers; 2 x 8 at 3 CTAs per SM spills and runs 12% slower).
constexpr int kUpdRT = 2;
__global__ void __launch_bounds__(512 / kUpdRT, 2) lu_big_update_r4_kernel(const int* __restrict__ blist,
                                                               const int* __restrict__ msz,
                                                               const long long* __restrict__ lu_off,
                                                               double* work, const int* __restrict__ bad, int k0) {
  constexpr int RT = kUpdRT, NT = 512 / RT, CT = 8;  // RT rows x 8 columns per thread
  const int bi = blockIdx.y;
  const int b = blist[bi];
  const int m = msz[b];
  const int r0 = k0 + kBigNB + blockIdx.x * kBigTile;
  const int cbeg = k0 + kBigNB;
  if (r0 >= m || cbeg >= m || bad[bi]) return;
  double* A = work + lu_off[b];
  __shared__ __align__(16) double Ls[kBigNB][kBigTile];
  __shared__ __align__(16) double Us[kBigNB][kBigTile];
  const int t = threadIdx.x;
  const int rl = t & 15, cg = (t >> 4) & 7;  // row lane, 8-column group
  const int rb = r0 + (t >> 7) * (16 * RT);  // RT < 4: several row groups per CTA
  constexpr int UPT = kBigNB * kBigTile / NT;
  for (int e = t; e < kBigNB * kBigTile; e += NT) {
    const int k = e / kBigTile, i = e % kBigTile;
    Ls[k][i] = r0 + i < m ? A[(size_t)(k0 + k) * m + r0 + i] : 0.0;
  }
  double nxt[RT][CT], un[UPT];
  auto load_tile = [&](int c0) {
#pragma unroll
    for (int jj = 0; jj < CT; ++jj) {
      const int c = c0 + cg * CT + jj;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int r = rb + rl + 16 * i;
        nxt[i][jj] = (r < m && c < m) ? A[(size_t)c * m + r] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      const int e = t + q * NT;
      const int j = e / kBigNB, k = e % kBigNB;  // coalesced over k
      un[q] = c0 + j < m ? A[(size_t)(c0 + j) * m + k0 + k] : 0.0;
    }
  };
  load_tile(cbeg);
  for (int c0 = cbeg; c0 < m; c0 += kBigTile) {
    __syncthreads();  // previous tile's Us reads are done
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      const int e = t + q * NT;
      Us[e % kBigNB][e / kBigNB] = un[q];
    }
    double acc[RT][CT];
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int jj = 0; jj < CT; ++jj) acc[i][jj] = nxt[i][jj];
    __syncthreads();
    if (c0 + kBigTile < m) load_tile(c0 + kBigTile);  // in flight during the math below
#pragma unroll 8
    for (int k = 0; k < kBigNB; ++k) {
      double l[RT], u[CT];
#pragma unroll
      for (int i = 0; i < RT; ++i) l[i] = Ls[k][rb - r0 + rl + 16 * i];
#pragma unroll
      for (int q = 0; q < CT; q += 2) {
        const double2 uu = *reinterpret_cast<const double2*>(&Us[k][cg * CT + q]);
        u[q] = uu.x;
        u[q + 1] = uu.y;
      }
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int jj = 0; jj < CT; ++jj) acc[i][jj] = sub_rn(acc[i][jj], mul_rn(l[i], u[jj]));
    }
#pragma unroll
    for (int jj = 0; jj < CT; ++jj) {
      const int c = c0 + cg * CT + jj;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int r = rb + rl + 16 * i;
        if (r < m && c < m) A[(size_t)c * m + r] = acc[i][jj];
      }
    }
  }
}

// Outputs of the blocked LU: gather map from the pivots, optional LU copy,
// solve format (lu_write_outputs on the factor in global memory).
// dynamic smem (doubles): [scratch: m][perm: m ints][S: 32*kTileLd]
__global__ void __launch_bounds__(256) lu_big_finish_kernel(const int* __restrict__ blist, const int* __restrict__ msz,
                                                            const long long* __restrict__ lu_off,
                                                            const long long* __restrict__ row_off,
                                                            const long long* __restrict__ sf_off,
                                                            const double* __restrict__ work,
                                                            double* __restrict__ sf_out, int* __restrict__ piv,
                                                            int* __restrict__ gsrc_out, int* __restrict__ lperm_out,
                                                            const int* __restrict__ src_pos, int pos_base,
                                                            const int* __restrict__ bad) {
  extern __shared__ __align__(16) double smem[];
  const int bi = blockIdx.x;
  if (bad[bi]) return;
  const int b = blist[bi];
  const int m = msz[b];
  const long long ro = row_off[b];
  double* scratch = smem;
  int* perm = reinterpret_cast<int*>(scratch + m);
  double* S = scratch + m + (m + 1) / 2;
  for (int k = threadIdx.x; k < m; k += blockDim.x) perm[k] = piv[ro + k];
  __syncthreads();
  lu_write_outputs<256, false>(work + lu_off[b], m, b, perm, scratch, S, row_off, lu_off, sf_off, nullptr, false,
                               sf_out, piv, gsrc_out, lperm_out, src_pos, pos_base);
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
