// GMRES(1) (minimal-residual) level smoother, BASELINE.json configs[0]:
// "1 pre- and 1 post-step GMRES(1) with FS". The reference only ships the
// damped Richardson smoother (precond.cpp:305-317); this is the
// step-wise optimal variant of the same sweep:
//   r = b - A x ;  z = FS r ;  w = A z ;  alpha = (w.r)/(w.w) ;  x += alpha z
// (alpha = 0 when w = 0). The smoother is non-linear in b, so the outer
// solver must be flexible (FGMRES, which the device solver is). CPU
// restatement: oracle/fsi_oracle.c mr_smooth().
//
// Two kernels after the two SpMVs: k_mr_alpha reduces (w.r, w.w) over a
// FIXED grid (deterministic: per-CTA fixed trees, the last CTA sums the
// partials in CTA order) and writes alpha to device memory, so the sweep is
// graph-capturable; k_mr_update applies x = x + alpha z (optionally zeroing
// the level's constrained columns: last write of a coarse iterate, gmg.cpp:230-231).
#pragma once

namespace fsigpu {

constexpr int kMrThreads = 256;
constexpr int kMrCtas = 296;  // 2 per SM; fixed so the summation order never changes

__global__ void __launch_bounds__(kMrThreads) k_mr_alpha(int n, const double* __restrict__ w,
                                                         const double* __restrict__ r, double* part,
                                                         unsigned int* ticket, double* alpha) {
  pdl_trigger();
  pdl_wait();
  __shared__ double s_wr[kMrThreads / 32], s_ww[kMrThreads / 32];
  double wr = 0.0, ww = 0.0;
  for (int i = blockIdx.x * kMrThreads + threadIdx.x; i < n; i += kMrCtas * kMrThreads) {
    const double wi = __ldg(w + i);
    wr = fma(wi, __ldg(r + i), wr);
    ww = fma(wi, wi, ww);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wr += __shfl_xor_sync(kFull, wr, o);
    ww += __shfl_xor_sync(kFull, ww, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_wr[warp] = wr;
    s_ww[warp] = ww;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < kMrThreads / 32; ++q) a += s_wr[q], b += s_ww[q];
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
  // last CTA: fixed-order sum of the partials
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  if (warp == 0) {
    double a = 0.0, b = 0.0;
    for (int c = lane; c < kMrCtas; c += 32) {
      a += __ldcg(part + 2 * c);
      b += __ldcg(part + 2 * c + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(kFull, a, o);
      b += __shfl_xor_sync(kFull, b, o);
    }
    if (lane == 0) {
      *alpha = b > 0.0 ? a / b : 0.0;
      *ticket = 0;
    }
  }
}

// x = (x_zero ? 0 : x) + alpha z ; mask: constrained columns -> 0 (or null)
__global__ void __launch_bounds__(256) k_mr_update(int n, const double* __restrict__ alpha,
                                                   const double* __restrict__ z, double* __restrict__ x,
                                                   int x_zero, const unsigned char* __restrict__ mask) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  const double a = __ldg(alpha);
  const double xo = x_zero ? 0.0 : x[i];
  const double v = add_rn(xo, mul_rn(a, __ldg(z + i)));
  x[i] = (mask && mask[i]) ? 0.0 : v;
}

}  // namespace fsigpu
