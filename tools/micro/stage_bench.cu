// Microbenchmark: vector CSR vs shared-memory staged CSR variants on a
// synthetic FS-like matrix (rows of ~NNZ entries in two column windows).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stage_bench.cu -o stage_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "../../include/fsigpu.h"
#include "../../paper_1909_13201_b200/csrc/common.cuh"
#include "../../paper_1909_13201_b200/csrc/sparse.cuh"
using namespace fsigpu;

// variant: plain cooperative staging (no TMA)
template <int LPR, int U = 8>
__global__ void __launch_bounds__(256) staged_plain(const int* rb, const int* ptr, const int* idx, const double* val,
                                                    int cap, GatherPlain gx, EpiPlain epi) {
  extern __shared__ __align__(128) unsigned char stage[];
  double* s_val = reinterpret_cast<double*>(stage);
  int* s_idx = reinterpret_cast<int*>(stage + 8 * (size_t)((cap + 3) & ~1));
  const int t = threadIdx.x;
  const int r0 = rb[blockIdx.x], r1 = rb[blockIdx.x + 1];
  const int k0 = ptr[r0], k1 = ptr[r1];
  for (int k = k0 + t; k < k1; k += 256) {
    s_val[k - k0] = __ldg(val + k);
    s_idx[k - k0] = __ldg(idx + k);
  }
  __syncthreads();
  for (int kb = k0 + t; kb < k1; kb += 256 * U) {
    int c[U];
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + 256 * u;
      c[u] = k < k1 ? s_idx[k - k0] : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? gx(c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + 256 * u;
      if (k < k1) s_val[k - k0] *= xv[u];
    }
  }
  __syncthreads();
  const int lane = t & (LPR - 1);
  for (int base = r0; base < r1; base += 256 / LPR) {
    const int row = base + t / LPR;
    const bool ok = row < r1;
    const int a = ok ? ptr[row] : 0, b = ok ? ptr[row + 1] : 0;
    double s = 0.0;
    for (int k = a + lane; k < b; k += LPR) s += s_val[k - k0];
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o, LPR);
    if (ok && lane == 0) epi(row, s);
  }
}
// variant: TMA copy only
__global__ void __launch_bounds__(256) copy_only(const int* rb, const int* ptr, const int* idx, const double* val,
                                                 int cap, double* out) {
  extern __shared__ __align__(128) unsigned char stage[];
  __shared__ __align__(8) unsigned long long bar;
  double* s_val = reinterpret_cast<double*>(stage);
  int* s_idx = reinterpret_cast<int*>(stage + 8 * (size_t)((cap + 3) & ~1));
  const int t = threadIdx.x;
  const int r0 = rb[blockIdx.x], r1 = rb[blockIdx.x + 1];
  const int k0 = ptr[r0], k1 = ptr[r1];
  const int kv0 = k0 & ~1, ki0 = k0 & ~3;
  const unsigned bv = 8u * (unsigned)(((k1 + 1) & ~1) - kv0);
  const unsigned bi = 4u * (unsigned)(((k1 + 3) & ~3) - ki0);
  if (t == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  __syncthreads();
  if (t == 0) {
    mbar_arrive_expect_tx(&bar, bv + bi);
    tma_bulk_g2s(s_val, val + kv0, bv, &bar);
    tma_bulk_g2s(s_idx, idx + ki0, bi, &bar);
  }
  mbar_wait(&bar, 0);
  if (t == 0) out[blockIdx.x] = s_val[t] + s_idx[t];
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 20000;
  const int nnzr = argc > 2 ? atoi(argv[2]) : 270;
  std::mt19937 rng(1);
  std::vector<int> hp(n + 1), hi;
  std::vector<double> hv;
  hp[0] = 0;
  for (int r = 0; r < n; ++r) {
    const int len = nnzr / 2 + (int)(rng() % (unsigned)nnzr);
    std::vector<int> cols;
    for (int k = 0; k < len; ++k) {
      const int w = (k & 1) ? n / 2 : 0;
      int c = (r / 2 + w + (int)(rng() % 2000)) % n;
      cols.push_back(c);
    }
    std::sort(cols.begin(), cols.end());
    for (int c : cols) { hi.push_back(c); hv.push_back(1e-3 * (rng() % 1000)); }
    hp[r + 1] = (int)hi.size();
  }
  const long long nnz = hi.size();
  printf("n %d nnz %lld (%.1f/row) matrix %.1f MB\n", n, nnz, (double)nnz / n, nnz * 12e-6);
  int *dp, *di, *drb; double *dv, *dx, *dy, *dout, *flush;
  cudaMalloc(&dp, 4 * (n + 1)); cudaMalloc(&di, 4 * (nnz + 8)); cudaMalloc(&dv, 8 * (nnz + 8));
  cudaMalloc(&dx, 8 * n); cudaMalloc(&dy, 8 * n); cudaMalloc(&flush, 256 << 20);
  cudaMemcpy(dp, hp.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(di, hi.data(), 4 * nnz, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), 8 * nnz, cudaMemcpyHostToDevice);
  std::vector<double> hx(n, 1.0); cudaMemcpy(dx, hx.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, bool cold) {
    float best = 1e9, tot = 0;
    for (int it = 0; it < 12; ++it) {
      if (cold) cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { tot += ms; best = std::min(best, ms); }
    }
    cudaError_t err = cudaGetLastError();
    printf("%-28s %s avg %8.2f us  best %8.2f us  %7.0f GB/s %s\n", name, cold ? "cold" : "warm", tot / 10 * 1000,
           best * 1000, nnz * 12.0 / (tot / 10) / 1e6, err ? cudaGetErrorString(err) : "");
  };
  for (int cold = 0; cold < 2; ++cold) {
    timeit("vector lpr32 u4", [&] { csr_kernel<32, GatherPlain, EpiPlain, 4><<<(n * 32 + 255) / 256, 256>>>(n, dp, di, dv, GatherPlain{dx}, EpiPlain{dy}); }, cold);
    timeit("vector lpr16 u4", [&] { csr_kernel<16, GatherPlain, EpiPlain, 4><<<(n * 16 + 255) / 256, 256>>>(n, dp, di, dv, GatherPlain{dx}, EpiPlain{dy}); }, cold);
    for (int cap : {1024, 2048, 4096, 8192}) {
      std::vector<int> b{0};
      int r = 0;
      while (r < n) {
        long long e = 0;
        const int beg = r;
        while (r < n && e + (hp[r + 1] - hp[r]) <= cap) e += hp[r + 1] - hp[r], ++r;
        if (r == beg) { r = -1; break; }
        b.push_back(r);
      }
      if (r < 0) continue;
      const int nb = (int)b.size() - 1;
      cudaMalloc(&drb, 4 * b.size());
      cudaMalloc(&dout, 8 * nb);
      cudaMemcpy(drb, b.data(), 4 * b.size(), cudaMemcpyHostToDevice);
      const size_t sm = 8 * (size_t)((cap + 3) & ~1) + 4 * (size_t)(cap + 8);
      cudaFuncSetAttribute(csr_staged_kernel<32, GatherPlain, EpiPlain>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(staged_plain<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(copy_only, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      char nm[64];
      snprintf(nm, 64, "staged tma cap%d (%d cta)", cap, nb);
      timeit(nm, [&] { csr_staged_kernel<32, GatherPlain, EpiPlain><<<nb, 256, sm>>>(drb, dp, di, dv, cap, GatherPlain{dx}, EpiPlain{dy}); }, cold);
      snprintf(nm, 64, "staged plain cap%d", cap);
      timeit(nm, [&] { staged_plain<32><<<nb, 256, sm>>>(drb, dp, di, dv, cap, GatherPlain{dx}, EpiPlain{dy}); }, cold);
      snprintf(nm, 64, "copy only cap%d", cap);
      timeit(nm, [&] { copy_only<<<nb, 256, sm>>>(drb, dp, di, dv, cap, dout); }, cold);
      cudaFree(drb); cudaFree(dout);
    }
  }
  return 0;
}
