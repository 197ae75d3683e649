// SPDX-License-Identifier: Apache-2.0
// Shared device/host helpers for libfsigpu (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace fsigpu {

// Error carrying a C-ABI status code (see include/fsigpu.h).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FSI_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::fsigpu::Error(FSIGPU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define FSI_CHECK_LAUNCH() FSI_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(FSIGPU_ERR_INVALID, msg);
}

// Owning device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = true;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), owned(o.owned) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      owned = o.owned;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  // Move the contents into caller-owned device memory (an arena slice) and
  // keep only a non-owning view.
  void rebase(T* dst, cudaStream_t s) {
    if (n) FSI_CUDA(cudaMemcpyAsync(dst, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    FSI_CUDA(cudaStreamSynchronize(s));
    const size_t keep = n;
    release();
    p = dst;
    n = keep;
    owned = false;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    owned = true;
    n = count;
    if (count) FSI_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    n = 0;
    owned = true;
  }
  void upload(const T* h, size_t count, cudaStream_t s = 0) {
    if (count != n) alloc(count);
    if (count) FSI_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s = 0) { upload(v.data(), v.size(), s); }
  std::vector<T> download(cudaStream_t s = 0) const {
    std::vector<T> h(n);
    if (n) {
      FSI_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
      FSI_CUDA(cudaStreamSynchronize(s));
    }
    return h;
  }
  void zero(cudaStream_t s = 0) {
    if (n) FSI_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Non-fused double ops: the reference is built with -ffp-contract=off
// (proj/CMakeLists.txt:10-12); using explicit round-to-nearest mul/sub keeps
// the LU, the forward substitution and the FS glue bit-identical to it.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch (sm_90+): a kernel lets its dependents be
// scheduled immediately and waits for its producers only before touching
// their data. Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- device-clock launch stamps (opt-in profiling of kernels INSIDE a CUDA graph) ----
// A slot is four u64: {start, end, accumulated ns, launches}. Thread 0 of CTA
// 0 folds the previous launch of the same graph node into the accumulator on
// entry, and stamps `start` once the launch's dependencies are resolved
// (after griddepcontrol.wait); thread 0 of every CTA raises `end` with a
// fire-and-forget atomic max on exit. Duration = last CTA exit - dependency
// release. A null slot (the default) costs one predicated branch.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp_fold(unsigned long long* slot) {
  if (slot && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const unsigned long long s0 = slot[0], e0 = *(volatile unsigned long long*)(slot + 1);
    if (s0 && e0 > s0) {
      slot[2] += e0 - s0;
      slot[3] += 1;
    }
    slot[0] = 0;
  }
}
__device__ __forceinline__ void stamp_start(unsigned long long* slot) {
  if (slot && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) slot[0] = global_ns();
}
__device__ __forceinline__ void stamp_end(unsigned long long* slot) {
  if (slot && threadIdx.x == 0) atomicMax(slot + 1, global_ns());
}

// ---- mbarrier + bulk-copy (TMA, non-tensor) helpers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Bulk prefetch of [src, src + bytes) into L2 (16-B aligned, multiple of 16).
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Per-thread asynchronous 8-byte global -> shared copies (LDGSTS), grouped
// by commit; wait_group<N> leaves at most N newest groups in flight.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace fsigpu
