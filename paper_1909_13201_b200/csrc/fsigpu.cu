// SPDX-License-Identifier: Apache-2.0
//
// libfsigpu: host orchestration and C ABI (include/fsigpu.h) of the B200
// FS-GMG-FGMRES solve path.  See DESIGN.md for the data layout and the
// kernel/roofline table; each object below names the reference class it
// stands in for.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <type_traits>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/reduce.h>
#include <thrust/scan.h>
#include <thrust/sort.h>

#include "../../include/fsigpu.h"
#include "common.cuh"
#include "dense.cuh"
#include "krylov.cuh"
#include "krylov_wide.cuh"
#include "sparse.cuh"
#include "mr.cuh"
#include "mult.cuh"
#include "sets.cuh"

namespace fsigpu {

// ------------------------------------------------------------ launches
// Solve-path kernels are launched with programmatic stream serialization
// (PDL): inside the captured graphs consecutive kernels overlap launch and
// prologue with the predecessor's tail (kernels call pdl_trigger/pdl_wait).
// on by default: the kernels fetch their setup data (matrix rows) before
// griddepcontrol.wait, which overlaps it with the predecessor's tail
// (config 0: 8.45 -> 7.96 ms per solve, tools/ab_pdl.py)
static std::atomic<bool> g_pdl{true};
template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw Error(FSIGPU_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
}

// ------------------------------------------------------------ errors
static thread_local std::string g_err;
static thread_local int g_bad_block = -1;
static thread_local int g_bad_level = -1;  // GMG level of the failing block (-1: standalone batch)

// ------------------------------------------------------------ profiler
struct Profiler {
  bool on = false;
  struct Rec {
    int cls;
    double bytes;
    cudaEvent_t a, b;
    int lvl;
  };
  // GMG level the current launches belong to (set by Gmg::cycle; -1 outside)
  int level = -1;
  static constexpr int kLv = 32;
  double lv_ms[FSIGPU_K_COUNT][kLv + 1] = {};
  long long lv_launches[FSIGPU_K_COUNT][kLv + 1] = {};
  double lv_bytes[FSIGPU_K_COUNT][kLv + 1] = {};
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[FSIGPU_K_COUNT] = {0};
  long long launches[FSIGPU_K_COUNT] = {0};
  double bytes[FSIGPU_K_COUNT] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    FSI_CUDA(cudaEventCreate(&e));
    return e;
  }
  int begin(int cls, double by, cudaStream_t s) {
    if (!on) return -1;
    Rec r{cls, by, get(), get(), level};
    FSI_CUDA(cudaEventRecord(r.a, s));
    recs.push_back(r);
    return (int)recs.size() - 1;
  }
  void end(int id, cudaStream_t s) {
    if (id < 0) return;
    FSI_CUDA(cudaEventRecord(recs[id].b, s));
  }
  void flush() {
    for (auto& r : recs) {
      FSI_CUDA(cudaEventSynchronize(r.b));
      float t = 0;
      FSI_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.cls] += t;
      launches[r.cls] += 1;
      bytes[r.cls] += r.bytes;
      const int li = (r.lvl >= 0 && r.lvl < kLv) ? r.lvl + 1 : 0;
      lv_ms[r.cls][li] += t;
      lv_launches[r.cls][li] += 1;
      lv_bytes[r.cls][li] += r.bytes;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    recs.clear();
  }
};
static Profiler g_prof;
static std::mutex g_prof_mu;

// Device-clock launch stamps (common.cuh stamp_*): kernel durations INSIDE
// the captured restart-cycle graph, where CUDA events cannot bracket a
// launch. One slot of four u64 per (kernel class, GMG level, kernel of the
// class); the pointers are baked into the graph at capture, so switching the
// stamps bumps g_stamp_epoch and every solver re-captures.
constexpr int kStampSubs = 4;
static unsigned long long* g_stamp_buf = nullptr;
static bool g_stamp_on = false;
static std::atomic<int> g_stamp_epoch{0};
static thread_local int g_cur_cls = -1;
static inline size_t stamp_slots() { return (size_t)FSIGPU_K_COUNT * (Profiler::kLv + 1) * kStampSubs; }
// slot of the kernel being launched under the current ProfScope
static inline unsigned long long* cur_stamp(int sub = 0) {
  if (!g_stamp_on || g_cur_cls < 0) return nullptr;
  const int li = (g_prof.level >= 0 && g_prof.level < Profiler::kLv) ? g_prof.level + 1 : 0;
  return g_stamp_buf + 4 * (((size_t)g_cur_cls * (Profiler::kLv + 1) + li) * kStampSubs + sub);
}

struct ProfScope {
  int id;
  cudaStream_t s;
  int prev_cls;
  ProfScope(int cls, double bytes, cudaStream_t st) : s(st), prev_cls(g_cur_cls) {
    g_cur_cls = cls;
    id = g_prof.begin(cls, bytes, st);
  }
  ~ProfScope() {
    g_cur_cls = prev_cls;
    try {
      g_prof.end(id, s);
    } catch (...) {
    }
  }
};

// Host-side count of our kernel launches (graph replays are added from the
// per-graph counts taken at capture time).
static std::atomic<long long> g_launches{0};
static inline void counted(int k = 1) { g_launches += k; }

// ------------------------------------------------------------ CSR
// Lanes per row: the power of two nearest to avg_nnz / target. The entries
// per lane that hide latency best grow with the level size: ~2 on tiny
// levels (< 16k rows), 8 from 16k to 64k rows, 16 on HBM-bound levels, where
// fewer lanes per row keep more rows -- hence more independent loads -- in
// flight per warp. Batch depth: tiny levels take the smallest batch that
// holds a lane's whole share (4 or 8), 16k..64k rows 8, larger levels 4.
// Levels below 64k rows are tuned on the kernels' IN-GRAPH durations
// (device-clock stamps inside a config-0 solve, tools/tune_ingraph.py,
// profiles/r02_tune_ingraph_cfg0.txt: fine FS 7.8 -> 6.6 us, fine A 4.05 ->
// 3.55, L1 A 2.9 -> 1.5); the isolated cold/warm sweeps of round 1
// (profiles/r01_tune_spmv_*.txt) had picked 4 entries per lane there. The
// HBM-bound levels keep the cold-sweep rule.
static int choose_lpr(long long rows, long long nnz) {
  if (rows <= 0) return 2;
  const double target = rows < 16384 ? 2.0 : rows < 65536 ? 8.0 : 16.0;
  const double want = (double)nnz / rows / target;
  int l = 2;
  while (l < 32 && want > l * 1.41421356) l *= 2;
  return l;
}
static int choose_unroll(long long rows, long long nnz, int lpr) {
  if (rows >= 65536) return 4;
  if (rows >= 16384) return 8;
  return rows > 0 && (double)nnz / rows / lpr <= 4.0 ? 4 : 8;
}

struct Csr {
  int rows = 0, cols = 0;
  long long nnz = 0;
  int lpr = 8;
  DevBuf<int> ptr, idx;
  DevBuf<double> val;
  std::vector<int> h_ptr, h_idx;  // host copies (setup-side index work)
  std::vector<double> h_val;

  void create(int r, int c, const int* p, const int* ix, const double* v, cudaStream_t s,
              bool keep_host = false) {
    require(r >= 0 && c >= 0, "csr: negative dimension");
    require(p != nullptr || r == 0, "csr: null row offsets");
    rows = r;
    cols = c;
    nnz = r ? p[r] : 0;
    require(nnz >= 0 && (r == 0 || p[0] == 0), "csr: bad row offsets");
    ptr.upload(p, (size_t)r + 1, s);
    // padded by 4 entries (the paired-load kernels read 16-byte pairs)
    idx.alloc((size_t)nnz + 4);
    val.alloc((size_t)nnz + 4);
    if (nnz) {
      FSI_CUDA(cudaMemcpyAsync(idx.p, ix, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
      FSI_CUDA(cudaMemcpyAsync(val.p, v, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    lpr = choose_lpr(r, nnz);
    unroll = choose_unroll(r, nnz, lpr);
    h_ptr.assign(p, p + r + 1);
    if (keep_host) {
      h_idx.assign(ix, ix + nnz);
      h_val.assign(v, v + nnz);
    }
    // offsets and column ranges checked on the device (host loops over
    // ~1e8 entries took seconds at config 2)
    int bad = 0;
    if (r) {
      DevBuf<int> flag(1);
      flag.zero(s);
      csr_check_kernel<<<ceil_div(r, 256), 256, 0, s>>>(r, c, nnz, ptr.p, idx.p, flag.p);
      FSI_CHECK_LAUNCH();
      FSI_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    FSI_CUDA(cudaStreamSynchronize(s));
    require(!(bad & 1), "csr: offsets not nondecreasing");
    require(!(bad & 2), "csr: column range");
  }
  // take ownership of device CSR arrays built on the GPU
  void adopt(int r, int c, DevBuf<int>&& p, DevBuf<int>&& ix, DevBuf<double>&& v) {
    rows = r;
    cols = c;
    ptr = std::move(p);
    nnz = (long long)ix.n;
    idx.alloc((size_t)nnz + 4);
    val.alloc((size_t)nnz + 4);
    if (nnz) {
      FSI_CUDA(cudaMemcpy(idx.p, ix.p, sizeof(int) * nnz, cudaMemcpyDeviceToDevice));
      FSI_CUDA(cudaMemcpy(val.p, v.p, sizeof(double) * nnz, cudaMemcpyDeviceToDevice));
    }
    ix.release();
    v.release();
    lpr = choose_lpr(r, nnz);
    unroll = choose_unroll(r, nnz, lpr);
    h_ptr = ptr.download();
  }
  // column-pair format (sparse.cuh csr2_kernel): built for the FS operator
  // and the level operator when the column count is even
  DevBuf<int> ptr2, idx2;
  DevBuf<double2> val2;
  long long n2 = 0;  // elements (pairs)
  bool pairs = false;
  void build_pairs(cudaStream_t s, bool any_size = false) {
    pairs = false;
    // HBM-bound levels only: on L2-resident levels the bytes saved do not
    // matter and the wider loads cost occupancy (config 0 in-graph: fine FS
    // 6.5 -> 6.9 us, fine residual 3.5 -> 4.5 us with pairs; config 2: 1.25M rows
    // FS 692 -> 669 us, residual 220 -> 195 us, 20k rows FS 13.9 -> 14.9 us)
    const char* fb = std::getenv("FSIGPU_FORCE_BIG");  // the parity tests take the large-level formats on small fixtures
    if (fb && fb[0] == '1') any_size = true;
    if ((rows < 65536 && !any_size) || !rows || (cols & 1) || pairs_disabled()) return;
    ptr2.alloc((size_t)rows + 1);
    ptr2.zero(s);
    csr2_build_kernel<<<ceil_div(rows, 128), 128, 0, s>>>(rows, ptr.p, idx.p, val.p, ptr2.p, nullptr, nullptr, 0);
    FSI_CHECK_LAUNCH();
    thrust::device_ptr<int> pp(ptr2.p);
    thrust::inclusive_scan(thrust::cuda::par.on(s), pp, pp + rows + 1, pp);
    int total = 0;
    FSI_CUDA(cudaMemcpyAsync(&total, ptr2.p + rows, sizeof(int), cudaMemcpyDeviceToHost, s));
    FSI_CUDA(cudaStreamSynchronize(s));
    n2 = total;
    // worth it only when most entries pair up (20 B per element against 12 B per entry)
    if (20.0 * n2 > 0.95 * 12.0 * nnz) return;
    idx2.alloc((size_t)n2 + 4);
    val2.alloc((size_t)n2 + 4);
    csr2_build_kernel<<<ceil_div(rows, 128), 128, 0, s>>>(rows, ptr.p, idx.p, val.p, ptr2.p, idx2.p, val2.p, 1);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(s));
    pairs = true;
    // launch shape of csr2_kernel from the in-graph sweep on config 2
    // (profiles/r02_tune_pairs_cfg2.txt): ~16 elements per lane (8 on levels
    // below 128k rows with short rows), batches of 2 elements
    const double per_row = (double)n2 / rows;
    const double want = per_row / ((rows >= 131072 || per_row > 64.0) ? 16.0 : 8.0);
    int l = 2;
    while (l < 32 && want > l * 1.41421356) l *= 2;
    lpr = l;
    unroll = 4;
  }
  // 2 x 2 blocks on top of the column pairs (sparse.cuh bsr22_kernel): the FS
  // operator of the large levels, where the two component rows of a node
  // share their pattern
  DevBuf<int> ptrb, idxb;
  DevBuf<double2> valb;
  long long nb22 = 0;
  bool blocks22 = false;
  void build_blocks22(cudaStream_t s) {
    blocks22 = false;
    const char* e = std::getenv("FSIGPU_BLOCKS22");
    if (!pairs || (rows & 1) || (e && e[0] == '0')) return;
    const int rp = rows / 2;
    ptrb.alloc((size_t)rp + 1);
    ptrb.zero(s);
    bsr22_build_kernel<<<ceil_div(rp, 128), 128, 0, s>>>(rp, ptr2.p, idx2.p, val2.p, ptrb.p, nullptr, nullptr, 0);
    FSI_CHECK_LAUNCH();
    thrust::device_ptr<int> pp(ptrb.p);
    thrust::inclusive_scan(thrust::cuda::par.on(s), pp, pp + rp + 1, pp);
    int total = 0;
    FSI_CUDA(cudaMemcpyAsync(&total, ptrb.p + rp, sizeof(int), cudaMemcpyDeviceToHost, s));
    FSI_CUDA(cudaStreamSynchronize(s));
    nb22 = total;
    if (36.0 * nb22 > 0.98 * 20.0 * n2) return;  // the row patterns differ too often
    idxb.alloc((size_t)nb22 + 4);
    valb.alloc(2 * (size_t)nb22 + 8);
    bsr22_build_kernel<<<ceil_div(rp, 128), 128, 0, s>>>(rp, ptr2.p, idx2.p, val2.p, ptrb.p, idxb.p, valb.p, 1);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(s));
    blocks22 = true;
    // the column pairs were only the intermediate: free them (3.4 GB for the
    // fine FS operator of config 2)
    pairs = false;
    ptr2.release();
    idx2.release();
    val2.release();
    // launch shape of bsr22_kernel (in-graph sweeps): the HBM-bound levels keep
    // the pair format's lane count; L2-resident levels take ~3 blocks per lane
    // (config 0 fine FS: 32 lanes 5.4 us, 8 lanes 22 us)
    if (rows < 65536) {
      const double want = (double)nb22 / (rows / 2) / 3.0;
      int l = 2;
      while (l < 32 && want > l * 1.41421356) l *= 2;
      lpr = l;
      unroll = 4;
    } else if (lpr < 4) {
      lpr = 4;  // A on config 2: 1.25M rows 151 -> 145 us, 313k rows 44 -> 38 us (4 lanes per row pair)
    }
  }
  static bool pairs_disabled() {
    const char* e = std::getenv("FSIGPU_COLUMN_PAIRS");
    return e && e[0] == '0';
  }
  double bytes(bool resid) const {
    const double mat = blocks22 ? 36.0 * nb22 : pairs ? 20.0 * n2 : 12.0 * nnz;
    return mat + 4.0 * (rows + 1) + 8.0 * cols + 8.0 * rows + (resid ? 8.0 * rows : 0.0);
  }
  int unroll = 4;  // entries per lane per predicated batch (4 or 8); 22/24: paired loads, 2/4 pairs
  template <class G, class E>
  void launch(G g, E e, cudaStream_t s) const {
    if (!rows) return;
    const long long threads = (long long)rows * lpr;
    const int grid = ceil_div(threads, 256);
    // the pair / block kernels gather x as double2: a caller-supplied vector
    // that is only 8-byte aligned takes the CSR kernels
    const bool x16 = (reinterpret_cast<uintptr_t>(g.x) & 15) == 0;
    if (blocks22 && lpr >= 2 && x16) {
      const int grid2 = ceil_div((long long)(rows / 2) * lpr, 256);
#define FSI_BSR(LP, UU) launch_k(bsr22_kernel<LP, G, E, UU>, dim3(grid2), dim3(256), 0, s, rows / 2, (const int*)ptrb.p, (const int*)idxb.p, (const double2*)valb.p, g, e, cur_stamp(0))
      if (unroll == 8 || unroll == 24) {  // batches of 4 blocks per lane
        switch (lpr) {
          case 2: FSI_BSR(2, 4); break;
          case 4: FSI_BSR(4, 4); break;
          case 8: FSI_BSR(8, 4); break;
          case 16: FSI_BSR(16, 4); break;
          default: FSI_BSR(32, 4); break;
        }
      } else {
        switch (lpr) {
          case 2: FSI_BSR(2, 2); break;
          case 4: FSI_BSR(4, 2); break;
          case 8: FSI_BSR(8, 2); break;
          case 16: FSI_BSR(16, 2); break;
          default: FSI_BSR(32, 2); break;
        }
      }
#undef FSI_BSR
      FSI_CHECK_LAUNCH();
      counted();
      return;
    }
    if (pairs && lpr >= 2 && x16) {
      // column-pair format: batches of 2 (unroll 4 / 22) or 4 (unroll 8 / 24) elements per lane
#define FSI_CSR2(LP, UU) launch_k(csr2_kernel<LP, G, E, UU>, dim3(grid), dim3(256), 0, s, rows, (const int*)ptr2.p, (const int*)idx2.p, (const double2*)val2.p, g, e, cur_stamp(0))
      if (unroll == 8 || unroll == 24) {
        switch (lpr) {
          case 2: FSI_CSR2(2, 4); break;
          case 4: FSI_CSR2(4, 4); break;
          case 8: FSI_CSR2(8, 4); break;
          case 16: FSI_CSR2(16, 4); break;
          default: FSI_CSR2(32, 4); break;
        }
      } else {
        switch (lpr) {
          case 2: FSI_CSR2(2, 2); break;
          case 4: FSI_CSR2(4, 2); break;
          case 8: FSI_CSR2(8, 2); break;
          case 16: FSI_CSR2(16, 2); break;
          default: FSI_CSR2(32, 2); break;
        }
      }
#undef FSI_CSR2
      FSI_CHECK_LAUNCH();
      counted();
      return;
    }
#define FSI_CSR(LP, UU) launch_k(csr_kernel<LP, G, E, UU>, dim3(grid), dim3(256), 0, s, rows, (const int*)ptr.p, (const int*)idx.p, (const double*)val.p, g, e, cur_stamp(0))
#define FSI_CSRP(LP, UU) launch_k(csr_pair_kernel<LP, G, E, UU>, dim3(grid), dim3(256), 0, s, rows, (const int*)ptr.p, (const int*)idx.p, (const double*)val.p, g, e, cur_stamp(0))
    if (unroll == 22 || unroll == 24) {  // paired loads, 2 or 4 pairs per lane per batch
      if (unroll == 22) {
        switch (lpr) {
          case 1: FSI_CSRP(1, 2); break;
          case 2: FSI_CSRP(2, 2); break;
          case 4: FSI_CSRP(4, 2); break;
          case 8: FSI_CSRP(8, 2); break;
          case 16: FSI_CSRP(16, 2); break;
          default: FSI_CSRP(32, 2); break;
        }
      } else {
        switch (lpr) {
          case 1: FSI_CSRP(1, 4); break;
          case 2: FSI_CSRP(2, 4); break;
          case 4: FSI_CSRP(4, 4); break;
          case 8: FSI_CSRP(8, 4); break;
          case 16: FSI_CSRP(16, 4); break;
          default: FSI_CSRP(32, 4); break;
        }
      }
    } else if (unroll == 8) {
      switch (lpr) {
        case 2: FSI_CSR(2, 8); break;
        case 4: FSI_CSR(4, 8); break;
        case 8: FSI_CSR(8, 8); break;
        case 16: FSI_CSR(16, 8); break;
        default: FSI_CSR(32, 8); break;
      }
    } else {
      switch (lpr) {
        case 2: FSI_CSR(2, 4); break;
        case 4: FSI_CSR(4, 4); break;
        case 8: FSI_CSR(8, 4); break;
        case 16: FSI_CSR(16, 4); break;
        default: FSI_CSR(32, 4); break;
      }
    }
#undef FSI_CSR
#undef FSI_CSRP
    FSI_CHECK_LAUNCH();
    counted();
  }
};

// ------------------------------------------------------------ dense blocks
// Batched DenseFactorization: one LU per block, column-major.
// Block solve modes: LU forward/back substitution (tiled, tile inverses) or
// explicit block inverse (computed at setup from the bit-exact LU).
enum BlockMode { kModeLU = 0, kModeInverse = 1, kModeAssembled = 2 };
static std::atomic<int> g_default_mode{kModeAssembled};

// FSIGPU_FORCE_BIG=1: take the large-system kernel variants at any size
// (the split (A), the multi-row Arnoldi updates, paired
// loads, the column-pair / 2 x 2 block formats), so the parity tests cover
// them on the small committed fixtures.
static bool force_big() {
  const char* e = std::getenv("FSIGPU_FORCE_BIG");
  return e && e[0] == '1';
}

struct Blocks {
  int mode = kModeLU;
  long long nb = 0;
  long long total_rows = 0;
  int max_m = 0;
  bool keep_lu = false;
  std::vector<int> h_m;
  std::vector<long long> h_lu_off, h_row_off, h_sf_off;
  DevBuf<int> m;
  DevBuf<long long> lu_off, row_off, sf_off;
  DevBuf<double> lu, orig, sf;
  DevBuf<int> gsrc, piv, pos, lperm;
  DevBuf<double> inv;
  DevBuf<long long> inv_off;
  std::vector<long long> h_inv_off;
  DevBuf<SolveItem> items, inv_items;
  int n_inv_items = 0;
  int n_items = 0;
  int smem_cap = 0;        // doubles per TMA panel buffer
  int pipe_cap = 2;        // doubles of the largest block solve format (pipelined small solve)
  double solve_bytes = 0;  // algorithmic bytes of one batched solve
  double factor_flops = 0;

  void layout(const std::vector<int>& sizes, cudaStream_t s, bool keep = false) {
    nb = (long long)sizes.size();
    keep_lu = keep;
    h_m = sizes;
    h_lu_off.assign(nb + 1, 0);
    h_row_off.assign(nb + 1, 0);
    h_sf_off.assign(nb + 1, 0);
    max_m = 0;
    solve_bytes = 0;
    factor_flops = 0;
    smem_cap = 0;
    pipe_cap = 2;
    for (long long b = 0; b < nb; ++b) {
      const long long mm = sizes[b];
      require(mm >= 1 && mm <= kBigPanelMaxM, "blocks: block size must be in [1, 850]");
      h_lu_off[b + 1] = h_lu_off[b] + mm * mm;
      h_row_off[b + 1] = h_row_off[b] + mm;
      h_sf_off[b + 1] = h_sf_off[b] + even_up((int)solve_format_size((int)mm));
      pipe_cap = std::max<int>(pipe_cap, (int)(h_sf_off[b + 1] - h_sf_off[b]));
      max_m = std::max<int>(max_m, (int)mm);
      solve_bytes += 8.0 * solve_format_size((int)mm) + 4.0 * mm + 8.0 * mm + 8.0 * mm;
      factor_flops += 2.0 / 3.0 * mm * mm * mm;
      if (mm > kSmallMax && mm <= kTmaMax)
        for (int p = 0; p < (mm + 31) / 32; ++p) {
          const PanelGeom g((int)mm, p);
          smem_cap = std::max<int>(smem_cap, (int)std::max(g.fwd_size(), g.bwd_size()));
        }
    }
    smem_cap = even_up(smem_cap);
    total_rows = h_row_off[nb];
    m.upload(h_m, s);
    lu_off.upload(h_lu_off, s);
    row_off.upload(h_row_off, s);
    sf_off.upload(h_sf_off, s);
    if (keep_lu || max_m > 164) lu.alloc((size_t)h_lu_off[nb]);
    sf.alloc((size_t)std::max<long long>(h_sf_off[nb], 2));
    gsrc.alloc((size_t)total_rows);
    piv.alloc((size_t)total_rows);
    lperm.alloc((size_t)total_rows);
    // solve work items: small blocks 8 per CTA (warp each), large 1 per CTA
    std::vector<SolveItem> it;
    long long b = 0;
    while (b < nb) {
      if (h_m[b] <= kSmallMax) {
        SolveItem x{0, (int)b, 0, 0};
        while (b < nb && h_m[b] <= kSmallMax && x.count < 8) {
          ++x.count;
          ++b;
        }
        it.push_back(x);
      } else {
        it.push_back(SolveItem{1, (int)b, 1, 0});
        ++b;
      }
    }
    require(nb < INT_MAX && total_rows < INT_MAX, "blocks: too many blocks/rows for int32 maps");
    n_items = (int)it.size();
    items.upload(it, s);
    if (smem_cap > 0) {
      const int bytes = 2 * smem_cap * 8;
      FSI_CUDA(cudaFuncSetAttribute(block_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    }
  }

  // LU of every block from src (column-major, lu_off offsets). The three
  // size classes (register/smem small, smem large, global) and their block
  // lists are fixed at layout time, so a refactor only launches kernels.
  // classes 0..4: register LU, rows of MM = 16/32/48/56/64 (one thread per
  // row); 5: shared-memory staged (m <= 164); 6: in place in global memory.
  static constexpr int kNumCls = 7;
  static constexpr int kRegMM[5] = {16, 32, 48, 56, 64};
  std::vector<int> h_cls[kNumCls];
  DevBuf<int> d_cls_all;  // the class lists back to back (one allocation)
  const int* d_cls[kNumCls] = {};
  int cls_max[kNumCls] = {};
  DevBuf<int> fail;
  DevBuf<double> big_rowmax;  // blocked LU: original row maxima, swapped with their rows
  DevBuf<int> big_bad;        // blocked LU: per-block singular flag
  void build_classes(cudaStream_t s) {
    for (int c = 0; c < kNumCls; ++c) {
      h_cls[c].clear();
      cls_max[c] = 0;
    }
    for (long long b = 0; b < nb; ++b) {
      const int mm = h_m[b];
      int c = mm <= 164 ? 5 : 6;
      if (mm <= 64) {
        c = 0;
        while (mm > kRegMM[c]) ++c;
      }
      h_cls[c].push_back((int)b);
      cls_max[c] = std::max(cls_max[c], mm);
    }
    std::vector<int> all;
    std::vector<size_t> off(kNumCls, 0);
    for (int c = 0; c < kNumCls; ++c) {
      off[c] = all.size();
      all.insert(all.end(), h_cls[c].begin(), h_cls[c].end());
    }
    if (!all.empty()) d_cls_all.upload(all, s);
    for (int c = 0; c < kNumCls; ++c) d_cls[c] = h_cls[c].empty() ? nullptr : d_cls_all.p + off[c];
    fail.alloc(1);
  }
  template <int MM>
  void launch_reg(int which, const double* src, double* luo, const int* src_pos, int pos_base, cudaStream_t s) {
    const int mx = cls_max[which];
    const size_t sm = (size_t)((size_t)mx * mx + mx + (mx + 1) / 2 + 32 * kTileLd + 8) * 8;
    auto k = lu_reg_kernel<MM>;
    FSI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k<<<(int)h_cls[which].size(), MM <= 32 ? 32 : 64, sm, s>>>(d_cls[which], m.p, lu_off.p, row_off.p,
                                                             sf_off.p, src, luo, sf.p, piv.p, gsrc.p, lperm.p,
                                                             src_pos, pos_base, fail.p);
  }
  void factor(const double* src, const int* src_pos, int pos_base, cudaStream_t s) {
    if (!fail.n) build_classes(s);
    const int big = INT_MAX;
    FSI_CUDA(cudaMemcpyAsync(fail.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    double* luo = keep_lu ? lu.p : nullptr;
    auto smem_bytes = [](int mx) { return (size_t)((size_t)mx * mx + mx + (mx + 1) / 2 + 32 * 33 + 8) * 8; };
    auto run = [&](int which) {
      if (h_cls[which].empty()) return;
      const int grid = (int)h_cls[which].size();
      const int mx = cls_max[which];
      const int* bl = d_cls[which];
      switch (which) {
        case 0: launch_reg<16>(which, src, luo, src_pos, pos_base, s); break;
        case 1: launch_reg<32>(which, src, luo, src_pos, pos_base, s); break;
        case 2: launch_reg<48>(which, src, luo, src_pos, pos_base, s); break;
        case 3: launch_reg<56>(which, src, luo, src_pos, pos_base, s); break;
        case 4: launch_reg<64>(which, src, luo, src_pos, pos_base, s); break;
        case 5: {
          const size_t sm = smem_bytes(mx);
          auto k = lu_factor_kernel<256>;
          FSI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          k<<<grid, 256, sm, s>>>(bl, m.p, lu_off.p, row_off.p, sf_off.p, src, luo, sf.p, piv.p, gsrc.p, lperm.p,
                                  src_pos, pos_base, fail.p);
          break;
        }
        default: {
          // blocked LU in global memory: init, (panel, trailing update) per
          // 32-column panel for the whole class, then the outputs
          if (big_rowmax.n < (size_t)total_rows) big_rowmax.alloc((size_t)total_rows);
          if (big_bad.n < (size_t)grid) big_bad.alloc((size_t)grid);
          lu_big_init_kernel<<<grid, 256, 0, s>>>(bl, m.p, lu_off.p, row_off.p, src, lu.p, big_rowmax.p, big_bad.p);
          require(mx <= kBigPanelMaxM, "blocks: block size above the blocked-LU panel limit");
          FSI_CUDA(cudaFuncSetAttribute(lu_big_panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)((size_t)mx * (kBigNB + 1) * 8)));
          for (int k0 = 0; k0 < mx; k0 += kBigNB) {
            lu_big_panel_smem_kernel<<<grid, kPanelThreads, (size_t)(mx - k0) * (kBigNB + 1) * 8, s>>>(
                bl, m.p, lu_off.p, row_off.p, lu.p, big_rowmax.p, piv.p, big_bad.p, fail.p, k0);
            if (k0 + kBigNB < mx) {
              // 2-row x 8-column register tiles, 256 threads
              const int tiles = ceil_div(mx - k0 - kBigNB, kBigTile);
              lu_big_update_r4_kernel<<<dim3(tiles, grid), 256, 0, s>>>(bl, m.p, lu_off.p, lu.p, big_bad.p, k0);
            }
          }
          const size_t smf = (size_t)(mx + (mx + 1) / 2 + 32 * kTileLd + 8) * 8;
          FSI_CUDA(cudaFuncSetAttribute(lu_big_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smf));
          lu_big_finish_kernel<<<grid, 256, smf, s>>>(bl, m.p, lu_off.p, row_off.p, sf_off.p, lu.p, sf.p, piv.p,
                                                      gsrc.p, lperm.p, src_pos, pos_base, big_bad.p);
        }
      }
      FSI_CHECK_LAUNCH();
    };
    for (int c = 0; c < kNumCls; ++c) run(c);
    int bad = 0;
    FSI_CUDA(cudaMemcpyAsync(&bad, fail.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FSI_CUDA(cudaStreamSynchronize(s));
    if (bad != INT_MAX) {
      g_bad_block = bad;
      throw Error(FSIGPU_ERR_SINGULAR, "singular block: " + std::to_string(bad));
    }
    if (mode == kModeInverse) build_inverse(s);
  }

  // Explicit inverses: column c of inv(A_b) = LU solve with e_c, batched
  // over all (block, column) pairs with the same solve kernel.
  void build_inverse(cudaStream_t s) {
    h_inv_off.assign(nb + 1, 0);
    solve_bytes = 0;
    std::vector<SolveItem> it;
    for (long long b = 0; b < nb; ++b) {
      const int mm = h_m[b];
      h_inv_off[b + 1] = h_inv_off[b] + (long long)even_up(mm) * mm;
      solve_bytes += 8.0 * even_up(mm) * mm + 4.0 * mm + 8.0 * mm + 8.0 * mm;
      if (mm <= kSmallMax) {
        for (int c = 0; c < mm; c += 8) it.push_back(SolveItem{2, (int)b, std::min(8, mm - c), c});
      } else {
        for (int c = 0; c < mm; ++c) it.push_back(SolveItem{3, (int)b, 1, c});
      }
    }
    inv.alloc((size_t)std::max<long long>(h_inv_off[nb], 2));
    inv_off.upload(h_inv_off, s);
    // GEMV work items for the solves: one CTA per 64-row tile of every
    // block (8 column groups per tile keep each thread to <= 1-3 batches)
    std::vector<SolveItem> gi;
    for (long long b = 0; b < nb; ++b)
      for (int r0 = 0; r0 < h_m[b]; r0 += kInvTileRows) gi.push_back(SolveItem{1, (int)b, 1, r0});
    inv_items.upload(gi, s);
    n_inv_items = (int)gi.size();
    DevBuf<SolveItem> citems;
    citems.upload(it, s);
    SolveArgs a{};
    a.m = m.p;
    a.sf_off = sf_off.p;
    a.row_off = row_off.p;
    a.sf = sf.p;
    a.gsrc = gsrc.p;
    a.items = citems.p;
    a.smem_cap = 0;
    a.g1 = INT_MAX;
    a.lperm = lperm.p;
    a.inv = inv.p;
    a.inv_off = inv_off.p;
    block_solve_kernel<<<(int)it.size(), kSolveThreads, 0, s>>>(a);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(s));
  }

  // Blocks all <= 64 with a plain gathered right-hand side (config 1): one
  // shared buffer per warp filled by a bulk copy, with an L2 bulk prefetch
  // of each warp's next block issued before it solves the current one, so
  // the next copy is an L2 hit (small_pipe_solve_kernel). Config-1 solve:
  // 1.54 ms = 6.64 TB/s, against 2.33 ms for block_solve_kernel and 2.36 ms
  // for two buffers per warp (only 4 warps per SM, whose dependent solve
  // phases then run at ~0.9 IPC).
  void solve_small_pipe(const SolveArgs& base, cudaStream_t s) const {
    const int cap = pipe_cap;
    const size_t per_warp = (size_t)(cap + 64) * 8;
    const int nw = (int)std::max<size_t>(1, std::min<size_t>(kPipeMaxWarps, (size_t)(200 * 1024) / per_warp));
    const size_t smem = per_warp * nw;
    FSI_CUDA(cudaFuncSetAttribute(small_pipe_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, occ = 0;
    FSI_CUDA(cudaGetDevice(&dev));
    FSI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, small_pipe_solve_kernel, nw * 32, smem));
    const int grid = (int)std::max<long long>(1, std::min<long long>((long long)sms * std::max(occ, 1),
                                                                     (nb + nw - 1) / nw));
    SmallPipeArgs a{m.p, sf_off.p, row_off.p, sf.p, gsrc.p, base.r, base.out, nb, cap, 1};
    ProfScope ps(FSIGPU_K_BLOCK_SOLVE, solve_bytes, s);
    launch_k(small_pipe_solve_kernel, dim3(grid), dim3(nw * 32), smem, s, a);
    FSI_CHECK_LAUNCH();
    counted();
  }
  void solve(const SolveArgs& base, cudaStream_t s) const {
    if (!n_items) return;
    if (mode == kModeInverse) {
      SolveArgs a = base;
      a.m = m.p;
      a.row_off = row_off.p;
      a.items = inv_items.p;
      a.inv = const_cast<double*>(inv.p);
      a.inv_off = inv_off.p;
      a.pos = pos.n ? pos.p : nullptr;
      ProfScope ps(FSIGPU_K_BLOCK_SOLVE, solve_bytes, s);
      launch_k(inv_gemv_kernel, dim3(n_inv_items), dim3(kSolveThreads), 0, s, a);
      FSI_CHECK_LAUNCH();
      counted();
      return;
    }
    if (max_m <= kSmallMax && base.g1 == INT_MAX) {
      solve_small_pipe(base, s);
      return;
    }
    SolveArgs a = base;
    a.m = m.p;
    a.sf_off = sf_off.p;
    a.row_off = row_off.p;
    a.sf = sf.p;
    a.gsrc = gsrc.p;
    a.items = items.p;
    a.smem_cap = smem_cap;
    ProfScope ps(FSIGPU_K_BLOCK_SOLVE, solve_bytes, s);
    launch_k(block_solve_kernel, dim3(n_items), dim3(kSolveThreads), (size_t)2 * smem_cap * 8, s, a);
    FSI_CHECK_LAUNCH();
    counted();
  }
};

}  // namespace fsigpu

// C-ABI handle types
struct fsigpu_csr_t {
  fsigpu::Csr a;
  cudaStream_t s = nullptr;
};
struct fsigpu_blocks_t {
  fsigpu::Blocks b;
  cudaStream_t s = nullptr;
  int have_orig = 0;
  int own_stream = 0;
};

namespace fsigpu {

// ------------------------------------------------------------ GMG level
struct Level {
  int n = 0, nc = 0;
  Csr A, P, R;
  DevBuf<unsigned char> rmask, cmask;
  // FS smoother (levels >= 1)
  int g1 = 0, n_us = 0;
  DevBuf<double> lumped;
  Blocks blocks;  // AS1 blocks then AS2 blocks, positions in the frame
  int n_as1 = 0;
  DevBuf<int> inv_ptr, inv_idx;
  DevBuf<int> aus_ptr, aus_col;
  DevBuf<double> aus_val;
  DevBuf<double> delta, bbuf, xbuf, rbuf;
  DevBuf<double> mr_z, mr_w;  // GMRES(1) smoother: z = FS r, w = A z
  bool assembled = false;  // FS smoother as one sparse operator (kModeAssembled)
  // multiplicative FS (mult.cuh): group-restricted matrix, blocks by colour
  bool mult = false;
  Csr AG;
  DevBuf<int> col_blocks;
  std::vector<int> h_col_off;  // colour c = col_blocks[h_col_off[c] .. h_col_off[c+1])
  DevBuf<double> mz;           // FS(r) of the sweep
  double mult_bytes = 0;
  Csr FS;
  Csr AP;  // A * diag(!col_mask) * P : fused prolongation + post-smoothing residual
  double* b = nullptr;  // level rhs (top level: external)
  double* x = nullptr;  // level iterate (top level: external)
  double combine_bytes = 0;
};

// x += P ec ; r = r_pre - AP ec on level L (ec: the next-coarser iterate;
// cmask_coarse: nullptr when ec is already masked). Lanes per row follow AP.
static void launch_prolong_resid(const Level& L, const double* ec, const unsigned char* cmask_coarse,
                                 const double* r_pre, double* r, cudaStream_t s) {
  const int grid = ceil_div((long long)L.n * L.AP.lpr, 256);
  if (L.AP.blocks22 && L.AP.lpr >= 2) {
    const int grid2 = ceil_div((long long)(L.n / 2) * L.AP.lpr, 256);
#define FSI_PR22(LP)                                                                                              \
  launch_k(prolong_resid22_kernel<LP, 2>, dim3(grid2), dim3(256), 0, s, L.n / 2, (const int*)L.P.ptr.p,          \
           (const int*)L.P.idx.p, (const double*)L.P.val.p, (const int*)L.AP.ptrb.p, (const int*)L.AP.idxb.p,     \
           (const double2*)L.AP.valb.p, ec, cmask_coarse, (const unsigned char*)L.cmask.p, L.x, r_pre, r,         \
           cur_stamp(1))
    switch (L.AP.lpr) {
      case 2: FSI_PR22(2); break;
      case 4: FSI_PR22(4); break;
      case 8: FSI_PR22(8); break;
      case 16: FSI_PR22(16); break;
      default: FSI_PR22(32); break;
    }
#undef FSI_PR22
    FSI_CHECK_LAUNCH();
    return;
  }
  if (L.AP.pairs && L.AP.lpr >= 2) {
#define FSI_PR2(LP, UA)                                                                                         \
  launch_k(prolong_resid2_kernel<LP, UA>, dim3(grid), dim3(256), 0, s, L.n, (const int*)L.P.ptr.p,             \
           (const int*)L.P.idx.p, (const double*)L.P.val.p, (const int*)L.AP.ptr2.p, (const int*)L.AP.idx2.p,  \
           (const double2*)L.AP.val2.p, ec, cmask_coarse, (const unsigned char*)L.cmask.p, L.x, r_pre, r,      \
           cur_stamp(1))
    const bool four = L.AP.unroll == 8 || L.AP.unroll == 24;
    switch (L.AP.lpr) {
      case 2: if (four) FSI_PR2(2, 4); else FSI_PR2(2, 2); break;
      case 4: if (four) FSI_PR2(4, 4); else FSI_PR2(4, 2); break;
      case 8: if (four) FSI_PR2(8, 4); else FSI_PR2(8, 2); break;
      case 16: if (four) FSI_PR2(16, 4); else FSI_PR2(16, 2); break;
      default: if (four) FSI_PR2(32, 4); else FSI_PR2(32, 2); break;
    }
#undef FSI_PR2
    FSI_CHECK_LAUNCH();
    return;
  }
#define FSI_PR(K, LP, UA)                                                                                        \
  launch_k(K<LP, UA>, dim3(grid), dim3(256), 0, s, L.n, (const int*)L.P.ptr.p, (const int*)L.P.idx.p,         \
           (const double*)L.P.val.p, (const int*)L.AP.ptr.p, (const int*)L.AP.idx.p, (const double*)L.AP.val.p, \
           ec, cmask_coarse, (const unsigned char*)L.cmask.p, L.x, r_pre, r, cur_stamp(1))
#define FSI_PR_L(K, UA)                 \
  switch (L.AP.lpr) {                   \
    case 2: FSI_PR(K, 2, UA); break;    \
    case 4: FSI_PR(K, 4, UA); break;    \
    case 8: FSI_PR(K, 8, UA); break;    \
    case 16: FSI_PR(K, 16, UA); break;  \
    default: FSI_PR(K, 32, UA); break;  \
  }
  switch (L.AP.unroll) {
    case 22: FSI_PR_L(prolong_resid_pair_kernel, 2) break;  // paired A*P loads, 2 / 4 pairs
    case 24: FSI_PR_L(prolong_resid_pair_kernel, 4) break;
    case 4: FSI_PR_L(prolong_resid_kernel, 4) break;
    default: FSI_PR_L(prolong_resid_kernel, 8) break;
  }
#undef FSI_PR_L
#undef FSI_PR
  FSI_CHECK_LAUNCH();
}

struct Gmg {
  std::vector<Level> lv;
  // read-only hot data (level matrices, transfers, block inverses, coarse
  // inverse) packed in one arena
  DevBuf<char> arena;
  double omega = 0.7;
  int pre = 1, post = 1;
  char cyc = 'v';
  // level smoother: 0 damped Richardson (precond.cpp:305-317), 1 GMRES(1)
  // minimal-residual step (mr.cuh); `version` bumps on every change so a
  // solver's captured graphs are rebuilt
  int smoother = 0;
  int version = 0;
  DevBuf<double> mr_part, mr_alpha;
  DevBuf<unsigned int> mr_ticket;
  DevBuf<double> coarse_inv;  // equilibrated explicit inverse, row-major
  cudaStream_t s = nullptr;
  DevBuf<double> tmp_in, tmp_out;
  // Every entry point that launches on this hierarchy holds the lock: the
  // V-cycle rewires the top level's b/x pointers and shares per-level
  // scratch, so concurrent callers of one handle are serialised (the
  // reference's const apply is re-entrant, precond.cpp:45,61).
  std::mutex mu;

  int size() const { return lv.back().n; }

  void smooth_solve(int l, const double* rhs) {
    Level& L = lv[l];
    SolveArgs a{};
    a.r = rhs;
    a.g1 = L.g1;
    a.lumped = L.lumped.p;
    a.aus_ptr = L.aus_ptr.p;
    a.aus_col = L.aus_col.p;
    a.aus_val = L.aus_val.p;
    a.out = L.delta.p;
    L.blocks.solve(a, s);
  }
  void combine(int l, const double* r, int x_zero) {
    Level& L = lv[l];
    ProfScope ps(FSIGPU_K_COMBINE, L.combine_bytes, s);
    launch_k(fs_combine_kernel, dim3(ceil_div(L.n, 256)), dim3(256), 0, s, L.n, L.g1, L.n_us,
             (const int*)L.inv_ptr.p, (const int*)L.inv_idx.p, (const double*)L.delta.p, r,
             (const double*)L.lumped.p, omega, L.x, x_zero);
    FSI_CHECK_LAUNCH();
    counted();
  }
  void resid(int l, double* r) {
    Level& L = lv[l];
    ProfScope ps(FSIGPU_K_SPMV, L.A.bytes(true), s);
    L.A.launch(GatherPlain{L.x}, EpiResid{L.b, r}, s);
  }
  // x (+)= omega * FS r, fused into the FS SpMV epilogue; mask_out: the
  // level's constrained columns are zeroed on the way out (last write of a
  // coarse level in a V-cycle, see cycle())
  void fs_spmv(int l, const double* r, int x_zero, bool mask_out = false) {
    Level& L = lv[l];
    ProfScope ps(FSIGPU_K_BLOCK_SOLVE, L.FS.bytes(false) + 8.0 * L.n, s);
    if (x_zero)
      L.FS.launch(GatherPlain{r}, EpiSetScaled{omega, L.x}, s);
    else if (mask_out)
      L.FS.launch(GatherPlain{r}, EpiAxpyMasked{omega, L.x, L.cmask.p}, s);
    else
      L.FS.launch(GatherPlain{r}, EpiAxpy{omega, L.x}, s);
  }
  void set_smoother(int kind) {
    if (kind == 1 && !mr_part.p) {
      mr_part.alloc(2 * kMrCtas);
      mr_alpha.alloc(1);
      mr_ticket.alloc(1);
      FSI_CUDA(cudaMemsetAsync(mr_ticket.p, 0, sizeof(unsigned int), s));
      for (size_t l = 1; l < lv.size(); ++l) {
        lv[l].mr_z.alloc(lv[l].n);
        lv[l].mr_w.alloc(lv[l].n);
      }
      FSI_CUDA(cudaStreamSynchronize(s));
    }
    smoother = kind;
    ++version;
  }
  // multiplicative FS (mult.cuh): z = FS_mult r; x (optional) += omega z
  void mult_apply(int l, const double* r, double* z, double* x, int x_zero) {
    Level& L = lv[l];
    ProfScope ps(FSIGPU_K_BLOCK_SOLVE, L.mult_bytes, s);
    launch_k(mult_init_kernel, dim3(std::max(1, std::min(ceil_div(L.n, 256), 4 * 148))), dim3(256), 0, s, L.n, L.g1,
             L.n_us, r, (const double*)L.lumped.p, z, x, omega, x_zero);
    MultArgs a{L.col_blocks.p, L.blocks.m.p, L.blocks.row_off.p, L.blocks.pos.p, L.blocks.inv.p,
               L.blocks.inv_off.p, L.AG.ptr.p, L.AG.idx.p, L.AG.val.p, r, z, x, omega};
    const int nc = (int)L.h_col_off.size() - 1;
    for (int c = 0; c < nc; ++c) {
      const int cnt = L.h_col_off[c + 1] - L.h_col_off[c];
      if (cnt) launch_k(mult_colour_kernel, dim3(cnt), dim3(kMultThreads), 0, s, a, L.h_col_off[c]);
    }
    FSI_CHECK_LAUNCH();
    counted(1 + nc);
  }
  // z = FS r (the FS smoother applied once, no damping)
  void fs_into(int l, const double* r, double* z) {
    Level& L = lv[l];
    if (L.mult) {
      mult_apply(l, r, z, nullptr, 1);
      return;
    }
    if (L.assembled) {
      ProfScope ps(FSIGPU_K_BLOCK_SOLVE, L.FS.bytes(false), s);
      L.FS.launch(GatherPlain{r}, EpiSetScaled{1.0, z}, s);
      return;
    }
    smooth_solve(l, r);
    ProfScope ps(FSIGPU_K_COMBINE, L.combine_bytes, s);
    launch_k(fs_combine_kernel, dim3(ceil_div(L.n, 256)), dim3(256), 0, s, L.n, L.g1, L.n_us,
             (const int*)L.inv_ptr.p, (const int*)L.inv_idx.p, (const double*)L.delta.p, r,
             (const double*)L.lumped.p, 1.0, z, 1);
    FSI_CHECK_LAUNCH();
    counted();
  }
  // one GMRES(1) sweep (mr.cuh): r = b - A x, z = FS r, w = A z,
  // alpha = (w.r)/(w.w), x += alpha z
  void mr_sweep(int l, int x_zero, bool r_ready, bool mask_out) {
    Level& L = lv[l];
    const double* r = L.b;  // x == 0: r = b exactly (precond.cpp:312-313)
    if (!x_zero) {
      if (!r_ready) resid(l, L.rbuf.p);
      r = L.rbuf.p;
    }
    fs_into(l, r, L.mr_z.p);
    {
      ProfScope ps(FSIGPU_K_SPMV, L.A.bytes(false), s);
      L.A.launch(GatherPlain{L.mr_z.p}, EpiPlain{L.mr_w.p}, s);
    }
    ProfScope ps(FSIGPU_K_COMBINE, 32.0 * L.n, s);
    launch_k(k_mr_alpha, dim3(kMrCtas), dim3(kMrThreads), 0, s, L.n, (const double*)L.mr_w.p, r, mr_part.p,
             mr_ticket.p, mr_alpha.p);
    FSI_CHECK_LAUNCH();
    launch_k(k_mr_update, dim3(ceil_div(L.n, 256)), dim3(256), 0, s, L.n, (const double*)mr_alpha.p,
             (const double*)L.mr_z.p, L.x, x_zero, (const unsigned char*)(mask_out ? L.cmask.p : nullptr));
    FSI_CHECK_LAUNCH();
    counted(2);
  }
  // one FS-preconditioned Richardson sweep; x_zero: x == 0 on entry;
  // r_ready: rbuf already holds b - A x (fused prolongation kernel)
  void sweep(int l, int x_zero, bool r_ready = false, bool mask_out = false) {
    Level& L = lv[l];
    if (smoother == 1) {
      mr_sweep(l, x_zero, r_ready, mask_out);
      return;
    }
    if (L.mult) {
      const double* r = L.b;  // x == 0: res = b exactly (precond.cpp:312-313)
      if (!x_zero) {
        if (!r_ready) resid(l, L.rbuf.p);
        r = L.rbuf.p;
      }
      mult_apply(l, r, L.mz.p, L.x, x_zero);
      return;
    }
    if (L.assembled) {
      if (x_zero) {
        fs_spmv(l, L.b, 1);  // res = b - A*0 = b (precond.cpp:312-313)
      } else {
        if (!r_ready) resid(l, L.rbuf.p);
        fs_spmv(l, L.rbuf.p, 0, mask_out);
      }
      return;
    }
    if (r_ready && !x_zero) {
      smooth_solve(l, L.rbuf.p);
      combine(l, L.rbuf.p, 0);
      return;
    }
    if (x_zero) {
      // res = b - A*0 = b exactly (precond.cpp:312-313)
      smooth_solve(l, L.b);
      combine(l, L.b, 1);
    } else {
      resid(l, L.rbuf.p);
      smooth_solve(l, L.rbuf.p);
      combine(l, L.rbuf.p, 0);
    }
  }
  // x (+)= A0^-1 rhs through the equilibrated explicit inverse
  void coarse_gemv(const double* rhs, double* x, int accumulate, const unsigned char* mask_out) {
    Level& L = lv[0];
    ProfScope ps(FSIGPU_K_COARSE, 8.0 * L.n * L.n + 16.0 * L.n, s);
    // 64-thread CTAs (one batch of 22 loads per thread) when 256-thread
    // CTAs would need a second wave (5 resident per SM)
    if (L.n > 5 * 148 && L.n <= 64 * 22)
      launch_k(gemv_kernel<64, 22>, dim3(L.n), dim3(64), 0, s, L.n, (const double*)coarse_inv.p, rhs, x,
               accumulate, mask_out, cur_stamp(0));
    else
      launch_k(gemv_kernel<kGemvThreads, 8>, dim3(L.n), dim3(kGemvThreads), 0, s, L.n,
               (const double*)coarse_inv.p, rhs, x, accumulate, mask_out, cur_stamp(0));
    FSI_CHECK_LAUNCH();
    counted();
  }
  void coarse(int x_zero, bool mask_out = false) {
    Level& L = lv[0];
    const double* rhs = L.b;
    if (!x_zero) {
      resid(0, L.rbuf.p);
      rhs = L.rbuf.p;
    }
    coarse_gemv(rhs, L.x, x_zero ? 0 : 1, mask_out ? L.cmask.p : nullptr);
  }
  // GmgPreconditioner::cycle (gmg.cpp:188-239). mask_out: this is the last
  // visit of a coarse level, so its final kernel may write the iterate with
  // the constrained columns already zeroed (the caller's ec mask).
  void cycle(int l, char mode, int x_zero, bool mask_out = false) {
    g_prof.level = l;
    if (l == 0) {
      coarse(x_zero, mask_out);
      return;
    }
    Level& L = lv[l];
    Level& B = lv[l - 1];
    if (pre == 0 && x_zero) FSI_CUDA(cudaMemsetAsync(L.x, 0, sizeof(double) * L.n, s));
    for (int k = 0; k < pre; ++k) sweep(l, x_zero && k == 0);
    resid(l, L.rbuf.p);
    {
      ProfScope ps(FSIGPU_K_TRANSFER, L.R.bytes(false) + L.nc, s);
      L.R.launch(GatherPlain{L.rbuf.p}, EpiRestrict{B.rmask.p, B.b}, s);
    }
    // the last visit of level l-1 masks its output iff that level ends in a
    // kernel that can (a post sweep of an assembled level or of the GMRES(1)
    // smoother, or the coarse GEMV)
    const bool fused_mask = L.AP.rows && post > 0 && (l - 1 == 0 || ((B.assembled || smoother == 1) && post > 0));
    switch (mode) {
      case 'v': cycle(l - 1, 'v', 1, fused_mask); break;
      case 'w': cycle(l - 1, 'w', 1); cycle(l - 1, 'w', 0, fused_mask); break;
      case 'f': cycle(l - 1, 'f', 1); cycle(l - 1, 'v', 0, fused_mask); break;
      default: throw Error(FSIGPU_ERR_INVALID, "gmg: unknown cycle type");
    }
    g_prof.level = l;
    if (post > 0 && L.AP.rows) {
      // x += P ec ; r = r_pre - AP ec  (one kernel; rbuf holds r_pre)
      ProfScope ps(FSIGPU_K_TRANSFER, L.P.bytes(false) + L.AP.bytes(false) + 24.0 * L.n + L.n + L.nc, s);
      launch_prolong_resid(L, B.x, fused_mask ? nullptr : B.cmask.p, L.rbuf.p, L.rbuf.p, s);
      counted();
      for (int k = 0; k < post; ++k) sweep(l, 0, k == 0, mask_out && k == post - 1);
      return;
    }
    {
      ProfScope ps(FSIGPU_K_TRANSFER, L.P.bytes(false) + 8.0 * L.n + L.n + L.nc, s);
      L.P.launch(GatherMasked{B.x, B.cmask.p}, EpiProlongAdd{L.cmask.p, L.x}, s);
    }
    for (int k = 0; k < post; ++k) sweep(l, 0);
  }
  // z = M r on device pointers
  void apply(const double* r, double* z) {
    struct LevelReset {
      ~LevelReset() { g_prof.level = -1; }
    } reset_level;
    Level& T = lv.back();
    T.b = const_cast<double*>(r);
    T.x = z;
    if (lv.size() == 1) {
      coarse(1);
    } else {
      cycle((int)lv.size() - 1, cyc, 1);
    }
  }
};

// Assemble the additive FS smoother of one level as a single sparse
// operator (linear in r, so exactly the same map as the block solves +
// combine of precond.cpp:271-303 / SURVEY §8c, up to summation order):
//   AS1 and AS2 blocks:  sum_b R_b^T inv(A_b) R_b / cover
//   u^s rows:            1 / lumped                    (precond.cpp:281-283)
//   AS2 <- u^s coupling: -inv(A_b) A_g2[:, u^s] / lumped (Jacobi update, :284-287)
// COO keys sorted stably and duplicates summed on the device (deterministic).
static void assemble_fs(Level& L, const fsigpu_level_desc& d, const std::vector<int>& pos,
                        const std::vector<int>& cover_ptr, const std::vector<int>& ap, const std::vector<int>& ac,
                        const std::vector<double>& av, cudaStream_t s) {
  Blocks& B = L.blocks;
  const int g1 = d.g1;
  std::vector<long long> coo_off(B.nb + 1, 0);
  for (long long b = 0; b < B.nb; ++b) coo_off[b + 1] = coo_off[b] + (long long)B.h_m[b] * B.h_m[b];
  const long long nblk = coo_off[B.nb];
  std::vector<unsigned long long> hk;
  std::vector<double> hv;
  for (int k = 0; k < d.n_us; ++k) {
    const unsigned long long p = (unsigned long long)(g1 + k);
    hk.push_back((p << 32) | p);
    hv.push_back(1.0 / d.lumped[k]);
  }
  // the coupling entries of the AS2 blocks touching u^s columns, built on
  // the device (fs_coo_coupling_kernel) in the order the host loop emitted
  // them: per block its (j, k) couplings, j-major
  std::vector<int> cblk, clj, clk;
  std::vector<long long> cloff{0}, coff{0};
  for (long long b = L.n_as1; b < B.nb; ++b) {
    const int m = B.h_m[b];
    const long long ro = B.h_row_off[b];
    const size_t before = clj.size();
    for (int j = 0; j < m; ++j) {
      const int q = pos[ro + j] - g1;
      for (int k = ap[q]; k < ap[q + 1]; ++k) {
        clj.push_back(j);
        clk.push_back(k);
      }
    }
    if (clj.size() == before) continue;
    cblk.push_back((int)b);
    cloff.push_back((long long)clj.size());
    coff.push_back(coff.back() + (long long)m * (long long)(clj.size() - before));
  }
  const long long ncoup = coff.back();
  const long long N = nblk + (long long)hk.size() + ncoup;
  DevBuf<unsigned long long> keys(N), ukeys(N);
  DevBuf<double> vals(N), uvals(N);
  DevBuf<long long> dco;
  dco.upload(coo_off, s);
  if (B.nb) {
    DevBuf<int> inv_ptr_d;
    inv_ptr_d.upload(cover_ptr, s);
    fs_coo_blocks_kernel<<<(int)B.nb, 256, 0, s>>>((int)B.nb, B.m.p, B.row_off.p, B.inv.p, B.inv_off.p, B.pos.p,
                                                   inv_ptr_d.p, dco.p, keys.p, vals.p);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(s));
  }
  if (!hk.empty()) {
    FSI_CUDA(cudaMemcpyAsync(keys.p + nblk, hk.data(), sizeof(unsigned long long) * hk.size(), cudaMemcpyHostToDevice, s));
    FSI_CUDA(cudaMemcpyAsync(vals.p + nblk, hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, s));
  }
  if (ncoup) {
    for (auto& o : coff) o += nblk + (long long)hk.size();
    DevBuf<int> dblk, dj, dk, dac;
    DevBuf<long long> dcl, dco;
    DevBuf<double> dav, dlm;
    dblk.upload(cblk, s);
    dj.upload(clj, s);
    dk.upload(clk, s);
    dcl.upload(cloff, s);
    dco.upload(coff, s);
    dac.upload(ac.empty() ? std::vector<int>{0} : ac, s);
    dav.upload(av.empty() ? std::vector<double>{0.0} : av, s);
    dlm.upload(d.lumped, (size_t)std::max(d.n_us, 1), s);
    DevBuf<int> inv_ptr_c;
    inv_ptr_c.upload(cover_ptr, s);
    fs_coo_coupling_kernel<<<(int)cblk.size(), 256, 0, s>>>(dblk.p, B.m.p, B.row_off.p, B.inv.p, B.inv_off.p,
                                                            B.pos.p, inv_ptr_c.p, dcl.p, dj.p, dk.p, dac.p, dav.p,
                                                            dlm.p, g1, dco.p, keys.p, vals.p);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(s));
  }
  auto pol = thrust::cuda::par.on(s);
  thrust::device_ptr<unsigned long long> kp(keys.p), ukp(ukeys.p);
  thrust::device_ptr<double> vp(vals.p), uvp(uvals.p);
  thrust::stable_sort_by_key(pol, kp, kp + N, vp);
  auto ends = thrust::reduce_by_key(pol, kp, kp + N, vp, ukp, uvp);
  const long long nnz = ends.first - ukp;
  DevBuf<int> ptr(L.n + 1), cols(nnz);
  DevBuf<double> fv(nnz);
  ptr.zero(s);
  coo_row_count_kernel<<<ceil_div(nnz, 256), 256, 0, s>>>(nnz, ukeys.p, ptr.p);
  coo_cols_kernel<<<ceil_div(nnz, 256), 256, 0, s>>>(nnz, ukeys.p, cols.p);
  FSI_CHECK_LAUNCH();
  thrust::device_ptr<int> pp(ptr.p);
  thrust::inclusive_scan(pol, pp, pp + L.n + 1, pp);
  FSI_CUDA(cudaMemcpyAsync(fv.p, uvals.p, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
  FSI_CUDA(cudaStreamSynchronize(s));
  L.FS.adopt(L.n, L.n, std::move(ptr), std::move(cols), std::move(fv));
  // the 3D FS operator's rows are several hundred entries long: 16 lanes with
  // batches of 8 on large levels (232k rows: 220 -> 211 us in-graph)
  if (L.n >= 65536 && (double)L.FS.nnz / L.n > 400.0) {
    L.FS.lpr = 16;
    L.FS.unroll = 8;
  }
  // 2 x 2 blocks from 16k rows up (in-graph: they also pay on the L2-resident
  // fine level of config 0); the column pairs alone only on HBM-bound levels
  {
    const int keep_lpr = L.FS.lpr, keep_unroll = L.FS.unroll;
    L.FS.build_pairs(s, L.n >= 16384);
    L.FS.build_blocks22(s);
    if (!L.FS.blocks22 && L.n < 65536 && !force_big()) {  // plain CSR with its own launch shape
      L.FS.pairs = false;
      L.FS.lpr = keep_lpr;
      L.FS.unroll = keep_unroll;
    }
  }
  L.assembled = true;
}

// Multicolour order of the blocks of one group of the multiplicative FS
// smoother (mult.cuh). Blocks b, b' conflict when they share a dof or the
// group matrix A[base:base+dim, base:base+dim] stores an entry coupling them
// in either direction; greedy in block order, colour(b) = the smallest colour
// no conflicting earlier block has. Same rule as the oracle's colour_blocks
// (oracle/fsi_oracle.c). bidx: group-local positions. Returns the count.
static int colour_group(int nb, const int* bptr, const int* bidx, int base, int dim, const fsigpu_level_desc& d,
                        std::vector<int>& colour) {
  colour.assign(nb, 0);
  if (nb == 0) return 0;
  std::vector<int> rp(dim + 1, 0), rc;
  for (int i = 0; i < dim; ++i) {
    for (int k = d.a_ptr[base + i]; k < d.a_ptr[base + i + 1]; ++k) {
      const int j = d.a_idx[k] - base;
      if (j >= 0 && j < dim) rc.push_back(j);
    }
    rp[i + 1] = (int)rc.size();
  }
  std::vector<int> cp(dim + 1, 0), cr(rc.size());
  for (int j : rc) cp[j + 1]++;
  for (int j = 0; j < dim; ++j) cp[j + 1] += cp[j];
  {
    std::vector<int> nx(cp.begin(), cp.end() - 1);
    for (int i = 0; i < dim; ++i)
      for (int k = rp[i]; k < rp[i + 1]; ++k) cr[nx[rc[k]]++] = i;
  }
  std::vector<int> dptr(dim + 1, 0), dblk(bptr[nb]);
  for (int k = 0; k < bptr[nb]; ++k) dptr[bidx[k] + 1]++;
  for (int i = 0; i < dim; ++i) dptr[i + 1] += dptr[i];
  {
    std::vector<int> nx(dptr.begin(), dptr.end() - 1);
    for (int b = 0; b < nb; ++b)
      for (int k = bptr[b]; k < bptr[b + 1]; ++k) dblk[nx[bidx[k]]++] = b;
  }
  std::vector<int> seen(nb + 1, -1);
  int ncol = 0;
  for (int b = 0; b < nb; ++b) {
    auto mark = [&](int j) {
      for (int q = dptr[j]; q < dptr[j + 1]; ++q)
        if (dblk[q] < b) seen[colour[dblk[q]]] = b;
    };
    for (int k = bptr[b]; k < bptr[b + 1]; ++k) {
      const int i = bidx[k];
      mark(i);
      for (int e = rp[i]; e < rp[i + 1]; ++e) mark(rc[e]);
      for (int e = cp[i]; e < cp[i + 1]; ++e) mark(cr[e]);
    }
    int c = 0;
    while (seen[c] == b) ++c;
    colour[b] = c;
    ncol = std::max(ncol, c + 1);
  }
  return ncol;
}

// Multiplicative FS data of a level: the group-restricted matrix
// blockdiag(A_g1, A_g2) and the AS1 / AS2 blocks sorted by colour (merged:
// colour c = the AS1 blocks of colour c, then the AS2 blocks of colour c;
// the groups never couple, precond.cpp:137-139).
static void build_mult(Level& L, const fsigpu_level_desc& d, cudaStream_t s) {
  const int n = d.n, g1 = d.g1;
  std::vector<int> c1, c2;
  const int n1 = colour_group(d.as1_n, d.as1_ptr, d.as1_idx, 0, g1, d, c1);
  const int n2 = colour_group(d.as2_n, d.as2_ptr, d.as2_idx, g1, n - g1, d, c2);
  const int nc = std::max(n1, n2);
  std::vector<int> order;
  L.h_col_off.assign(1, 0);
  for (int c = 0; c < nc; ++c) {
    for (int b = 0; b < d.as1_n; ++b)
      if (c1[b] == c) order.push_back(b);
    for (int b = 0; b < d.as2_n; ++b)
      if (c2[b] == c) order.push_back(d.as1_n + b);
    L.h_col_off.push_back((int)order.size());
  }
  L.col_blocks.upload(order.empty() ? std::vector<int>{0} : order, s);
  std::vector<int> ap(n + 1, 0), ai;
  std::vector<double> av;
  for (int i = 0; i < n; ++i) {
    for (int k = d.a_ptr[i]; k < d.a_ptr[i + 1]; ++k)
      if ((i < g1) == (d.a_idx[k] < g1)) {
        ai.push_back(d.a_idx[k]);
        av.push_back(d.a_val[k]);
      }
    ap[i + 1] = (int)ai.size();
  }
  if (ai.empty()) {
    ai.push_back(0);
    av.push_back(0.0);
  }
  L.AG.create(n, n, ap.data(), ai.data(), av.data(), s);
  L.mz.alloc(n);
  double by = 40.0 * n;  // init: r, lumped, z and x
  const Blocks& B = L.blocks;
  for (long long b = 0; b < B.nb; ++b) {
    const int m = B.h_m[b];
    by += 8.0 * even_up(m) * m + 36.0 * m;  // inverse, pos, r, z and x updates
  }
  for (int b = 0; b < d.as1_n; ++b)
    for (int k = d.as1_ptr[b]; k < d.as1_ptr[b + 1]; ++k) by += 20.0 * (ap[d.as1_idx[k] + 1] - ap[d.as1_idx[k]]);
  for (int b = 0; b < d.as2_n; ++b)
    for (int k = d.as2_ptr[b]; k < d.as2_ptr[b + 1]; ++k)
      by += 20.0 * (ap[g1 + d.as2_idx[k] + 1] - ap[g1 + d.as2_idx[k]]);
  L.mult_bytes = by;
  L.mult = true;
}

// AP = A diag(!cmask) P on the device; false if a row overflows the
// per-CTA product buffer (then the caller runs the host loop)
static bool build_ap_device(Level& L, cudaStream_t s) {
  const int n = L.n;
  DevBuf<int> cnt(n), flag(1);
  DevBuf<long long> off(n + 1);
  flag.zero(s);
  ap_row_kernel<<<n, kApThreads, 0, s>>>(n, L.A.ptr.p, L.A.idx.p, L.A.val.p, L.cmask.p, L.P.ptr.p, L.P.idx.p,
                                         L.P.val.p, 0, cnt.p, nullptr, nullptr, nullptr, flag.p);
  FSI_CHECK_LAUNCH();
  int of = 0;
  FSI_CUDA(cudaMemcpyAsync(&of, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  FSI_CUDA(cudaStreamSynchronize(s));
  if (of) return false;
  std::vector<int> c = cnt.download(s);
  std::vector<long long> o(n + 1, 0);
  std::vector<int> p32(n + 1, 0);
  for (int i = 0; i < n; ++i) o[i + 1] = o[i] + c[i];
  require(o[n] < INT_MAX, "A*P: too many entries for int32 offsets");
  for (int i = 0; i <= n; ++i) p32[i] = (int)o[i];
  off.upload(o, s);
  const long long nnz = std::max<long long>(o[n], 1);
  DevBuf<int> ptr, idx(nnz);
  DevBuf<double> val(nnz);
  idx.zero(s);
  val.zero(s);
  ptr.upload(p32, s);
  ap_row_kernel<<<n, kApThreads, 0, s>>>(n, L.A.ptr.p, L.A.idx.p, L.A.val.p, L.cmask.p, L.P.ptr.p, L.P.idx.p,
                                         L.P.val.p, 1, nullptr, off.p, idx.p, val.p, flag.p);
  FSI_CHECK_LAUNCH();
  FSI_CUDA(cudaStreamSynchronize(s));
  L.AP.adopt(n, L.nc, std::move(ptr), std::move(idx), std::move(val));
  return true;
}

// FSIGPU_SETUP_TRACE=1: wall time of the setup phases on stderr
struct SetupTrace {
  const char* what;
  int level;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  static bool on() {
    static const bool v = [] {
      const char* e = std::getenv("FSIGPU_SETUP_TRACE");
      return e && e[0] == '1';
    }();
    return v;
  }
  SetupTrace(const char* w, int l) : what(w), level(l) {}
  ~SetupTrace() {
    if (!on()) return;
    cudaDeviceSynchronize();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[fsigpu setup] L%d %-24s %9.1f ms\n", level, what, ms);
  }
};

// Build one level from its descriptor (host arrays).
static void build_level(Gmg& g, int l, const fsigpu_level_desc& d, cudaStream_t s, bool mult) {
  Level& L = g.lv[l];
  require(d.n > 0, "gmg: empty level");
  L.n = d.n;
  require(d.a_ptr && d.a_idx && d.a_val && d.row_mask && d.col_mask, "gmg: null level arrays");
  std::unique_ptr<SetupTrace> tr(new SetupTrace("A, P, R upload", l));
  L.A.create(d.n, d.n, d.a_ptr, d.a_idx, d.a_val, s);
  // level operators (~65 entries per row) on HBM-bound levels: paired
  // 16-byte index/value loads, 4 pairs per lane (csr_pair_kernel). Cold
  // sweeps on config 2 (profiles/r01_tune_cfg2full_pair.txt): L4 5.0 -> 5.3,
  // L3 3.9 -> 4.2, L2 2.6 -> 2.8 TB/s. The FS operator (long rows) stays on
  // the scalar kernel, which is faster there.
  // In-graph sweep on config 2 (profiles/r02_tune_ingraph_cfg2.txt): 4 lanes
  // with 2 pairs per batch on every such level (1.25M rows 237 -> 217 us,
  // 313k 61 -> 55, 78k 19.4 -> 15.6).
  // Rows of the 3D hierarchies are longer (~176 entries): 8 lanes and
  // scalar batches of 8 there (232k rows: 111 -> 90 us, r02_tune_ingraph_3d.txt).
  if (d.n >= 65536 || force_big()) {
    const double per_row = (double)L.A.nnz / std::max(1, d.n);
    L.A.lpr = per_row > 100.0 ? 8 : 4;
    L.A.unroll = per_row > 100.0 ? 8 : 22;
  }
  L.A.build_pairs(s);
  L.A.build_blocks22(s);
  L.rmask.upload(d.row_mask, (size_t)d.n, s);
  L.cmask.upload(d.col_mask, (size_t)d.n, s);
  L.rbuf.alloc(d.n);
  if (l > 0) {
    L.bbuf.alloc(d.n);
    L.xbuf.alloc(d.n);
  } else {
    L.bbuf.alloc(d.n);
    L.xbuf.alloc(d.n);
  }
  L.b = L.bbuf.p;
  L.x = L.xbuf.p;
  if (l == 0) return;
  L.nc = d.nc;
  require(d.nc == g.lv[l - 1].n, "gmg: transfer size does not match the coarser level");
  L.P.create(d.n, d.nc, d.p_ptr, d.p_idx, d.p_val, s);
  L.R.create(d.nc, d.n, d.r_ptr, d.r_idx, d.r_val, s);
  // restriction rows are short (~14 entries): on large coarse levels paired
  // 16-byte loads with two lanes per row hold a whole row in one batch. Cold
  // sweeps on config 2 (profiles/r01_tune_restrict_cfg2.txt): 313k rows
  // 30.7 -> 24.4 us, 78k rows 13.9 -> 12.1; 20k rows: 8 lanes, batch 8.
  if (d.nc >= 65536) {
    L.R.lpr = 2;
    L.R.unroll = 24;
  } else if (d.nc >= 16384) {  // in-graph on config 2 (20k coarse rows): 3.5 -> 1.6 us with pairs
    L.R.lpr = 8;
    L.R.unroll = 22;
  } else {
    // small coarse levels: 32 lanes keep every SM busy (in-graph sweeps: the 3D
    // hierarchy's 4.6k coarse rows 4.1 -> 1.7 us; config 0 within 0.1 us of its best)
    L.R.lpr = 32;
    L.R.unroll = 22;
  }
  tr.reset(new SetupTrace("A*P", l));
  // AP_m = A * diag(!col_mask) * P on the device (ap_row_kernel); rows with
  // more than kApCap products (not in the 2D Q2 hierarchies) use the host loop
  if (!build_ap_device(L, s)) {
    std::vector<int> app(d.n + 1, 0), api;
    std::vector<double> apv, acc(d.nc, 0.0);
    std::vector<int> mark(d.nc, -1), touched;
    for (int i = 0; i < d.n; ++i) {
      touched.clear();
      for (int k = d.a_ptr[i]; k < d.a_ptr[i + 1]; ++k) {
        const int c = d.a_idx[k];
        if (d.col_mask[c]) continue;
        const double a = d.a_val[k];
        for (int q = d.p_ptr[c]; q < d.p_ptr[c + 1]; ++q) {
          const int cc = d.p_idx[q];
          if (mark[cc] != i) {
            mark[cc] = i;
            acc[cc] = 0.0;
            touched.push_back(cc);
          }
          acc[cc] += a * d.p_val[q];
        }
      }
      std::sort(touched.begin(), touched.end());
      for (int cc : touched) {
        api.push_back(cc);
        apv.push_back(acc[cc]);
      }
      app[i + 1] = (int)api.size();
    }
    if (api.empty()) {
      api.push_back(0);
      apv.push_back(0.0);
    }
    L.AP.create(d.n, d.nc, app.data(), api.data(), apv.data(), s);
  }
  {
    // its P half already adds 2 loads per lane to each batch: on large
    // (HBM-bound) levels batches of 4 AP entries; on small (L2-resident)
    // ones half the lanes with batches of 8 (warm sweeps, tools/tune_spmv.py)
    const bool pair_ap = d.n >= 65536 || (force_big() && d.n >= 4096);
    if (d.n < 16384 && !pair_ap) {
      L.AP.lpr = std::max(2, L.AP.lpr / 2);
      L.AP.unroll = 8;
    } else if (d.n < 65536 && !pair_ap) {
      // in-graph sweeps: config 0 (20k rows, 56 entries per row) 4.5 -> 4.3 us at
      // 8 lanes x 2 pairs (16 lanes: 6.0 us); the 3D hierarchy (31k rows, longer
      // rows) 8 lanes x 4 pairs
      L.AP.lpr = 8;
      L.AP.unroll = (double)L.AP.nnz / std::max(1, d.n) > 64.0 ? 24 : 22;
    } else if (pair_ap) {
      // HBM-bound levels: the A*P half as 16-byte pairs (cold sweeps on the
      // config-2 hierarchy, profiles/r01_tune_cfg2full_ap.txt: L4 227 -> 190
      // us at 2 lanes x 4 pairs, L3 67 -> 60 us at 4 lanes x 2 pairs)
      // (78k rows, in-graph: 18.1 -> 14.1 us at 4 lanes x 4 pairs)
      L.AP.lpr = d.n >= 1048576 ? 2 : 4;
      L.AP.unroll = 24;  // 4 pairs per batch on every such level (232k rows 3D: 82.6 -> 73.1 us)
    } else {
      L.AP.unroll = 4;
    }
    // column-pair format of A*P on the large levels (keeps the lane count, 2 elements per batch)
    {
      const int keep_lpr = L.AP.lpr, keep_unroll = L.AP.unroll;
      // 2 x 2 blocks of A*P on the HBM-bound levels (config 2 in-graph: 1.25M rows
      // 174 -> 159 us, 313k rows 48 -> 39 us; on config 0's 20k rows 3.7 -> 4.5 us, so not there)
      L.AP.build_pairs(s);
      L.AP.build_blocks22(s);
      if (L.AP.blocks22) {
        L.AP.lpr = std::max(keep_lpr, 4);  // 1.25M rows: 159 -> 148 us at 4 lanes per row pair
        L.AP.unroll = 4;
      } else if (L.AP.pairs && (d.n >= 65536 || force_big())) {
        L.AP.lpr = keep_lpr;
        L.AP.unroll = 4;
      } else {
        L.AP.pairs = false;
        L.AP.lpr = keep_lpr;
        L.AP.unroll = keep_unroll;
      }
    }
  }
  require(d.g1 >= 0 && d.n_us >= 0 && d.g1 + d.n_us <= d.n, "fs: bad group sizes");
  L.g1 = d.g1;
  L.n_us = d.n_us;
  L.lumped.upload(d.lumped, (size_t)d.n_us, s);
  // blocks: AS1 (frame positions) then AS2 (group-2 local -> +g1)
  const int nb1 = d.as1_n, nb2 = d.as2_n;
  std::vector<int> sizes;
  std::vector<int> pos;
  for (int b = 0; b < nb1; ++b) {
    const int m = d.as1_ptr[b + 1] - d.as1_ptr[b];
    sizes.push_back(m);
    for (int k = d.as1_ptr[b]; k < d.as1_ptr[b + 1]; ++k) {
      const int p = d.as1_idx[k];
      require(p >= 0 && p < d.g1, "fs: AS1 index outside group 1");
      require(k == d.as1_ptr[b] || p > d.as1_idx[k - 1], "fs: AS1 set not sorted/unique");
      pos.push_back(p);
    }
  }
  for (int b = 0; b < nb2; ++b) {
    const int m = d.as2_ptr[b + 1] - d.as2_ptr[b];
    sizes.push_back(m);
    for (int k = d.as2_ptr[b]; k < d.as2_ptr[b + 1]; ++k) {
      const int p = d.as2_idx[k];
      require(p >= 0 && p < d.n - d.g1, "fs: AS2 index outside group 2");
      require(k == d.as2_ptr[b] || p > d.as2_idx[k - 1], "fs: AS2 set not sorted/unique");
      require(p >= d.n_us, "fs: AS2 block touches the lumped solid-velocity range");
      pos.push_back(p + d.g1);
    }
  }
  L.n_as1 = nb1;
  tr.reset(new SetupTrace("blocks extract + LU", l));
  Blocks& B = L.blocks;
  // assembled and multiplicative smoothers build on the inverses
  B.mode = (g_default_mode == kModeLU && !mult) ? kModeLU : kModeInverse;
  B.layout(sizes, s);
  B.pos.upload(pos, s);
  DevBuf<double> dense((size_t)std::max<long long>(B.h_lu_off[B.nb], 1));
  L.delta.alloc((size_t)std::max<long long>(B.total_rows, 1));
  // extract + factor (factor_principal_block for every block)
  if (B.nb) {
    dense.zero(s);
    extract_blocks_kernel<<<(int)B.nb, 256, 0, s>>>((int)B.nb, B.m.p, B.lu_off.p, B.row_off.p, B.pos.p, 0, L.A.ptr.p,
                                                    L.A.idx.p, L.A.val.p, dense.p);
    FSI_CHECK_LAUNCH();
    try {
      B.factor(dense.p, B.pos.p, 0, s);
    } catch (Error& e) {
      if (e.code == FSIGPU_ERR_SINGULAR) g_bad_level = l;
      throw Error(e.code, std::string(e.what()) + " (level " + std::to_string(l) + ")");
    }
  }
  // inverse map position -> delta slots in block order (precond.cpp:52-55)
  tr.reset(new SetupTrace("maps", l));
  std::vector<int> cnt(d.n + 1, 0);
  for (int p : pos) cnt[p + 1]++;
  for (int i = 0; i < d.n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int> inv(pos.size()), nxt(cnt.begin(), cnt.end() - 1);
  for (size_t k = 0; k < pos.size(); ++k) inv[nxt[pos[k]]++] = (int)k;
  L.inv_ptr.upload(cnt, s);
  L.inv_idx.upload(inv, s);
  L.combine_bytes = 4.0 * (d.n + 1) + 4.0 * inv.size() + 8.0 * inv.size() + 8.0 * 2 * d.n + 8.0 * d.n_us;
  // A_g2[:, :n_us] rows (Jacobi residual update, precond.cpp:281-287)
  const int g2 = d.n - d.g1;
  std::vector<int> ap(g2 + 1, 0), ac;
  std::vector<double> av;
  for (int q = 0; q < g2; ++q) {
    const int row = d.g1 + q;
    for (int k = d.a_ptr[row]; k < d.a_ptr[row + 1]; ++k) {
      const int c = d.a_idx[k] - d.g1;
      if (c >= 0 && c < d.n_us) {
        ac.push_back(c);
        av.push_back(d.a_val[k]);
      }
    }
    ap[q + 1] = (int)ac.size();
  }
  L.aus_ptr.upload(ap, s);
  L.aus_col.upload(ac.empty() ? std::vector<int>{0} : ac, s);
  L.aus_val.upload(av.empty() ? std::vector<double>{0.0} : av, s);
  // the reference rejects a non-positive lumped row sum (precond.cpp:239-241)
  for (int i = 0; i < d.n_us; ++i)
    if (!(d.lumped[i] > 0.0)) {
      g_bad_block = -1;
      g_bad_level = l;
      throw Error(FSIGPU_ERR_SINGULAR, "singular block: fs lumped mass row " + std::to_string(i));
    }
  FSI_CUDA(cudaStreamSynchronize(s));
  tr.reset(new SetupTrace(mult ? "multicolour" : "assembled FS", l));
  if (mult)
    build_mult(L, d, s);
  else if (g_default_mode == kModeAssembled)
    assemble_fs(L, d, pos, cnt, ap, ac, av, s);
}

// Coarse operator: equilibrate (sparse_lu.cpp:104-121), Gauss-Jordan
// inverse on the device, fold the scalings into the inverse.
static void build_coarse(Gmg& g, const fsigpu_level_desc& d, cudaStream_t s) {
  SetupTrace tr("coarse inverse", 0);
  const int n = d.n;
  std::vector<double> rs(n, 1.0), cs(n, 1.0), cm(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double mx = 0.0;
    for (int k = d.a_ptr[i]; k < d.a_ptr[i + 1]; ++k) mx = std::max(mx, std::fabs(d.a_val[k]));
    if (mx > 0.0) rs[i] = 1.0 / mx;
  }
  for (int i = 0; i < n; ++i)
    for (int k = d.a_ptr[i]; k < d.a_ptr[i + 1]; ++k)
      cm[d.a_idx[k]] = std::max(cm[d.a_idx[k]], std::fabs(d.a_val[k]) * rs[i]);
  for (int j = 0; j < n; ++j)
    if (cm[j] > 0.0) cs[j] = 1.0 / cm[j];
  // [diag(rs) A diag(cs) | I] built on the device from the level's CSR
  const Csr& A0 = g.lv[0].A;
  DevBuf<double> Wd((size_t)n * 2 * n), f(n), drs, dcs;
  Wd.zero(s);
  drs.upload(rs, s);
  dcs.upload(cs, s);
  DevBuf<int> fail(1), piv(n);
  fail.zero(s);
  gj_init_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, A0.ptr.p, A0.idx.p, A0.val.p, drs.p, dcs.p, Wd.p);
  for (int k = 0; k < n; ++k) {
    gj_pivot_kernel<<<1, 1024, 0, s>>>(n, Wd.p, k, f.p, fail.p, piv.p);
    dim3 grid(ceil_div((long long)n, 256), n);
    gj_eliminate_kernel<<<grid, 256, 0, s>>>(n, Wd.p, k, f.p);
  }
  FSI_CHECK_LAUNCH();
  // the right half's columns, unpermuted: apply the swaps (k <-> piv[k]) in reverse
  std::vector<int> pv = piv.download(s), col(n);
  for (int j = 0; j < n; ++j) col[j] = j;
  for (int k = n - 1; k >= 0; --k) std::swap(col[k], col[pv[k]]);
  DevBuf<int> dcol;
  dcol.upload(col, s);
  g.coarse_inv.alloc((size_t)n * n);
  gj_extract_kernel<<<ceil_div((long long)n * n, 256), 256, 0, s>>>(n, Wd.p, dcol.p, drs.p, dcs.p, g.coarse_inv.p);
  FSI_CHECK_LAUNCH();
  int bad = 0;
  FSI_CUDA(cudaMemcpyAsync(&bad, fail.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  FSI_CUDA(cudaStreamSynchronize(s));
  if (bad) {
    g_bad_block = -1;
    g_bad_level = 0;
    throw Error(FSIGPU_ERR_SINGULAR, "singular block: gmg-coarse");
  }
}

// Pack the read-only arrays every V-cycle streams into one arena (one
// contiguous allocation; an L2 persisting window over it measured slower on
// config 0 and was dropped).
static void pin_hot_data(Gmg& g) {
  std::vector<std::function<void(char*)>> movers;
  size_t total = 0;
  auto add = [&](auto& buf) {
    using T = typename std::remove_reference<decltype(*buf.p)>::type;
    if (!buf.n) return;
    const size_t bytes = (buf.n * sizeof(T) + 255) & ~size_t(255);
    const size_t off = total;
    total += bytes;
    movers.push_back([&buf, off, &g](char* base) { buf.rebase(reinterpret_cast<T*>(base + off), g.s); });
  };
  for (size_t l = 0; l < g.lv.size(); ++l) {
    Level& L = g.lv[l];
    add(L.A.val);
    add(L.A.idx);
    add(L.A.ptr);
    if (l == 0) continue;
    add(L.blocks.inv);
    add(L.P.val);
    add(L.P.idx);
    add(L.P.ptr);
    add(L.R.val);
    add(L.R.idx);
    add(L.R.ptr);
  }
  add(g.coarse_inv);
  if (!total) return;
  g.arena.alloc(total);
  for (auto& mv : movers) mv(g.arena.p);
}

// ------------------------------------------------------------ GMRES
struct Gmres {
  Gmg* g = nullptr;
  int n = 0, mr = 30;
  int grid = 0;
  bool graphs = true;
  DevBuf<double> scale, V, Z, w, zbuf, ubuf, r, x, b, H, cs, sn, gv, hist, partial, partial2, partialw;
  DevBuf<unsigned int> ticket;
  DevBuf<KState> st;
  KBufs kb{};
  int hist_cap = 0;
  cudaGraphExec_t cycle_exec = nullptr;
  cudaGraph_t cycle_graph = nullptr;
  int graph_version = -1;  // Gmg::version the graph was captured at
  int graph_stamp_epoch = 0;  // g_stamp_epoch the graph was captured at (stamp pointers are baked in)

  ~Gmres() {
    if (cycle_exec) cudaGraphExecDestroy(cycle_exec);
    if (cycle_graph) cudaGraphDestroy(cycle_graph);
  }

  void ensure_history(int max_iters) {
    if (max_iters + 2 > hist_cap) {
      hist_cap = max_iters + 2;
      hist.alloc(hist_cap);
      kb.history = hist.p;
      if (cycle_exec) {
        cudaGraphExecDestroy(cycle_exec);
        cudaGraphDestroy(cycle_graph);
        cycle_exec = nullptr;
        cycle_graph = nullptr;
      }
    }
  }

  // w = A_s z (scaled SpMV)
  void outer_spmv(const double* z, double* out) {
    Level& T = g->lv.back();
    ProfScope ps(FSIGPU_K_SPMV, T.A.bytes(false) + 8.0 * n, g->s);
    T.A.launch(GatherPlain{z}, EpiScaled{scale.p, out}, g->s);
  }
  void outer_resid() {
    Level& T = g->lv.back();
    ProfScope ps(FSIGPU_K_SPMV, T.A.bytes(true) + 8.0 * n, g->s);
    T.A.launch(GatherPlain{x.p}, EpiResidScaled{b.p, scale.p, r.p}, g->s);
  }
  // restart > 32: the chunked five-kernel step of krylov_wide.cuh
  void arnoldi_wide(const KBufs& kk) {
    cudaStream_t s = g->s;
    const int pw = kk.parts_w;
    const int chunks = ceil_div(mr, kRegRestart);
    {
      ProfScope ps(FSIGPU_K_SPMV, g->lv.back().A.bytes(false) + 8.0 * n * 3, s);
      launch_k(k_wide_spmv, dim3(pw), dim3(kWideThreads), 0, s, kk);
    }
    ProfScope ps(FSIGPU_K_ARNOLDI, 8.0 * n * 6, s);
    launch_k(k_wide_dots<false>, dim3(pw, chunks), dim3(kWideThreads), 0, s, kk);
    launch_k(k_wide_update, dim3(pw), dim3(kWideThreads), 0, s, kk);
    launch_k(k_wide_dots<true>, dim3(pw, chunks), dim3(kWideThreads), 0, s, kk);
    launch_k(k_wide_normalize, dim3(pw + 1), dim3(kWideThreads), 0, s, kk);
    FSI_CHECK_LAUNCH();
    counted(5);
  }
  // outer SpMV + CGS2 Arnoldi + Givens + normalisation: 3 fused kernels
  void arnoldi_fused(const KBufs& kin) {
    if (mr > kRegRestart) {
      arnoldi_wide(kin);
      return;
    }
    KBufs kk = kin;
    // device-clock stamps of (A), (B), (C): class ARNOLDI, no level, subs 0..2
    kk.stamp = g_stamp_on ? g_stamp_buf + 4 * ((size_t)FSIGPU_K_ARNOLDI * (Profiler::kLv + 1) * kStampSubs) : nullptr;
    cudaStream_t s = g->s;
    Level& T = g->lv.back();
    const int gs = kk.parts_a;
    {
      ProfScope ps(FSIGPU_K_SPMV, T.A.bytes(false) + 8.0 * n * 3, s);
      // small systems: 128-row tiles, 8 lanes per row (1024 threads), grid-stride over tiles
      if (kk.fuse_small) {
        // large systems: the SpMV as its own launch (bsr22_kernel when A is held
        // as 2 x 2 blocks, else the CSR kernels), then the dots and the Z[j] copy
        g_prof.level = -1;
        T.A.launch(GatherPlain{kk.zbuf}, EpiScaled{kk.scale, kk.w}, s);
        launch_k(k_dots_copy, dim3(gs), dim3(kDotsThreads), 0, s, kk);
        counted();
      } else if (gs == ceil_div(n, kFuseRows))
        launch_k(k_spmv_dots_1<8>, dim3(gs), dim3(kFuseThreads), 0, s, kk);
      else
        launch_k(k_spmv_dots<8>, dim3(gs), dim3(kFuseThreads), 0, s, kk);
    }
    {
      // (B) on parts_b CTAs; (C) on parts_b row CTAs + 1 Givens CTA
      ProfScope ps(FSIGPU_K_ARNOLDI, 8.0 * n * 4, s);
      if (kk.fuse_small) {  // large systems: multi-row register loops, (C) on its own grid
        launch_k(k_update_dots_norm_mr, dim3(kk.parts_b), dim3(kArnThreads), 0, s, kk);
        launch_k(k_update_normalize<false>, dim3(kk.parts_c + 1), dim3(kArnThreads), 0, s, kk);
      } else {
        launch_k(k_update_dots_norm<true>, dim3(kk.parts_b), dim3(kArnThreads), 0, s, kk);
        launch_k(k_update_normalize<true>, dim3(kk.parts_b + 1), dim3(kArnThreads), 0, s, kk);
      }
    }
    FSI_CHECK_LAUNCH();
    counted(3);
  }
  void step_body(const KBufs& kk) {
    g->apply(ubuf.p, zbuf.p);
    arnoldi_fused(kk);
  }
  void cycle_tail() {
    cudaStream_t s = g->s;
    launch_k(k_solve_y, dim3(1), dim3(256), 0, s, kb);
    // x += Z y: one row per thread (a grid-stride loop over ~16 rows per
    // thread left the config-2 update at 1.1 TB/s)
    launch_k(k_update_x, dim3(std::max(grid, (int)ceil_div(n, kKThreads))), dim3(kKThreads), 0, s, kb);
    outer_resid();
    launch_k(k_norm_r, dim3(grid), dim3(kKThreads), 0, s, kb);
    FSI_CHECK_LAUNCH();
    counted(3);
  }

  long long pre_launches = 0, body_launches = 0, post_launches = 0;

  void build_graph() {
    cudaStream_t s = g->s;
    FSI_CUDA(cudaGraphCreate(&cycle_graph, 0));
    cudaGraphConditionalHandle h;
    FSI_CUDA(cudaGraphConditionalHandleCreate(&h, cycle_graph, 1, cudaGraphCondAssignDefault));
    // prefix: v0 = r / beta
    cudaGraph_t pre_g, post_g;
    const long long c0 = g_launches;
    FSI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    k_cycle_start<<<grid, kKThreads, 0, s>>>(kb);
    FSI_CUDA(cudaStreamEndCapture(s, &pre_g));
    pre_launches = 1;
    cudaGraphNode_t n_pre, n_cond, n_post;
    FSI_CUDA(cudaGraphAddChildGraphNode(&n_pre, cycle_graph, nullptr, 0, pre_g));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    FSI_CUDA(cudaGraphAddNode(&n_cond, cycle_graph, &n_pre, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    FSI_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const long long c1 = g_launches;
    KBufs kc = kb;  // the Givens step sets the WHILE condition
    kc.cond = h;
    kc.use_cond = 1;
    step_body(kc);
    FSI_CUDA(cudaStreamEndCapture(s, &body));
    body_launches = g_launches - c1;
    const long long c2 = g_launches;
    FSI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cycle_tail();
    FSI_CUDA(cudaStreamEndCapture(s, &post_g));
    post_launches = g_launches - c2;
    g_launches = c0;  // capture itself launches nothing
    FSI_CUDA(cudaGraphAddChildGraphNode(&n_post, cycle_graph, &n_cond, 1, post_g));
    FSI_CUDA(cudaGraphInstantiate(&cycle_exec, cycle_graph, 0));
    cudaGraphDestroy(pre_g);
    cudaGraphDestroy(post_g);
  }

  KState read_state() {
    KState h;
    FSI_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(KState), cudaMemcpyDeviceToHost, g->s));
    FSI_CUDA(cudaStreamSynchronize(g->s));
    return h;
  }

  // krylov.cpp:20-126 control flow, device resident
  void solve(int max_iters, double rel_tol, double abs_tol, fsigpu_gmres_result* res) {
    require(max_iters >= 0, "gmres: invalid config");
    require(rel_tol > 0.0 && abs_tol > 0.0, "gmres: invalid config");
    ensure_history(max_iters);
    cudaStream_t s = g->s;
    KState h0{};
    h0.max_iters = max_iters;
    h0.restart = mr;
    h0.first = 1;
    h0.rel_tol = rel_tol;
    h0.abs_tol = abs_tol;
    FSI_CUDA(cudaMemcpyAsync(st.p, &h0, sizeof(KState), cudaMemcpyHostToDevice, s));
    outer_resid();
    k_norm_r<<<grid, kKThreads, 0, s>>>(kb);
    FSI_CHECK_LAUNCH();
    counted();
    KState h = read_state();
    long long cycles = 0;
    const bool use_graph = graphs && !g_prof.on;
    if (cycle_exec && (graph_version != g->version || graph_stamp_epoch != g_stamp_epoch)) {
      cudaGraphExecDestroy(cycle_exec);
      cudaGraphDestroy(cycle_graph);
      cycle_exec = nullptr;
      cycle_graph = nullptr;
    }
    if (use_graph && !cycle_exec) {
      build_graph();
      graph_version = g->version;
      graph_stamp_epoch = g_stamp_epoch;
    }
    while (!h.converged && h.its < max_iters) {
      const int its_before = h.its;
      if (use_graph) {
        FSI_CUDA(cudaGraphLaunch(cycle_exec, s));
      } else {
        k_cycle_start<<<grid, kKThreads, 0, s>>>(kb);
        FSI_CHECK_LAUNCH();
        counted();
        while (true) {
          step_body(kb);
          KState t = read_state();
          if (t.stop || t.j >= mr || t.its >= max_iters) break;
        }
        cycle_tail();
      }
      h = read_state();
      if (use_graph) g_launches += pre_launches + body_launches * (h.its - its_before) + post_launches;
      ++cycles;
      if (h.breakdown) break;
    }
    res->iterations = h.its;
    res->converged = h.converged;
    res->breakdown = h.breakdown;
    res->n_history = h.its + 1;
    res->m_applies = h.its;  // FGMRES: one V-cycle per Arnoldi step
    res->true_residual = h.beta;
    if (g_prof.on) g_prof.flush();
  }
};

}  // namespace fsigpu

struct fsigpu_gmg_t {
  fsigpu::Gmg g;
};
struct fsigpu_sets_t {
  std::vector<int> as1_ptr{0}, as1_idx, as2_ptr{0}, as2_idx;
  std::vector<double> lumped;
  std::vector<std::string> labels;  // AS1 then AS2 blocks
};

namespace fsigpu {

// Device-side block-set construction (sets.cuh). Host side: the element
// partition by region and the node -> element adjacency (index maps of the
// mesh, O(elements)), the count scan, and the labels.
struct SetBuilder {
  const fsigpu_mesh_desc& m;
  cudaStream_t s;
  std::vector<int> solid, fluid;
  DevBuf<int> d_solid, d_fluid, en, ne_ptr, ne_idx, dpos, upos, ppos, cnt, out, overflow;
  DevBuf<long long> off;
  DevBuf<unsigned char> esol, nsol, drop, g1e;
  SetBuilder(const fsigpu_mesh_desc& mesh, int n_frame, cudaStream_t st) : m(mesh), s(st) {
    require(m.n_elements >= 0 && m.n_nodes >= 0 && m.nodes_per_element >= 1 && m.nodes_per_element <= 27 &&
                m.dim >= 1 && m.dim <= 3 && m.p_per_element >= 0 && m.p_per_element <= 4,
            "sets: bad mesh sizes");
    require(m.element_nodes && m.elem_solid && m.node_solid && m.d_pos && m.u_pos && m.p_pos, "sets: null mesh arrays");
    const int E = m.n_elements, N = m.n_nodes, npe = m.nodes_per_element;
    for (int e = 0; e < E; ++e) (m.elem_solid[e] ? solid : fluid).push_back(e);
    std::vector<int> np(N + 1, 0), ni((size_t)E * npe);
    for (long long q = 0; q < (long long)E * npe; ++q) {
      const int node = m.element_nodes[q];
      require(node >= 0 && node < N, "sets: element node out of range");
      np[node + 1]++;
    }
    for (int i = 0; i < N; ++i) np[i + 1] += np[i];
    {
      std::vector<int> nx(np.begin(), np.end() - 1);
      for (int e = 0; e < E; ++e)
        for (int a = 0; a < npe; ++a) ni[nx[m.element_nodes[(size_t)e * npe + a]]++] = e;
    }
    for (long long q = 0; q < (long long)N * m.dim; ++q)
      require(m.d_pos[q] >= 0 && m.d_pos[q] < n_frame && m.u_pos[q] >= 0 && m.u_pos[q] < n_frame,
              "sets: d/u position out of the frame");
    for (long long q = 0; q < (long long)E * m.p_per_element; ++q)
      require(m.p_pos[q] >= 0 && m.p_pos[q] < n_frame, "sets: p position out of the frame");
    auto up = [&](DevBuf<int>& d, const std::vector<int>& v) { d.upload(v.empty() ? std::vector<int>{0} : v, s); };
    up(d_solid, solid);
    up(d_fluid, fluid);
    en.upload(m.element_nodes, (size_t)std::max<long long>((long long)E * npe, 1), s);
    up(ne_ptr, np);
    up(ne_idx, ni);
    dpos.upload(m.d_pos, (size_t)std::max(N * m.dim, 1), s);
    upos.upload(m.u_pos, (size_t)std::max(N * m.dim, 1), s);
    ppos.upload(m.p_pos, (size_t)std::max(E * m.p_per_element, 1), s);
    esol.upload(m.elem_solid, (size_t)std::max(E, 1), s);
    nsol.upload(m.node_solid, (size_t)std::max(N, 1), s);
    if (m.drop) drop.upload(m.drop, (size_t)std::max(n_frame, 1), s);
    overflow.alloc(1);
    overflow.zero(s);
  }
  // sets of one kind over `list` (element chunks of epb) appended to ptr/idx
  void run(int kind, const std::vector<int>& list, const DevBuf<int>& dlist, int epb, int overlap, int g1,
           std::vector<int>& ptr, std::vector<int>& idx) {
    const int np = list.empty() ? 0 : ceil_div((long long)list.size(), epb);
    if (np == 0) return;
    SetArgs a{};
    a.kind = kind;
    a.epb = epb;
    a.overlap = overlap;
    a.n_list = (int)list.size();
    a.npe = m.nodes_per_element;
    a.dim = m.dim;
    a.ppe = m.p_per_element;
    a.g1 = g1;
    a.list = dlist.p;
    a.en = en.p;
    a.elem_solid = esol.p;
    a.node_solid = nsol.p;
    a.ne_ptr = ne_ptr.p;
    a.ne_idx = ne_idx.p;
    a.d_pos = dpos.p;
    a.u_pos = upos.p;
    a.p_pos = ppos.p;
    a.drop = drop.n ? drop.p : nullptr;
    a.g1_empty = g1e.n ? g1e.p : nullptr;
    a.overflow = overflow.p;
    cnt.alloc(np);
    a.count = cnt.p;
    set_patch_kernel<<<np, kSetThreads, 0, s>>>(a, 0);
    FSI_CHECK_LAUNCH();
    std::vector<int> c = cnt.download(s);
    int of = 0;
    FSI_CUDA(cudaMemcpy(&of, overflow.p, sizeof(int), cudaMemcpyDeviceToHost));
    require(!of, "sets: a patch exceeds the per-CTA capacity (4096 dof positions, 1024 elements)");
    std::vector<long long> o(np + 1, 0);
    for (int q = 0; q < np; ++q) o[q + 1] = o[q] + c[q];
    require(o[np] < INT_MAX, "sets: too many positions");
    off.upload(o, s);
    out.alloc((size_t)std::max<long long>(o[np], 1));
    a.off = off.p;
    a.out = out.p;
    set_patch_kernel<<<np, kSetThreads, 0, s>>>(a, 1);
    FSI_CHECK_LAUNCH();
    std::vector<int> v = out.download(s);
    const int base = (int)idx.size();
    idx.insert(idx.end(), v.begin(), v.begin() + o[np]);
    for (int q = 0; q < np; ++q) ptr.push_back(base + (int)o[q + 1]);
  }
};

}  // namespace fsigpu
struct fsigpu_gmres_t {
  fsigpu::Gmres k;
};

using namespace fsigpu;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return FSIGPU_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return FSIGPU_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FSIGPU_ERR_CUDA;
  }
}

static cudaStream_t new_stream() {
  cudaStream_t s;
  FSI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

extern "C" {

const char* fsigpu_last_error(void) { return g_err.c_str(); }
int fsigpu_last_singular_block(void) { return g_bad_block; }
int fsigpu_last_singular_level(void) { return g_bad_level; }
int fsigpu_version(void) { return 1; }
long long fsigpu_launch_count(void) { return g_launches; }
int fsigpu_set_pdl(int enable) {
  return guarded([&] { g_pdl = enable != 0; });
}
// Tuning: launch shape (lanes per row, entries per lane per batch) of one
// level matrix. which: 0 A, 1 FS, 2 AP, 3 P, 4 R.
int fsigpu_gmg_set_launch(fsigpu_gmg h, int level, int which, int lpr, int unroll) {
  return guarded([&] {
    require(h != nullptr && level >= 0 && level < (int)h->g.lv.size(), "launch: bad level");
    require(lpr == 2 || lpr == 4 || lpr == 8 || lpr == 16 || lpr == 32 || (lpr == 1 && (unroll == 22 || unroll == 24)),
            "launch: lpr must be 2..32 (1 with paired loads)");
    require(unroll == 4 || unroll == 8 || unroll == 22 || unroll == 24,
            "launch: unroll must be 4 or 8 (22/24: paired loads, 2/4 pairs)");
    Level& L = h->g.lv[level];
    Csr* c = which == 0 ? &L.A : which == 1 ? &L.FS : which == 2 ? &L.AP : which == 3 ? &L.P : &L.R;
    c->lpr = lpr;
    c->unroll = unroll;
    ++h->g.version;  // captured solver graphs hold the old launch shape
  });
}
// Level smoother: 0 damped Richardson (the reference's richardson_smooth,
// precond.cpp:305-317), 1 GMRES(1) minimal-residual step (mr.cuh).
int fsigpu_gmg_set_smoother(fsigpu_gmg h, int kind) {
  return guarded([&] {
    require(h != nullptr, "gmg: null");
    require(kind == 0 || kind == 1, "smoother must be 0 (richardson) or 1 (gmres1)");
    std::lock_guard<std::mutex> lk(h->g.mu);
    h->g.set_smoother(kind);
  });
}
int fsigpu_set_block_mode(int mode) {
  return guarded([&] {
    require(mode == kModeLU || mode == kModeInverse || mode == kModeAssembled,
            "block mode must be 0 (LU), 1 (inverse) or 2 (assembled)");
    g_default_mode = mode;
  });
}
void* fsigpu_gmg_stream(fsigpu_gmg g) { return g ? (void*)g->g.s : nullptr; }

int fsigpu_init(int device) {
  return guarded([&] {
    int n = 0;
    FSI_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "init: no such CUDA device");
    FSI_CUDA(cudaSetDevice(device));
    FSI_CUDA(cudaFree(nullptr));
  });
}

// ---- CSR
int fsigpu_csr_create(int rows, int cols, const int* ptr, const int* idx, const double* val, fsigpu_csr* out) {
  return guarded([&] {
    auto h = std::make_unique<fsigpu_csr_t>();
    h->s = new_stream();
    h->a.create(rows, cols, ptr, idx, val, h->s, true);
    *out = h.release();
  });
}

int fsigpu_csr_multiply_dev(fsigpu_csr a, const double* dx, double* dy, void* stream) {
  return guarded([&] {
    require(a != nullptr, "spmv: null matrix");
    cudaStream_t s = stream ? (cudaStream_t)stream : a->s;
    ProfScope ps(FSIGPU_K_SPMV, a->a.bytes(false), s);
    a->a.launch(GatherPlain{dx}, EpiPlain{dy}, s);
  });
}

int fsigpu_csr_multiply(fsigpu_csr a, const double* x, double* y) {
  return guarded([&] {
    require(a != nullptr, "spmv: null matrix");
    DevBuf<double> dx, dy(a->a.rows);
    dx.upload(x, (size_t)a->a.cols, a->s);
    a->a.launch(GatherPlain{dx.p}, EpiPlain{dy.p}, a->s);
    FSI_CHECK_LAUNCH();
    if (a->a.rows) FSI_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * a->a.rows, cudaMemcpyDeviceToHost, a->s));
    FSI_CUDA(cudaStreamSynchronize(a->s));
  });
}

int fsigpu_csr_time(fsigpu_csr a, int reps, double* ms) {
  return guarded([&] {
    require(a != nullptr && reps > 0, "csr_time: bad args");
    DevBuf<double> dx(a->a.cols), dy(a->a.rows);
    FSI_CUDA(cudaMemsetAsync(dx.p, 0, sizeof(double) * dx.n, a->s));
    for (int i = 0; i < 3; ++i) a->a.launch(GatherPlain{dx.p}, EpiPlain{dy.p}, a->s);
    cudaEvent_t e0, e1;
    FSI_CUDA(cudaEventCreate(&e0));
    FSI_CUDA(cudaEventCreate(&e1));
    FSI_CUDA(cudaEventRecord(e0, a->s));
    for (int i = 0; i < reps; ++i) a->a.launch(GatherPlain{dx.p}, EpiPlain{dy.p}, a->s);
    FSI_CUDA(cudaEventRecord(e1, a->s));
    FSI_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    FSI_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

void fsigpu_csr_destroy(fsigpu_csr a) {
  if (!a) return;
  cudaStreamSynchronize(a->s);
  cudaStreamDestroy(a->s);
  delete a;
}

// ---- blocks
int fsigpu_blocks_factor_csr(fsigpu_csr a, int n_blocks, const int* block_ptr, const int* block_idx,
                             fsigpu_blocks* out) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(a != nullptr && n_blocks >= 0, "blocks: bad args");
    require(a->a.rows == a->a.cols, "schwarz: matrix not square");
    auto h = std::make_unique<fsigpu_blocks_t>();
    h->s = a->s;
    std::vector<int> sizes(n_blocks);
    std::vector<int> pos;
    for (int b = 0; b < n_blocks; ++b) {
      sizes[b] = block_ptr[b + 1] - block_ptr[b];
      for (int k = block_ptr[b]; k < block_ptr[b + 1]; ++k) {
        require(block_idx[k] >= 0 && block_idx[k] < a->a.rows, "index set: index out of range");
        require(k == block_ptr[b] || block_idx[k] > block_idx[k - 1], "index set: not sorted/unique");
        pos.push_back(block_idx[k]);
      }
    }
    Blocks& B = h->b;
    B.layout(sizes, h->s, true);
    B.pos.upload(pos, h->s);
    if (B.nb) {
      DevBuf<double> dense((size_t)B.h_lu_off[B.nb]);
      dense.zero(h->s);
      extract_blocks_kernel<<<(int)B.nb, 256, 0, h->s>>>((int)B.nb, B.m.p, B.lu_off.p, B.row_off.p, B.pos.p, 0,
                                                         a->a.ptr.p, a->a.idx.p, a->a.val.p, dense.p);
      FSI_CHECK_LAUNCH();
      B.factor(dense.p, nullptr, 0, h->s);
    }
    *out = h.release();
  });
}

int fsigpu_blocks_factor_dense(int n_blocks, const int* sizes, const double* mats, fsigpu_blocks* out) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(n_blocks >= 0, "blocks: bad args");
    auto h = std::make_unique<fsigpu_blocks_t>();
    h->s = new_stream();
    h->own_stream = 1;
    std::vector<int> sz(sizes, sizes + n_blocks);
    Blocks& B = h->b;
    B.layout(sz, h->s, true);
    // row-major (DenseMatrix) -> column-major device layout
    std::vector<double> cm((size_t)B.h_lu_off[B.nb]);
    for (long long b = 0; b < B.nb; ++b) {
      const int m = sz[b];
      const double* src = mats + B.h_lu_off[b];
      double* dst = cm.data() + B.h_lu_off[b];
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) dst[(size_t)j * m + i] = src[(size_t)i * m + j];
    }
    B.orig.upload(cm, h->s);
    h->have_orig = 1;
    if (B.nb) B.factor(B.orig.p, nullptr, 0, h->s);
    *out = h.release();
  });
}

int fsigpu_blocks_generate_dominant(long long n54, long long n59, unsigned long long seed, fsigpu_blocks* out) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(n54 >= 0 && n59 >= 0, "blocks: bad counts");
    auto h = std::make_unique<fsigpu_blocks_t>();
    h->s = new_stream();
    h->own_stream = 1;
    std::vector<int> sz;
    sz.reserve(n54 + n59);
    for (long long i = 0; i < n54; ++i) sz.push_back(54);
    for (long long i = 0; i < n59; ++i) sz.push_back(59);
    Blocks& B = h->b;
    B.layout(sz, h->s);
    B.orig.alloc((size_t)B.h_lu_off[B.nb]);
    std::vector<long long> rb(B.total_rows);
    for (long long b = 0; b < B.nb; ++b)
      for (long long r = B.h_row_off[b]; r < B.h_row_off[b + 1]; ++r) rb[r] = b;
    DevBuf<long long> drb;
    drb.upload(rb, h->s);
    gen_dominant_kernel<<<ceil_div(B.total_rows, 256), 256, 0, h->s>>>(B.nb, B.m.p, B.lu_off.p, B.row_off.p,
                                                                       B.total_rows, seed, B.orig.p, drb.p);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(h->s));
    h->have_orig = 1;
    if (B.nb) B.factor(B.orig.p, nullptr, 0, h->s);
    *out = h.release();
  });
}

int fsigpu_blocks_generate_rhs(fsigpu_blocks b, unsigned long long seed, double* d_rhs) {
  return guarded([&] {
    require(b != nullptr, "blocks: null");
    gen_rhs_kernel<<<ceil_div(b->b.total_rows, 256), 256, 0, b->s>>>(b->b.total_rows, seed, d_rhs);
    FSI_CHECK_LAUNCH();
    FSI_CUDA(cudaStreamSynchronize(b->s));
  });
}

int fsigpu_blocks_copy_matrix(fsigpu_blocks b, long long block, double* rowmajor) {
  return guarded([&] {
    require(b != nullptr && b->have_orig && block >= 0 && block < b->b.nb, "blocks: bad block");
    const int m = b->b.h_m[block];
    std::vector<double> cm((size_t)m * m);
    FSI_CUDA(cudaMemcpyAsync(cm.data(), b->b.orig.p + b->b.h_lu_off[block], sizeof(double) * m * m,
                             cudaMemcpyDeviceToHost, b->s));
    FSI_CUDA(cudaStreamSynchronize(b->s));
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) rowmajor[(size_t)i * m + j] = cm[(size_t)j * m + i];
  });
}

long long fsigpu_blocks_count(fsigpu_blocks b) { return b ? b->b.nb : 0; }
long long fsigpu_blocks_total_rows(fsigpu_blocks b) { return b ? b->b.total_rows : 0; }
long long fsigpu_blocks_factor_bytes(fsigpu_blocks b) { return b ? 8LL * b->b.h_lu_off[b->b.nb] : 0; }

int fsigpu_blocks_solve_dev(fsigpu_blocks b, const double* d_rhs, double* d_x, void* stream) {
  return guarded([&] {
    require(b != nullptr, "blocks: null");
    cudaStream_t s = stream ? (cudaStream_t)stream : b->s;
    SolveArgs a{};
    a.r = d_rhs;
    a.g1 = INT_MAX;
    a.out = d_x;
    b->b.solve(a, s);
  });
}

int fsigpu_blocks_solve(fsigpu_blocks b, const double* rhs, double* x) {
  return guarded([&] {
    require(b != nullptr, "blocks: null");
    DevBuf<double> dr, dx((size_t)std::max<long long>(b->b.total_rows, 1));
    dr.upload(rhs, (size_t)b->b.total_rows, b->s);
    SolveArgs a{};
    a.r = dr.p;
    a.g1 = INT_MAX;
    a.out = dx.p;
    b->b.solve(a, b->s);
    if (b->b.total_rows)
      FSI_CUDA(cudaMemcpyAsync(x, dx.p, sizeof(double) * b->b.total_rows, cudaMemcpyDeviceToHost, b->s));
    FSI_CUDA(cudaStreamSynchronize(b->s));
  });
}

int fsigpu_blocks_refactor(fsigpu_blocks b, void* stream) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(b != nullptr && b->have_orig, "blocks: no retained matrices");
    cudaStream_t s = stream ? (cudaStream_t)stream : b->s;
    b->b.factor(b->b.orig.p, nullptr, 0, s);
  });
}

int fsigpu_blocks_get_lu(fsigpu_blocks b, double* lu_rowmajor, int* piv) {
  return guarded([&] {
    require(b != nullptr && b->b.keep_lu, "blocks: LU factors not retained for this handle");
    const Blocks& B = b->b;
    auto lu = B.lu.download(b->s);
    auto pv = B.piv.download(b->s);
    for (long long k = 0; k < B.nb; ++k) {
      const int m = B.h_m[k];
      const double* src = lu.data() + B.h_lu_off[k];
      double* dst = lu_rowmajor + B.h_lu_off[k];
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) dst[(size_t)i * m + j] = src[(size_t)j * m + i];
    }
    std::memcpy(piv, pv.data(), sizeof(int) * pv.size());
  });
}

void fsigpu_blocks_destroy(fsigpu_blocks b) {
  if (!b) return;
  cudaStreamSynchronize(b->s);
  cudaStream_t s = b->own_stream ? b->s : nullptr;
  delete b;
  if (s) cudaStreamDestroy(s);
}

// ---- GMG
int fsigpu_gmg_create(int n_levels, const fsigpu_level_desc* levels, double omega, int pre, int post, char cycle,
                      fsigpu_gmg* out) {
  return fsigpu_gmg_create_ex(n_levels, levels, omega, pre, post, cycle, FSIGPU_SCHWARZ_ADDITIVE, out);
}

int fsigpu_gmg_create_ex(int n_levels, const fsigpu_level_desc* levels, double omega, int pre, int post, char cycle,
                         int schwarz, fsigpu_gmg* out) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(schwarz == FSIGPU_SCHWARZ_ADDITIVE || schwarz == FSIGPU_SCHWARZ_MULTIPLICATIVE,
            "fs: schwarz mode must be 0 (additive) or 1 (multiplicative)");
    require(n_levels >= 1 && levels != nullptr, "gmg: no levels");
    require(pre >= 0 && post >= 0 && !(pre == 0 && post == 0 && n_levels > 1), "gmg: need at least one smoothing sweep");
    require(omega >= 0.0 && omega < 2.0, "richardson: omega outside [0,2)");
    require(cycle == 'v' || cycle == 'w' || cycle == 'f', "gmg: unknown cycle type");
    auto h = std::make_unique<fsigpu_gmg_t>();
    Gmg& g = h->g;
    g.s = new_stream();
    g.omega = omega;
    g.pre = pre;
    g.post = post;
    g.cyc = cycle;
    g.lv.resize(n_levels);
    for (int l = 0; l < n_levels; ++l) build_level(g, l, levels[l], g.s, schwarz == FSIGPU_SCHWARZ_MULTIPLICATIVE);
    build_coarse(g, levels[0], g.s);
    pin_hot_data(g);
    g.tmp_in.alloc(g.size());
    g.tmp_out.alloc(g.size());
    *out = h.release();
  });
}

int fsigpu_gmg_size(fsigpu_gmg g) { return g ? g->g.size() : 0; }

int fsigpu_gmg_apply_dev(fsigpu_gmg g, const double* d_r, double* d_z, void* stream) {
  return guarded([&] {
    require(g != nullptr, "gmg: null");
    require(stream == nullptr || stream == (void*)g->g.s, "gmg: use the handle stream (NULL)");
    std::lock_guard<std::mutex> lk(g->g.mu);
    g->g.apply(d_r, d_z);
    if (g_prof.on) g_prof.flush();
  });
}

int fsigpu_gmg_apply(fsigpu_gmg g, const double* r, double* z) {
  return guarded([&] {
    require(g != nullptr, "gmg: null");
    Gmg& G = g->g;
    std::lock_guard<std::mutex> lk(G.mu);
    const int n = G.size();
    FSI_CUDA(cudaMemcpyAsync(G.tmp_in.p, r, sizeof(double) * n, cudaMemcpyHostToDevice, G.s));
    G.apply(G.tmp_in.p, G.tmp_out.p);
    FSI_CUDA(cudaMemcpyAsync(z, G.tmp_out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, G.s));
    FSI_CUDA(cudaStreamSynchronize(G.s));
    if (g_prof.on) g_prof.flush();
  });
}

int fsigpu_fs_apply(fsigpu_gmg g, int level, const double* r, double* z) {
  return guarded([&] {
    require(g != nullptr, "gmg: null");
    Gmg& G = g->g;
    require(level >= 1 && level < (int)G.lv.size(), "fs: level must be a smoothed level (>= 1)");
    std::lock_guard<std::mutex> lk(G.mu);
    Level& L = G.lv[level];
    DevBuf<double> dr, dz(L.n);
    dr.upload(r, (size_t)L.n, G.s);
    G.fs_into(level, dr.p, dz.p);  // z = M r (the smoother applied once, no damping)
    FSI_CUDA(cudaMemcpyAsync(z, dz.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, G.s));
    FSI_CUDA(cudaStreamSynchronize(G.s));
  });
}

int fsigpu_coarse_solve(fsigpu_gmg g, const double* b, double* x) {
  return guarded([&] {
    require(g != nullptr, "gmg: null");
    Gmg& G = g->g;
    std::lock_guard<std::mutex> lk(G.mu);
    Level& L = G.lv[0];
    DevBuf<double> db, dx(L.n);
    db.upload(b, (size_t)L.n, G.s);
    G.coarse_gemv(db.p, dx.p, 0, nullptr);
    FSI_CUDA(cudaMemcpyAsync(x, dx.p, sizeof(double) * L.n, cudaMemcpyDeviceToHost, G.s));
    FSI_CUDA(cudaStreamSynchronize(G.s));
  });
}

// Average device time of one launch of a V-cycle kernel on `level`, each
// launch timed alone with CUDA events on the hierarchy stream after an L2
// flush (cold, HBM-bound) or back to back (warm). Algorithmic bytes of one
// launch are returned alongside.
//   which: 0 FS smoother SpMV (x += omega FS r), 1 level SpMV residual,
//          2 prolongation (+ fused residual), 3 restriction, 4 coarse GEMV
int fsigpu_gmg_time_kernel(fsigpu_gmg h, int which, int level, int reps, int cold, double* ms, double* bytes) {
  return guarded([&] {
    require(h != nullptr && reps > 0, "time: bad args");
    Gmg& G = h->g;
    std::lock_guard<std::mutex> lk(G.mu);
    require(level >= 0 && level < (int)G.lv.size(), "time: bad level");
    Level& L = G.lv[level];
    cudaStream_t s = G.s;
    DevBuf<char> flush(cold ? (size_t)256 << 20 : 0);
    DevBuf<double> v1(L.n), v2(L.n), v3(L.n);
    v1.zero(s);
    v2.zero(s);
    v3.zero(s);
    double* sb = L.b;
    double* sx = L.x;
    L.b = v1.p;
    L.x = v2.p;
    double by = 0.0;
    auto launch = [&]() {
      switch (which) {
        case 0:
          require(L.assembled, "time: level has no assembled FS operator");
          L.FS.launch(GatherPlain{v3.p}, EpiAxpy{G.omega, L.x}, s);
          by = L.FS.bytes(false) + 8.0 * L.n;
          break;
        case 1:
          L.A.launch(GatherPlain{L.x}, EpiResid{L.b, v3.p}, s);
          by = L.A.bytes(true);
          break;
        case 2: {
          require(level > 0 && L.AP.rows, "time: no prolongation on this level");
          Level& B = G.lv[level - 1];
          launch_prolong_resid(L, B.x, nullptr, v3.p, v3.p, s);
          by = L.P.bytes(false) + L.AP.bytes(false) + 24.0 * L.n + L.n + L.nc;
          break;
        }
        case 3: {
          require(level > 0, "time: no restriction on level 0");
          Level& B = G.lv[level - 1];
          DevBuf<double> rc;  // reuse v1 prefix as coarse output
          L.R.launch(GatherPlain{L.x}, EpiRestrict{B.rmask.p, v1.p}, s);
          by = L.R.bytes(false) + L.nc;
          break;
        }
        case 4:
          require(level == 0, "time: coarse GEMV lives on level 0");
          gemv_kernel<kGemvThreads, 8><<<L.n, kGemvThreads, 0, s>>>(L.n, G.coarse_inv.p, L.b, L.x, 0, nullptr, nullptr);
          by = 8.0 * L.n * L.n + 16.0 * L.n;
          break;
        default:
          throw Error(FSIGPU_ERR_INVALID, "time: unknown kernel");
      }
      FSI_CHECK_LAUNCH();
    };
    for (int i = 0; i < 3; ++i) launch();
    cudaEvent_t e0, e1;
    FSI_CUDA(cudaEventCreate(&e0));
    FSI_CUDA(cudaEventCreate(&e1));
    double tot = 0.0;
    if (cold) {
      for (int i = 0; i < reps; ++i) {
        FSI_CUDA(cudaMemsetAsync(flush.p, i & 0xff, flush.n, s));
        FSI_CUDA(cudaEventRecord(e0, s));
        launch();
        FSI_CUDA(cudaEventRecord(e1, s));
        FSI_CUDA(cudaEventSynchronize(e1));
        float t = 0;
        FSI_CUDA(cudaEventElapsedTime(&t, e0, e1));
        tot += t;
      }
    } else {
      FSI_CUDA(cudaEventRecord(e0, s));
      for (int i = 0; i < reps; ++i) launch();
      FSI_CUDA(cudaEventRecord(e1, s));
      FSI_CUDA(cudaEventSynchronize(e1));
      float t = 0;
      FSI_CUDA(cudaEventElapsedTime(&t, e0, e1));
      tot = t;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    L.b = sb;
    L.x = sx;
    *ms = tot / reps;
    *bytes = by;
  });
}

void fsigpu_gmg_destroy(fsigpu_gmg g) {
  if (!g) return;
  cudaStreamSynchronize(g->g.s);
  cudaStream_t s = g->g.s;
  delete g;
  cudaStreamDestroy(s);
}

// ---- GMRES
int fsigpu_gmres_create(fsigpu_gmg g, const double* frame_scale, int restart, fsigpu_gmres* out) {
  return guarded([&] {
    require(g != nullptr && frame_scale != nullptr, "gmres: null args");
    require(restart >= 1 && restart <= kMaxRestart, "gmres: restart must be in [1, 128]");
    auto h = std::make_unique<fsigpu_gmres_t>();
    Gmres& k = h->k;
    k.g = &g->g;
    k.n = g->g.size();
    k.mr = restart;
    const int n = k.n;
    cudaStream_t s = g->g.s;
    k.scale.upload(frame_scale, (size_t)n, s);
    k.V.alloc((size_t)(restart + 1) * n);
    k.Z.alloc((size_t)restart * n);
    k.w.alloc(n);
    k.zbuf.alloc(n);
    k.ubuf.alloc(n);
    k.r.alloc(n);
    k.x.alloc(n);
    k.b.alloc(n);
    k.H.alloc((size_t)(restart + 1) * restart);
    k.H.zero(s);
    k.cs.alloc(restart);
    k.sn.alloc(restart);
    k.gv.alloc(restart + 1);
    k.grid = std::max(1, std::min(ceil_div(n, kKThreads), 2 * 148));
    k.partial.alloc((size_t)std::max(std::max(k.grid, ceil_div(n, kFuseRows)), 4 * 148) * kPartLd);
    k.partial2.alloc((size_t)(n > 8 * 148 * kFuseRows ? 16 : 4) * 148 * kPartLd);  // (B) grid <= 16 (big) / 4 CTAs per SM
    k.ticket.alloc(1);
    k.ticket.zero(s);
    k.st.alloc(1);
    KBufs& kb = k.kb;
    kb.n = n;
    kb.mr = restart;
    kb.scale = k.scale.p;
    kb.V = k.V.p;
    kb.Z = k.Z.p;
    kb.w = k.w.p;
    kb.zbuf = k.zbuf.p;
    kb.ubuf = k.ubuf.p;
    kb.r = k.r.p;
    kb.x = k.x.p;
    kb.b = k.b.p;
    kb.H = k.H.p;
    kb.cs = k.cs.p;
    kb.sn = k.sn.p;
    kb.g = k.gv.p;
    kb.partial = k.partial.p;
    kb.partial2 = k.partial2.p;
    if (restart > kRegRestart) {
      // wide path: one wave of 256-thread CTAs (<= 2 per SM)
      kb.parts_w = std::max(1, std::min(ceil_div(n, kWideThreads), 2 * 148));
      k.partialw.alloc((size_t)ceil_div(restart, kRegRestart) * kb.parts_w * kPartLd);
      kb.partialw = k.partialw.p;
    }
    {
      // resident CTAs of k_spmv_dots (1024 threads): the tile loop's grid
      int dev = 0, sms = 0, occ = 0;
      FSI_CUDA(cudaGetDevice(&dev));
      FSI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      FSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_dots<8>, kFuseThreads, 0));
      // small systems keep one 128-row tile per CTA (config 0: 157 tiles);
      // large ones run (A) as SpMV + k_dots_copy
      const int tiles = ceil_div(n, kFuseRows);
      kb.fuse_small = tiles > 8 * sms || force_big();
      if (kb.fuse_small) {
        kb.parts_a = sms * 4;  // grid of k_dots_copy (rows grid-stride): the partial rows (B) sums
      } else {
        kb.parts_a = tiles <= 8 * sms ? tiles : sms * std::max(occ, 1);
      }
    }
    {
      // (B)/(C) grid: one wave of resident CTAs of (B), at most 4 per SM
      int dev = 0, sms = 0, occ = 0;
      FSI_CUDA(cudaGetDevice(&dev));
      FSI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const bool big = ceil_div(n, kFuseRows) > 8 * sms || force_big();
      if (big) {
        FSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_dots_norm_mr, kArnThreads, 0));
        kb.parts_b = std::max(1, std::min(ceil_div(n, kArnThreads), sms * std::min(std::max(occ, 1), 16)));
        // (C): its own grid at its resident CTA count (168 registers with the
        // multi-row loop of normalize_rows)
        int occ_c = 0;
        FSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, k_update_normalize<false>, kArnThreads, 0));
        kb.parts_c = std::max(1, std::min(ceil_div(n, kArnThreads), sms * std::max(occ_c, 1) - 1));
      } else {
        FSI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_dots_norm<true>, kArnThreads, 0));
        kb.parts_b = std::max(1, std::min(ceil_div(n, kArnThreads), sms * std::min(std::max(occ, 1), 4)));
        kb.parts_c = kb.parts_b;
      }
    }
    kb.ticket = k.ticket.p;
    kb.st = k.st.p;
    {
      Level& T = g->g.lv.back();
      kb.a_ptr = T.A.ptr.p;
      kb.a_idx = T.A.idx.p;
      kb.a_val = T.A.val.p;
      kb.a_lpr = T.A.lpr;
      kb.use_cond = 0;
    }
    k.ensure_history(2000);
    FSI_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int fsigpu_gmres_set_graphs(fsigpu_gmres s, int enable) {
  return guarded([&] {
    require(s != nullptr, "gmres: null");
    s->k.graphs = enable != 0;
  });
}

int fsigpu_gmres_solve_dev(fsigpu_gmres s, const double* d_b, double* d_x, int max_iters, double rel_tol,
                           double abs_tol, double* history, fsigpu_gmres_result* res) {
  return guarded([&] {
    require(s != nullptr && d_b != nullptr && d_x != nullptr, "gmres: null args");
    Gmres& k = s->k;
    std::lock_guard<std::mutex> lk(k.g->mu);
    cudaStream_t st = k.g->s;
    const size_t nb = sizeof(double) * k.n;
    FSI_CUDA(cudaMemcpyAsync(k.b.p, d_b, nb, cudaMemcpyDeviceToDevice, st));
    FSI_CUDA(cudaMemcpyAsync(k.x.p, d_x, nb, cudaMemcpyDeviceToDevice, st));
    fsigpu_gmres_result r{};
    k.solve(max_iters, rel_tol, abs_tol, res ? res : &r);
    FSI_CUDA(cudaMemcpyAsync(d_x, k.x.p, nb, cudaMemcpyDeviceToDevice, st));
    if (history) {
      const int nh = (res ? res : &r)->n_history;
      FSI_CUDA(cudaMemcpyAsync(history, k.hist.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
    }
    FSI_CUDA(cudaStreamSynchronize(st));
  });
}

int fsigpu_gmres_solve(fsigpu_gmres s, const double* b, const double* x0, double* x, int max_iters, double rel_tol,
                       double abs_tol, double* history, fsigpu_gmres_result* res) {
  return guarded([&] {
    require(s != nullptr && b != nullptr && x != nullptr, "gmres: null args");
    Gmres& k = s->k;
    std::lock_guard<std::mutex> lk(k.g->mu);
    cudaStream_t st = k.g->s;
    const size_t nb = sizeof(double) * k.n;
    FSI_CUDA(cudaMemcpyAsync(k.b.p, b, nb, cudaMemcpyHostToDevice, st));
    if (x0)
      FSI_CUDA(cudaMemcpyAsync(k.x.p, x0, nb, cudaMemcpyHostToDevice, st));
    else
      FSI_CUDA(cudaMemsetAsync(k.x.p, 0, nb, st));
    fsigpu_gmres_result r{};
    k.solve(max_iters, rel_tol, abs_tol, res ? res : &r);
    FSI_CUDA(cudaMemcpyAsync(x, k.x.p, nb, cudaMemcpyDeviceToHost, st));
    if (history) {
      const int nh = (res ? res : &r)->n_history;
      FSI_CUDA(cudaMemcpyAsync(history, k.hist.p, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
    }
    FSI_CUDA(cudaStreamSynchronize(st));
  });
}

void fsigpu_gmres_destroy(fsigpu_gmres s) {
  if (!s) return;
  // the solver must not touch its hierarchy here: a garbage collector may
  // destroy the hierarchy first (its stream then no longer exists)
  cudaDeviceSynchronize();
  delete s;
}

// ---- block sets built on the device (sets.cuh)
int fsigpu_fs_sets_build(const fsigpu_level_desc* lv, const fsigpu_mesh_desc* mesh, int epb_as1, int epb_as2,
                         int overlap_layers, fsigpu_sets* out) {
  g_bad_block = -1;
  g_bad_level = -1;
  return guarded([&] {
    require(lv != nullptr && mesh != nullptr && out != nullptr, "sets: null args");
    require(epb_as1 >= 1 && epb_as2 >= 1 && overlap_layers >= 0, "fieldsplit: elems_per_block must be >= 1");
    const fsigpu_level_desc& d = *lv;
    require(d.n > 0 && d.a_ptr && d.a_idx && d.a_val, "sets: level matrix missing");
    require(d.g1 >= 0 && d.n_us >= 0 && d.g1 + d.n_us <= d.n, "fs: bad group sizes");
    cudaStream_t s = new_stream();
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    auto h = std::make_unique<fsigpu_sets_t>();
    SetBuilder B(*mesh, d.n, s);
    Csr A;
    A.create(d.n, d.n, d.a_ptr, d.a_idx, d.a_val, s);
    B.g1e.alloc((size_t)std::max(d.g1, 1));
    if (d.g1) {
      g1_empty_kernel<<<ceil_div(d.g1, 256), 256, 0, s>>>(d.g1, A.ptr.p, A.idx.p, A.val.p, B.g1e.p);
      FSI_CHECK_LAUNCH();
    }
    // AS1: solid [d^s, p^s] chunks, then overlapping fluid d^f chunks
    B.run(kSetSolidDp, B.solid, B.d_solid, epb_as1, 0, d.g1, h->as1_ptr, h->as1_idx);
    for (size_t st = 0; st < B.solid.size(); st += epb_as1) h->labels.push_back("fs-solid-dp-" + std::to_string(st));
    B.run(kSetFluidD, B.fluid, B.d_fluid, epb_as1, overlap_layers, d.g1, h->as1_ptr, h->as1_idx);
    for (size_t st = 0; st < B.fluid.size(); st += epb_as1) h->labels.push_back("fs-fluid-d-" + std::to_string(st));
    // AS2: fluid [u^f, p^f] chunks, group-2 local positions
    B.run(kSetFluidUp, B.fluid, B.d_fluid, epb_as2, 0, d.g1, h->as2_ptr, h->as2_idx);
    for (size_t st = 0; st < B.fluid.size(); st += epb_as2) h->labels.push_back("fs-fluid-up-" + std::to_string(st));
    // lumped u^s mass
    h->lumped.assign(d.n_us, 1.0);
    if (d.n_us) {
      DevBuf<double> lm(d.n_us);
      DevBuf<int> bad(1);
      const int big = INT_MAX;
      FSI_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
      lumped_kernel<<<ceil_div(d.n_us, 256), 256, 0, s>>>(d.g1, d.n_us, A.ptr.p, A.idx.p, A.val.p, lm.p, bad.p);
      FSI_CHECK_LAUNCH();
      h->lumped = lm.download(s);
      const int b = bad.download(s)[0];
      if (b != INT_MAX) throw Error(FSIGPU_ERR_SINGULAR, "singular block: fs lumped mass row " + std::to_string(b));
    }
    FSI_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int fsigpu_vanka_sets_build(int n, const fsigpu_mesh_desc* mesh, int epb, fsigpu_sets* out) {
  return guarded([&] {
    require(mesh != nullptr && out != nullptr && n > 0, "sets: null args");
    require(epb >= 1, "vanka: elems_per_block must be >= 1");
    cudaStream_t s = new_stream();
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    auto h = std::make_unique<fsigpu_sets_t>();
    SetBuilder B(*mesh, n, s);
    B.run(kSetVankaSolid, B.solid, B.d_solid, epb, 0, n, h->as1_ptr, h->as1_idx);
    int k = 0;
    for (size_t st = 0; st < B.solid.size(); st += epb) h->labels.push_back("vanka-solid-" + std::to_string(k++));
    B.run(kSetVankaFluid, B.fluid, B.d_fluid, epb, 0, n, h->as1_ptr, h->as1_idx);
    for (size_t st = 0; st < B.fluid.size(); st += epb) h->labels.push_back("vanka-fluid-" + std::to_string(k++));
    FSI_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int fsigpu_sets_counts(fsigpu_sets h, int* as1_n, int* as1_len, int* as2_n, int* as2_len, int* n_us) {
  return guarded([&] {
    require(h != nullptr, "sets: null");
    if (as1_n) *as1_n = (int)h->as1_ptr.size() - 1;
    if (as1_len) *as1_len = (int)h->as1_idx.size();
    if (as2_n) *as2_n = (int)h->as2_ptr.size() - 1;
    if (as2_len) *as2_len = (int)h->as2_idx.size();
    if (n_us) *n_us = (int)h->lumped.size();
  });
}

int fsigpu_sets_copy(fsigpu_sets h, int* as1_ptr, int* as1_idx, int* as2_ptr, int* as2_idx, double* lumped) {
  return guarded([&] {
    require(h != nullptr, "sets: null");
    auto cp = [](const auto& v, auto* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(h->as1_ptr, as1_ptr);
    cp(h->as1_idx, as1_idx);
    cp(h->as2_ptr, as2_ptr);
    cp(h->as2_idx, as2_idx);
    cp(h->lumped, lumped);
  });
}

const char* fsigpu_sets_label(fsigpu_sets h, int block) {
  if (!h || block < 0 || block >= (int)h->labels.size()) return "";
  return h->labels[block].c_str();
}

void fsigpu_sets_destroy(fsigpu_sets h) { delete h; }

// ---- profiler
int fsigpu_profile_enable(int enable) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.on = enable != 0;
  });
}
int fsigpu_profile_read(double* ms, long long* launches, double* bytes) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.flush();
    for (int i = 0; i < FSIGPU_K_COUNT; ++i) {
      if (ms) ms[i] = g_prof.ms[i];
      if (launches) launches[i] = g_prof.launches[i];
      if (bytes) bytes[i] = g_prof.bytes[i];
    }
  });
}
int fsigpu_profile_read_level(int cls, int level, double* ms, long long* launches, double* bytes) {
  return guarded([&] {
    require(cls >= 0 && cls < FSIGPU_K_COUNT, "profile: bad class");
    require(level >= -1 && level < Profiler::kLv, "profile: bad level");
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.flush();
    if (ms) *ms = g_prof.lv_ms[cls][level + 1];
    if (launches) *launches = g_prof.lv_launches[cls][level + 1];
    if (bytes) *bytes = g_prof.lv_bytes[cls][level + 1];
  });
}
int fsigpu_profile_reset(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.flush();
    for (int i = 0; i < FSIGPU_K_COUNT; ++i) {
      g_prof.ms[i] = 0;
      g_prof.launches[i] = 0;
      g_prof.bytes[i] = 0;
      for (int l = 0; l <= Profiler::kLv; ++l) {
        g_prof.lv_ms[i][l] = 0;
        g_prof.lv_launches[i][l] = 0;
        g_prof.lv_bytes[i][l] = 0;
      }
    }
  });
}

// Device-clock launch stamps: durations of the solve kernels inside the
// captured graphs (see common.cuh stamp_*). Enabling or disabling makes
// every solver re-capture its graph on the next solve.
int fsigpu_stamps_enable(int enable) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (enable && !g_stamp_buf) FSI_CUDA(cudaMalloc(&g_stamp_buf, stamp_slots() * 4 * sizeof(unsigned long long)));
    if (g_stamp_buf) FSI_CUDA(cudaMemset(g_stamp_buf, 0, stamp_slots() * 4 * sizeof(unsigned long long)));
    g_stamp_on = enable != 0;
    ++g_stamp_epoch;
  });
}
int fsigpu_stamps_read(int cls, int level, int sub, double* us_total, long long* launches) {
  return guarded([&] {
    require(cls >= 0 && cls < FSIGPU_K_COUNT, "stamps: bad class");
    require(level >= -1 && level < Profiler::kLv, "stamps: bad level");
    require(sub >= 0 && sub < kStampSubs, "stamps: bad kernel index");
    require(g_stamp_buf != nullptr, "stamps: not enabled");
    FSI_CUDA(cudaDeviceSynchronize());
    unsigned long long h[4];
    const size_t slot = ((size_t)cls * (Profiler::kLv + 1) + level + 1) * kStampSubs + sub;
    FSI_CUDA(cudaMemcpy(h, g_stamp_buf + 4 * slot, sizeof(h), cudaMemcpyDeviceToHost));
    unsigned long long ns = h[2], cnt = h[3];
    if (h[0] && h[1] > h[0]) {  // the last launch has not been folded yet
      ns += h[1] - h[0];
      cnt += 1;
    }
    if (us_total) *us_total = (double)ns / 1000.0;
    if (launches) *launches = (long long)cnt;
  });
}

}  // extern "C"
