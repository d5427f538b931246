// Internal: the pm_ctx layout shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/pmedian_b200.h"
#include "kernels.h"

namespace pmb {

// Reference message texts (errors thrown by the code each status replaces).
inline constexpr int kErrSlots = 8;  // error words: [0] the context's, [1..] pipelined chunks
inline constexpr const char* kMsgLength = "chromosome length must equal the site count";  // ordering.cpp:42
inline constexpr const char* kMsgRunoff =
    "no open site within the scan width; exactly p sites must be open";  // ordering.cpp:51
inline constexpr const char* kMsgNoneOpen = "at least one site must be open";  // instance.cpp:37

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace pmb

using pmb::DevBuf;
using pmb::DevTables;
using pmb::BuildPlan;

namespace pmb {
// Pinned host staging (grow-only): one transfer per generation for the
// block-best records and for migration.
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// GA working set (ga.cu), grow-only and kept across calls.  brec holds one
// record {cost, thread, words[wp]} per block (k_block_min).
struct GaBuffers {
  DevBuf pop, next, cost, before, child, ccost, ok, brec, evals, tmp, table, ranks, rflags, rstate;
  DevBuf lfact;  // ln x! for x <= m + 1 (double): the unranking's search guide
  size_t tab_m = 0, tab_p = 0, tab_L = 0;  // what `table` / `lfact` hold (0: nothing)
  // run_ga's device-resident generation state: grec = every island's block
  // records after the exchange, gstate = {best cost, kernel of best, stale,
  // kernels, stop, best words[wp]}, perk = per-kernel bests (grown on demand)
  DevBuf grec, gstate, perk;
  size_t perk_cap = 0;
  HostBuf hrec, hglob, hflag;  // pinned: host-callback exchange staging, the stop word
};
}  // namespace pmb
using pmb::GaBuffers;

struct pm_ctx {
  int device = 0;
  int sms = 148;
  size_t max_smem = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;
  int eval_kind = PM_EVAL_AUTO;

  bool has_instance = false;
  DevTables t;
  BuildPlan plan;
  DevBuf ord, dist, dT;

  // scratch
  DevBuf costs_in, sort_keys, sort_pay, sort_rows, words, costs_out, T, lists, counts, errw, scal;
  DevBuf c16, dT16;  // set_instance scratch: the u16 cost copies of the fused prep pass
  DevBuf gsync;      // fused gather: error word (kept at ~0) + arrival counter (kept at 0)
  DevBuf gpart, garr;  // fused gather over client slabs: partial sums, per-chromosome counters (kept at 0)
  pmb::HostBuf hout;  // host-buffer calls: costs + error words come back in one pinned copy
  int open_cap = 0;
  GaBuffers ga;
  cudaStream_t copy_stream = nullptr;  // H2D of pipelined host-buffer calls
  cudaStream_t draw_stream = nullptr;  // the GA's next-population draw, overlapped with evolution
  cudaEvent_t draw_ev = nullptr;
  cudaEvent_t entry_ev = nullptr;  // host-buffer calls: copies start after the stream's earlier work
  std::vector<cudaEvent_t> chunk_ev;
  std::vector<int64_t> per_kernel_best;  // RunResult::per_kernel_best_costs of the last run_ga

  // kernel timing hook: events around the dominant evaluation kernel
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
  std::pair<cudaEvent_t, cudaEvent_t> ev_get() {
    if (!ev_free.empty()) {
      auto e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    std::pair<cudaEvent_t, cudaEvent_t> e{nullptr, nullptr};
    cudaEventCreate(&e.first);
    cudaEventCreate(&e.second);
    return e;
  }

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* where) {
    err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return PM_CUDA;
  }
};

#define PM_CUDA_TRY(ctx, expr)                                 \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return (ctx)->cuda_fail(_e, #expr); \
  } while (0)

namespace pmb {
// Fitness of `count` device-resident chromosomes into device costs (mode 0:
// fitness, 1: min_cost_sum, 2: scan depths).  Asynchronous on ctx->stream.
// errw: device word receiving the lowest failing index (nullptr: the context's).
int evaluate_core(pm_ctx* c, const uint64_t* dwords, size_t count, int64_t* dcosts, int mode,
                  unsigned long long* errw = nullptr);
}  // namespace pmb
