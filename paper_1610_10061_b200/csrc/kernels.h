// Host-side declarations of the kernel launchers (internal to libpmedian_b200).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>

namespace pmb {

enum class KeyKind { kPacked32, kPacked64, kPayload64 };

// K1 launch plan, chosen by the host from the validated instance.
struct BuildPlan {
  int n = 0, m = 0, p = 0, W = 0, Wp = 0;
  int mP = 0;  // row stride of the u16 cost copy (round_up(m, 8))
  int site_bytes = 4, dist_bytes = 8;
  int sitebits = 0, costbits = 0, npasses = 0;
  KeyKind key_kind = KeyKind::kPacked64;
  bool smem_path = true;
  int grid = 0;
  // counting-sort path (k_build_rows_cs): packed u32 keys, u16 sites, costs < 2^15
  bool cs_path = false;
  int cs_bits = 0, cs_grid = 0;
};

size_t cs_smem(int m, int costbits);

size_t sort_smem_header();
cudaError_t launch_validate_costs(const int64_t* costs, size_t count, unsigned long long* out_max,
                              int* out_neg, int sms, cudaStream_t st);
// rows: device int[1 + n] (count, then the rows the counting-sort path hands
// to the radix kernel); used only when bp.cs_path
// c16: the u16 copy of the matrix (row stride bp.mP) when every cost fits 16
// bits and the tables are u16, else nullptr (rows come from the int64 matrix)
cudaError_t launch_build_rows(const BuildPlan& bp, const int64_t* costs, const uint16_t* c16, void* ord, void* dist,
                              void* scratch_keys, uint32_t* scratch_pay, int* rows, cudaStream_t st);
// One pass over the int64 matrix: max cost / negativity into out_max / out_neg
// (zeroed by the caller) and the speculative u16 copies c16 (n x mP) and dT (m x nP).
cudaError_t launch_prep_costs(const int64_t* costs, int n, int m, int mP, int nP, uint16_t* c16, uint16_t* dT,
                              unsigned long long* out_max, int* out_neg, int sms, cudaStream_t st);
cudaError_t launch_transpose_costs(const int64_t* costs, int n, int nP, int m, int dist_bytes, void* dT,
                                   cudaStream_t st);

// Device-resident tables as the evaluation kernels see them.
struct DevTables {
  int n = 0, m = 0, p = 0, W = 0, Wp = 0;
  int site_bytes = 2, dist_bytes = 2;
  int64_t max_cost = 0;
  const void* ord = nullptr;   // n x Wp, OrdT
  const void* dist = nullptr;  // n x Wp, DistT (sorted costs)
  const void* dT = nullptr;    // m x nP, DistT (site-major costs, gather kernel)
  int nP = 0;                  // dT row stride: round_up(n, 16)
};

// K2t: population words -> per-group transposed site masks T[g][s] (64 chromosomes / group).
size_t scan_t_stride(int m);  // u64 entries per group (>= m + 1, even)
// also zeroes costs[0, count) (the scan accumulates into it)
// err_init (nullable): an error word the launch sets to ~0 (no failure) first
cudaError_t launch_transpose_population(const uint64_t* words, size_t count, int words_per, int m,
                                        uint64_t* T, unsigned long long* costs, unsigned long long* err_init,
                                        cudaStream_t st);

// K2: bit-sliced scan.  costs_acc (count u64) must be zeroed; err_first_bad
// (u64) must hold ~0 before the launch.
struct ScanPlan {
  int warps = 8;
  int ctas = 0;
  bool acc32 = true;
  bool tsmem = true;  // masks staged in shared memory (else read from global)
  int G = 64;         // chromosomes per group (64 or 32)
  size_t smem = 0;
  int wide = 0;       // 1: the many-warp variant (kWideWarps per CTA, kWideQueue records, 2 row chunks)
  bool pair = false;  // the 24-warp variant appends column pairs (long walks)
  int coop = 0;       // cooperative tail: clients per warp at which it starts | log2(max lanes per client) << 8
  int tail_claim = 0; // clients left in a segment below which a warp claims only what its lanes need
};
ScanPlan plan_scan(const DevTables& t, size_t count, int sms, size_t max_smem, bool depth_mode);
// depth_mode != 0 accumulates the 1-based stopping columns k* instead of costs.
cudaError_t launch_scan(const DevTables& t, const ScanPlan& sp, const uint64_t* T, size_t count,
                        unsigned long long* costs_acc, unsigned long long* err_first_bad,
                        int depth_mode, cudaStream_t st);

// Measurement (not an evaluation path): per 32-chromosome group the sum over
// clients of the walk length max_{c in group} k*_ic, and per client the
// maximum over groups.  group_sum (ceil(count/32) u64) and client_max (n u32)
// must be zeroed.  T from launch_transpose_population.
cudaError_t launch_walks(const DevTables& t, const uint64_t* T, size_t count, unsigned long long* group_sum,
                         unsigned int* client_max, cudaStream_t st);

// K2b prep: per-chromosome open-site lists (cap entries) and popcounts.
// also zeroes costs[0, count) (the gather accumulates into it)
cudaError_t launch_open_lists(const uint64_t* words, size_t count, int words_per, int m,
                              uint32_t* open_lists, uint32_t* open_counts, int open_cap,
                              unsigned long long* costs, unsigned long long* err_init, cudaStream_t st);
// K2b fused (m <= 65535): one launch per evaluation, lists built in shared
// memory, costs stored (no zeroing needed).  Work items are (chromosome, client
// slab); with several slabs (gather_fused_slabs > 1) `partial` holds count x
// slabs sums and `arrive` count counters kept at 0 between calls.  err_work /
// done: a context word kept at ~0 and an arrival counter kept at 0 between
// calls; the last CTA writes the call's error into err_out (err_store: a store,
// else a min into a sticky word) and re-arms them.
bool gather_fused_fits(const DevTables& t);
int gather_fused_slabs(const DevTables& t);
cudaError_t launch_gather_fused(const DevTables& t, const uint64_t* words, size_t count, int words_per,
                                unsigned long long* costs, unsigned long long* partial, unsigned int* arrive,
                                unsigned long long* err_work, unsigned int* done, unsigned long long* err_out,
                                int err_store, int mode, int sms, cudaStream_t st);
// K2b: gather-min (needs launch_open_lists first).  mode 0 = fitness semantics (scan-width contract), 1 = min_cost_sum.
cudaError_t launch_gather(const DevTables& t, const uint64_t* words, size_t count, int words_per,
                          uint32_t* open_lists, uint32_t* open_counts, int open_cap,
                          unsigned long long* costs_acc, unsigned long long* err_first_bad, int mode,
                          int sms, cudaStream_t st);

}  // namespace pmb
