// C-ABI implementation (include/pmedian_b200.h): context, instance upload,
// K1 orchestration and the K2/K2b dispatch.  Host-side C++; no CPU compute
// path exists -- every cost is produced by a kernel.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pmedian_b200.h"
#include "kernels.h"
#include "ctx.h"

using namespace pmb;

extern "C" {

int pm_warmup(int device) {
  // load every kernel of the module with the context instead of at its first
  // launch (lazy loading costs milliseconds per kernel inside the first timed
  // call); only effective when this is the process's first CUDA call, and a
  // caller's own CUDA_MODULE_LOADING wins
  setenv("CUDA_MODULE_LOADING", "EAGER", 0);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return PM_CUDA;
  if (device < 0 || device >= ndev) return PM_DOMAIN;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return PM_CUDA;
  return PM_OK;
}

int pm_create(int device, pm_ctx** out) {
  if (!out) return PM_STRUCTURAL;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return PM_CUDA;
  if (device < 0 || device >= ndev) return PM_DOMAIN;
  if (cudaSetDevice(device) != cudaSuccess) return PM_CUDA;
  pm_ctx* c = new pm_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->max_smem = (size_t)optin;
  // the context's stream at the highest priority: the GA's population draw
  // for the next generation (draw_stream, default priority) fills the SMs the
  // evolution leaves idle instead of delaying it
  int prio_least = 0, prio_greatest = 0;
  cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest);
  if (cudaStreamCreateWithPriority(&c->own, cudaStreamNonBlocking, prio_greatest) != cudaSuccess) {
    delete c;
    return PM_CUDA;
  }
  c->stream = c->own;
  if (c->errw.ensure(kErrSlots * 8) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->draw_stream, cudaStreamNonBlocking, prio_least) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->draw_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->entry_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return PM_CUDA;
  }
  cudaMemsetAsync(c->errw.p, 0xff, kErrSlots * 8, c->stream);
  *out = c;
  return PM_OK;
}

void pm_destroy(pm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (DevBuf* b : {&c->ord, &c->dist, &c->dT, &c->costs_in, &c->sort_keys, &c->sort_pay, &c->words,
                    &c->costs_out, &c->T, &c->lists, &c->counts, &c->errw, &c->scal, &c->ga.pop,
                    &c->ga.next, &c->ga.cost, &c->ga.before, &c->ga.child, &c->ga.ccost, &c->ga.ok,
                    &c->ga.brec, &c->ga.evals, &c->ga.tmp, &c->ga.table, &c->ga.ranks, &c->ga.rflags,
                    &c->ga.rstate, &c->ga.lfact, &c->ga.grec, &c->ga.gstate, &c->ga.perk, &c->sort_rows,
                    &c->c16, &c->dT16, &c->gsync, &c->gpart, &c->garr})
    b->release();
  c->ga.hrec.release();
  c->ga.hglob.release();
  c->ga.hflag.release();
  c->hout.release();
  for (auto* v : {&c->ev_used, &c->ev_free})
    for (auto& e : *v) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  for (cudaEvent_t e : c->chunk_ev) cudaEventDestroy(e);
  if (c->draw_stream) {
    cudaStreamSynchronize(c->draw_stream);
    cudaStreamDestroy(c->draw_stream);
  }
  if (c->draw_ev) cudaEventDestroy(c->draw_ev);
  if (c->entry_ev) cudaEventDestroy(c->entry_ev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

const char* pm_last_error(const pm_ctx* c) { return c ? c->err.c_str() : "null context"; }

int pm_set_stream(pm_ctx* c, void* stream) {
  if (!c) return PM_STRUCTURAL;
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
  return PM_OK;
}

uint64_t pm_kernel_launches(const pm_ctx* c) { return c ? c->launches : 0; }

// ---- instance ------------------------------------------------------------------

static int bits_for(uint64_t v) { return v == 0 ? 0 : 64 - __builtin_clzll(v); }

// hcosts: the same matrix in host memory when the caller passed one (small
// matrices are validated there: no kernel, no synchronisation)
static int set_instance_impl(pm_ctx* c, const int64_t* dcosts, size_t n, size_t m, size_t p,
                             const int64_t* hcosts = nullptr) {
  // Instance::Instance checks, in the reference's order (instance.cpp:13-29).
  if (n == 0) return c->fail(PM_STRUCTURAL, "instance needs at least one client");
  if (m == 0) return c->fail(PM_STRUCTURAL, "instance needs at least one site");
  if (p < 1) return c->fail(PM_DOMAIN, "p must be >= 1");
  if (p >= m) return c->fail(PM_DOMAIN, "p must be < m");
  if (n > (size_t)INT_MAX / 2 || m > (size_t)INT_MAX / 2)
    return c->fail(PM_DOMAIN, "device tables support at most 2^30 clients and sites");

  unsigned long long host[2] = {0, 0};  // {max cost, negative seen}
  const size_t nP = (n + 15) / 16 * 16, mP = (m + 7) / 8 * 8;
  // Large matrices: one fused pass validates and writes the u16 copies K1
  // and K2b use (k_prep_costs), kept when every cost fits 16 bits.  Small
  // host matrices are validated on the host (no kernel, no synchronisation).
  bool prep = false;
  if (hcosts && n * m <= ((size_t)1 << 20)) {
    for (size_t x = 0; x < n * m; ++x) {
      host[1] |= hcosts[x] < 0;
      host[0] = std::max<unsigned long long>(host[0], hcosts[x] < 0 ? 0 : (unsigned long long)hcosts[x]);
    }
  } else {
    unsigned long long* scal = nullptr;
    PM_CUDA_TRY(c, c->scal.ensure(16));
    scal = c->scal.as<unsigned long long>();
    PM_CUDA_TRY(c, cudaMemsetAsync(scal, 0, 16, c->stream));
    prep = getenv("PMB_K1_PREP") == nullptr || getenv("PMB_K1_PREP")[0] != '0';
    // grow-only scratch, kept across instances of similar size (allocating
    // and freeing gigabytes per call costs more than the kernels)
    for (DevBuf* b : {&c->c16, &c->dT16})
      if (b->bytes > 4 * (n * std::max(mP, nP) * 2) + (1 << 20)) b->release();
    if (prep && (c->c16.ensure(n * mP * 2) != cudaSuccess || c->dT16.ensure(m * nP * 2) != cudaSuccess)) {
      (void)cudaGetLastError();  // not enough memory for the copies: the three-pass path
      c->c16.release();
      c->dT16.release();
      prep = false;
    }
    if (prep) {
      PM_CUDA_TRY(c, launch_prep_costs(dcosts, (int)n, (int)m, (int)mP, (int)nP, c->c16.as<uint16_t>(),
                                       c->dT16.as<uint16_t>(), scal, reinterpret_cast<int*>(scal + 1), c->sms,
                                       c->stream));
    } else {
      PM_CUDA_TRY(c, launch_validate_costs(dcosts, n * m, scal, reinterpret_cast<int*>(scal + 1), c->sms,
                                           c->stream));
    }
    c->launches += 1;
    PM_CUDA_TRY(c, cudaMemcpyAsync(host, scal, 16, cudaMemcpyDeviceToHost, c->stream));
    PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  if (prep && host[0] > 65535) prep = false;  // the speculative u16 copies do not hold these costs
  if (host[1] & 1) return c->fail(PM_STRUCTURAL, "costs must be non-negative");
  const int64_t max_cost = (int64_t)host[0];
  if (max_cost > 0 && max_cost > INT64_MAX / (int64_t)n)
    return c->fail(PM_STRUCTURAL, "costs too large: n * max(cost) would overflow 64-bit totals");

  BuildPlan bp;
  bp.n = (int)n;
  bp.m = (int)m;
  bp.p = (int)p;
  bp.W = (int)(m - p + 1);
  bp.Wp = (bp.W + 15) / 16 * 16;
  bp.mP = (int)mP;
  bp.site_bytes = m <= 65535 ? 2 : 4;  // sentinel site m must fit
  bp.dist_bytes = max_cost <= 65535 ? 2 : (max_cost <= 0xffffffffLL ? 4 : 8);
  bp.sitebits = std::max(1, bits_for((uint64_t)(m - 1)));
  bp.costbits = bits_for((uint64_t)max_cost);
  bp.npasses = (bp.costbits + 7) / 8;
  if (bp.costbits + bp.sitebits <= 32) bp.key_kind = KeyKind::kPacked32;
  else if (bp.costbits + bp.sitebits <= 64) bp.key_kind = KeyKind::kPacked64;
  else bp.key_kind = KeyKind::kPayload64;
  const size_t keyb = bp.key_kind == KeyKind::kPacked32 ? 4 : 8;
  const size_t payb = bp.key_kind == KeyKind::kPayload64 ? 4 : 0;
  const size_t need = sort_smem_header() + m * (keyb + payb) * 2;
  bp.smem_path = need <= c->max_smem;
  if (bp.smem_path) {
    bp.grid = (int)std::min<size_t>(n, (size_t)c->sms);
  } else {
    bp.grid = (int)std::min<size_t>(n, (size_t)c->sms);
    PM_CUDA_TRY(c, c->sort_keys.ensure((size_t)bp.grid * 2 * m * keyb));
    if (payb) PM_CUDA_TRY(c, c->sort_pay.ensure((size_t)bp.grid * 2 * m * payb));
  }

  // counting-sort path: one pass for small cost ranges; two CTAs per SM when
  // a row's counters + keys fit in half the shared memory (PMB_K1=radix: off)
  {
    const char* k1 = getenv("PMB_K1");
    const int cb = std::max(1, bp.costbits);
    // (per-row work is O(m + 2^costbits): only rows at least half as long as
    // the bucket count pay off -- shorter rows keep the radix kernel)
    if (bp.key_kind == KeyKind::kPacked32 && bp.site_bytes == 2 && cb <= 15 &&
        (m >= ((size_t)1 << cb) / 2 || (k1 && std::string(k1) == "count")) &&
        !(k1 && std::string(k1) == "radix")) {
      const size_t cs = cs_smem(bp.m, cb);
      if (cs <= c->max_smem) {
        bp.cs_path = true;
        bp.cs_bits = cb;
        const int per_sm = 2 * (cs + 2048) <= 228 * 1024 ? 2 : 1;
        bp.cs_grid = (int)std::min<size_t>(n, (size_t)c->sms * per_sm);
        PM_CUDA_TRY(c, c->sort_rows.ensure((n + 1) * sizeof(int)));
      }
    }
  }

  c->has_instance = false;
  const size_t cells = n * (size_t)bp.Wp;
  // tables are regrown only when they do not fit (a pooled context builds the
  // next small instance without allocating); a large previous instance is
  // dropped first so two never coexist
  // (regrown when too small, or dropped when more than 4x the need: a large
  // instance's tables do not linger behind a small one)
  auto fits = [](const DevBuf& b, size_t need) { return b.bytes >= need && b.bytes <= 4 * need + (1 << 20); };
  if (!fits(c->ord, cells * bp.site_bytes) || !fits(c->dist, cells * bp.dist_bytes)) {
    c->ord.release();
    c->dist.release();
  }
  if (!prep && !fits(c->dT, nP * m * (size_t)bp.dist_bytes)) c->dT.release();
  PM_CUDA_TRY(c, c->ord.ensure(cells * bp.site_bytes));
  PM_CUDA_TRY(c, c->dist.ensure(cells * bp.dist_bytes));
  const uint16_t* c16 = prep && bp.dist_bytes == 2 ? c->c16.as<uint16_t>() : nullptr;
  PM_CUDA_TRY(c, launch_build_rows(bp, dcosts, c16, c->ord.p, c->dist.p, c->sort_keys.p,
                                   c->sort_pay.as<uint32_t>(), c->sort_rows.as<int>(), c->stream));
  if (prep) {  // the u16 site-major table is already built: adopt it (the old one becomes scratch)
    std::swap(c->dT, c->dT16);
  } else {
    PM_CUDA_TRY(c, c->dT.ensure(nP * m * (size_t)bp.dist_bytes));
    PM_CUDA_TRY(c, launch_transpose_costs(dcosts, (int)n, (int)nP, (int)m, bp.dist_bytes, c->dT.p, c->stream));
    c->launches += 1;
  }
  c->launches += 1;
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (!bp.smem_path) {
    c->sort_keys.release();
    c->sort_pay.release();
  }

  c->plan = bp;
  DevTables& t = c->t;
  t.n = bp.n;
  t.m = bp.m;
  t.p = bp.p;
  t.W = bp.W;
  t.Wp = bp.Wp;
  t.site_bytes = bp.site_bytes;
  t.dist_bytes = bp.dist_bytes;
  t.max_cost = max_cost;
  t.ord = c->ord.p;
  t.dist = c->dist.p;
  t.dT = c->dT.p;
  t.nP = (int)nP;
  // a multiple of 4: the gather reads the lists 16 bytes at a time
  c->open_cap = (int)((std::min<size_t>(m, std::max<size_t>(p, 16)) + 3) / 4 * 4);
  c->has_instance = true;
  c->err.clear();
  return PM_OK;
}

int pm_set_instance(pm_ctx* c, const int64_t* costs, size_t n, size_t m, size_t p) {
  if (!c) return PM_STRUCTURAL;
  if (!costs && n != 0 && m != 0) return c->fail(PM_STRUCTURAL, "cost matrix must be exactly n rows by m columns");
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  if (n == 0 || m == 0 || p < 1 || p >= m) return set_instance_impl(c, nullptr, n, m, p);
  PM_CUDA_TRY(c, c->costs_in.ensure(n * m * 8));
  PM_CUDA_TRY(c, cudaMemcpyAsync(c->costs_in.p, costs, n * m * 8, cudaMemcpyHostToDevice, c->stream));
  const int rc = set_instance_impl(c, c->costs_in.as<int64_t>(), n, m, p, costs);
  if (c->costs_in.bytes > ((size_t)64 << 20)) c->costs_in.release();  // small staging is kept for the next call
  return rc;
}

int pm_set_instance_device(pm_ctx* c, const int64_t* costs_device, size_t n, size_t m, size_t p) {
  if (!c) return PM_STRUCTURAL;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  return set_instance_impl(c, costs_device, n, m, p);
}

int pm_table_info_get(pm_ctx* c, pm_table_info* out) {
  if (!c || !out) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  out->clients = c->t.n;
  out->sites = c->t.m;
  out->open_count = c->t.p;
  out->width = c->t.W;
  out->row_stride = c->t.Wp;
  out->site_bytes = c->t.site_bytes;
  out->dist_bytes = c->t.dist_bytes;
  out->max_cost = c->t.max_cost;
  return PM_OK;
}

int pm_get_tables(pm_ctx* c, uint32_t* site_order, int64_t* increments) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  const DevTables& t = c->t;
  const size_t cells = (size_t)t.n * t.Wp;
  std::vector<unsigned char> o(cells * t.site_bytes), d(cells * t.dist_bytes);
  PM_CUDA_TRY(c, cudaMemcpyAsync(o.data(), t.ord, o.size(), cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaMemcpyAsync(d.data(), t.dist, d.size(), cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int i = 0; i < t.n; ++i) {
    int64_t prev = 0;
    for (int k = 0; k < t.W; ++k) {
      const size_t x = (size_t)i * t.Wp + k;
      const uint32_t s = t.site_bytes == 2 ? reinterpret_cast<uint16_t*>(o.data())[x]
                                           : reinterpret_cast<uint32_t*>(o.data())[x];
      int64_t v;
      if (t.dist_bytes == 2) v = reinterpret_cast<uint16_t*>(d.data())[x];
      else if (t.dist_bytes == 4) v = reinterpret_cast<uint32_t*>(d.data())[x];
      else v = reinterpret_cast<int64_t*>(d.data())[x];
      site_order[(size_t)i * t.W + k] = s;
      increments[(size_t)i * t.W + k] = v - prev;  // ordering.cpp:33
      prev = v;
    }
  }
  return PM_OK;
}

// ---- evaluation ------------------------------------------------------------------

int pm_set_eval_kernel(pm_ctx* c, int kind) {
  if (!c) return PM_STRUCTURAL;
  if (kind < PM_EVAL_AUTO || kind > PM_EVAL_GATHER) return c->fail(PM_DOMAIN, "unknown evaluation kernel");
  c->eval_kind = kind;
  return PM_OK;
}

static bool scan_fits(pm_ctx* c, size_t count) {
  return plan_scan(c->t, std::max<size_t>(count, 64), c->sms, c->max_smem, false).ctas > 0;
}

// Measured crossover (profiles/r02_p_sweep.md): the scan touches
// ~(m+1)/(p+1) columns per client (time ~ a m / p + c), the gather p sites
// (time ~ b p), so they meet near p* ~ sqrt(a m / b); the n=m=10000 sweep with
// the fused gather (scan 0.700 / 0.408 ms, gather 0.621 / 0.943 ms at p = 100 /
// 200) puts it at p* ~ 110, i.e. p* ~ 1.1 sqrt(m).
static double auto_pstar(int m) { return 1.1 * std::sqrt((double)m); }

static int auto_kind(pm_ctx* c, size_t count) {
  if (!scan_fits(c, count)) return PM_EVAL_GATHER;
  return (double)c->t.p >= auto_pstar(c->t.m) ? PM_EVAL_SCAN : PM_EVAL_GATHER;
}

int pm_auto_eval_kernel(pm_ctx* c) {
  if (!c || !c->has_instance) return 0;
  return auto_kind(c, 4096);
}

// mode: 0 fitness (ordering.cpp:40-59), 1 min_cost_sum (instance.cpp:32-48),
// 2 scan depths (sum_i k*_i, the roofline's work measure).
}  // extern "C"

namespace pmb {
int evaluate_core(pm_ctx* c, const uint64_t* dwords, size_t count, int64_t* dcosts, int mode,
                  unsigned long long* errw_override) {
  const DevTables& t = c->t;
  const int wp = (t.m + 63) / 64;
  unsigned long long* errw = errw_override ? errw_override : c->errw.as<unsigned long long>();
  // one plan per evaluation (AUTO's fit check reuses it)
  ScanPlan sp;
  bool planned = false;
  auto plan = [&]() {
    if (!planned) sp = plan_scan(t, count, c->sms, c->max_smem, mode == 2);
    planned = true;
    return sp;
  };
  int kind = c->eval_kind;
  if (mode == 1) kind = PM_EVAL_GATHER;
  else if (mode == 2) kind = PM_EVAL_SCAN;
  else if (kind == PM_EVAL_AUTO)
    kind = (double)t.p >= auto_pstar(t.m) && plan().ctas > 0 ? PM_EVAL_SCAN : PM_EVAL_GATHER;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (kind == PM_EVAL_SCAN) {
    plan();
    if (sp.ctas == 0)
      return c->fail(PM_DOMAIN, "instance too large for the scan kernel's shared-memory masks; use PM_EVAL_GATHER");
    const size_t groups = (count + 63) / 64;
    PM_CUDA_TRY(c, c->T.ensure(groups * scan_t_stride(t.m) * 8));
    PM_CUDA_TRY(c, launch_transpose_population(dwords, count, wp, t.m, c->T.as<uint64_t>(),
                                               reinterpret_cast<unsigned long long*>(dcosts), errw_override,
                                               c->stream));
    if (c->profiling) {
      ev = c->ev_get();
      cudaEventRecord(ev.first, c->stream);
    }
    PM_CUDA_TRY(c, launch_scan(t, sp, c->T.as<uint64_t>(), count,
                               reinterpret_cast<unsigned long long*>(dcosts), errw, mode == 2, c->stream));
  } else if (gather_fused_fits(t)) {
    // one launch: lists in shared memory, costs stored; the error handoff
    // words are armed once per context
    if (!c->gsync.p) {
      PM_CUDA_TRY(c, c->gsync.ensure(16));
      PM_CUDA_TRY(c, cudaMemsetAsync(c->gsync.p, 0xff, 8, c->stream));
      PM_CUDA_TRY(c, cudaMemsetAsync(c->gsync.as<char>() + 8, 0, 8, c->stream));
    }
    if (c->profiling) {
      ev = c->ev_get();
      cudaEventRecord(ev.first, c->stream);
    }
    // several client slabs per chromosome: partial sums + arrival counters
    // (grown zeroed; the kernel leaves them at 0)
    const int ns = gather_fused_slabs(t);
    if (ns > 1) {
      PM_CUDA_TRY(c, c->gpart.ensure(count * ns * 8));
      if (c->garr.bytes < count * 4) {
        PM_CUDA_TRY(c, c->garr.ensure(count * 4));
        PM_CUDA_TRY(c, cudaMemsetAsync(c->garr.p, 0, c->garr.bytes, c->stream));
      }
    }
    PM_CUDA_TRY(c, launch_gather_fused(t, dwords, count, wp, reinterpret_cast<unsigned long long*>(dcosts),
                                       c->gpart.as<unsigned long long>(), c->garr.as<unsigned int>(),
                                       c->gsync.as<unsigned long long>(),
                                       reinterpret_cast<unsigned int*>(c->gsync.as<char>() + 8),
                                       errw_override ? errw_override : errw, errw_override != nullptr, mode,
                                       c->sms, c->stream));
    c->launches -= 1;  // one launch, not two
  } else {
    PM_CUDA_TRY(c, c->lists.ensure(count * (size_t)c->open_cap * 4));
    PM_CUDA_TRY(c, c->counts.ensure(count * 4));
    PM_CUDA_TRY(c, launch_open_lists(dwords, count, wp, t.m, c->lists.as<uint32_t>(),
                                     c->counts.as<uint32_t>(), c->open_cap,
                                     reinterpret_cast<unsigned long long*>(dcosts), errw_override, c->stream));
    if (c->profiling) {
      ev = c->ev_get();
      cudaEventRecord(ev.first, c->stream);
    }
    PM_CUDA_TRY(c, launch_gather(t, dwords, count, wp, c->lists.as<uint32_t>(), c->counts.as<uint32_t>(),
                                 c->open_cap, reinterpret_cast<unsigned long long*>(dcosts), errw, mode,
                                 c->sms, c->stream));
  }
  if (c->profiling) {
    cudaEventRecord(ev.second, c->stream);
    c->ev_used.push_back(ev);
  }
  c->launches += 2;
  return PM_OK;
}

}  // namespace pmb

extern "C" {

int pm_check_errors(pm_ctx* c, size_t* first_bad) {
  if (!c) return PM_STRUCTURAL;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  unsigned long long h = ~0ull;
  PM_CUDA_TRY(c, cudaMemcpyAsync(&h, c->errw.p, 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  PM_CUDA_TRY(c, cudaMemsetAsync(c->errw.p, 0xff, 8, c->stream));
  if (h != ~0ull) {
    if (first_bad) *first_bad = (size_t)h;
    return c->fail(PM_CONTRACT, kMsgRunoff);
  }
  return PM_OK;
}

static int evaluate_dev(pm_ctx* c, const uint64_t* dwords, size_t count, size_t words_per,
                        int64_t* dcosts, size_t* first_bad, int mode) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  if (words_per != (size_t)(c->t.m + 63) / 64) return c->fail(PM_STRUCTURAL, kMsgLength);
  if (count == 0) return PM_OK;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  if (first_bad) {  // synchronous error report for this call alone
    PM_CUDA_TRY(c, cudaMemsetAsync(c->errw.p, 0xff, 8, c->stream));
  }
  int rc = evaluate_core(c, dwords, count, dcosts, mode);
  if (rc != PM_OK) return rc;
  if (first_bad) {
    rc = pm_check_errors(c, first_bad);
    if (rc == PM_CONTRACT && mode == 1) c->err = kMsgNoneOpen;
    return rc;
  }
  return PM_OK;
}

int pm_evaluate_device(pm_ctx* c, const uint64_t* bitsets_device, size_t count, size_t words_per,
                       int64_t* costs_out_device, size_t* first_bad) {
  return evaluate_dev(c, bitsets_device, count, words_per, costs_out_device, first_bad, 0);
}

// Host-buffer calls: the population is copied in chunks on a copy stream and
// each chunk is evaluated on the compute stream as soon as it lands, so the
// H2D transfer overlaps the kernels; costs and the per-chunk error words come
// back with one synchronisation.
static int evaluate_host(pm_ctx* c, const uint64_t* bitsets, size_t count, size_t words_per,
                         int64_t* costs_out, size_t* first_bad, int mode) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  if (words_per != (size_t)(c->t.m + 63) / 64) return c->fail(PM_STRUCTURAL, kMsgLength);
  if (count == 0) return PM_OK;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  PM_CUDA_TRY(c, c->words.ensure(count * words_per * 8));
  // costs followed by the per-chunk error words: one device-to-host copy into pinned staging
  PM_CUDA_TRY(c, c->costs_out.ensure((count + kErrSlots) * 8));
  PM_CUDA_TRY(c, c->hout.ensure((count + kErrSlots) * 8));
  // Chunks of whole 64-chromosome groups: the copy of chunk k+1 overlaps the
  // kernels of chunk k, so only the first chunk's copy is exposed.  Each extra
  // launch costs a CTA-segment tail (round 1: equal chunks only paid off from
  // 8192 chromosomes and 16 MB on), so a batch of >= 4 MB is split into a short
  // lead chunk (a twelfth: its copy is the exposed part) and the rest;
  // PMB_H2D_LEAD=0 sends it in one piece, PMB_H2D_LEAD=<d> leads with 1/d.
  // Measured at syn20k, host-clock e2e (profiles/r02_e2e_ab.log): one piece
  // 2.63 M evals/s, lead 1/6 2.75 M, 1/8 2.80 M, 1/12 2.82 M, 1/16 2.76 M.
  const size_t bytes = count * words_per * 8;
  std::vector<size_t> starts{0};
  {
    const char* le = getenv("PMB_H2D_LEAD");
    const size_t lead_div = le ? (size_t)std::atoll(le) : 12;
    const int equal = (int)std::max<size_t>(
        1, std::min<size_t>({(size_t)kErrSlots - 1, count / 8192, bytes / (16u << 20)}));
    if (equal > 1) {
      const size_t per = ((count + equal - 1) / equal + 63) / 64 * 64;
      for (size_t off = per; off < count; off += per) starts.push_back(off);
    } else if (lead_div >= 2 && bytes >= ((size_t)4 << 20) && count >= 256) {
      const size_t lead = (count / lead_div + 63) / 64 * 64;
      if (lead > 0 && lead < count) starts.push_back(lead);
    }
  }
  const int chunks = (int)starts.size();
  while ((int)c->chunk_ev.size() < chunks) {
    cudaEvent_t e;
    PM_CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->chunk_ev.push_back(e);
  }
  // each chunk's error word sits after the costs and is set to "none" by the
  // chunk's first kernel (errw_override of evaluate_core)
  unsigned long long* slots = c->costs_out.as<unsigned long long>() + count;
  // the copies follow everything already queued on the compute stream (the
  // call is ordered like one stream operation: a caller's event recorded
  // before it brackets the whole transfer), and the scratch buffer `words` is
  // free again once the previous call's kernels have read it
  PM_CUDA_TRY(c, cudaEventRecord(c->entry_ev, c->stream));
  PM_CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->entry_ev, 0));
  int used = 0;
  for (; used < chunks; ++used) {
    const size_t off = starts[used];
    const size_t cnt = (used + 1 < chunks ? starts[used + 1] : count) - off;
    PM_CUDA_TRY(c, cudaMemcpyAsync(c->words.as<uint64_t>() + off * words_per, bitsets + off * words_per,
                                   cnt * words_per * 8, cudaMemcpyHostToDevice, c->copy_stream));
    PM_CUDA_TRY(c, cudaEventRecord(c->chunk_ev[used], c->copy_stream));
    PM_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->chunk_ev[used], 0));
    const int rc = evaluate_core(c, c->words.as<uint64_t>() + off * words_per, cnt,
                                 c->costs_out.as<int64_t>() + off, mode, slots + used);
    if (rc != PM_OK) return rc;
  }
  PM_CUDA_TRY(c, cudaMemcpyAsync(c->hout.p, c->costs_out.p, (count + used) * 8, cudaMemcpyDeviceToHost, c->stream));
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::memcpy(costs_out, c->hout.p, count * 8);
  const unsigned long long* errs = c->hout.as<unsigned long long>() + count;
  for (int i = 0; i < used; ++i)
    if (errs[i] != ~0ull) {
      if (first_bad) *first_bad = starts[i] + (size_t)errs[i];
      return c->fail(PM_CONTRACT, mode == 1 ? kMsgNoneOpen : kMsgRunoff);
    }
  return PM_OK;
}

int pm_evaluate(pm_ctx* c, const uint64_t* bitsets, size_t count, size_t words_per, int64_t* costs_out,
                size_t* first_bad) {
  return evaluate_host(c, bitsets, count, words_per, costs_out, first_bad, 0);
}

int pm_scan_depths_device(pm_ctx* c, const uint64_t* bitsets_device, size_t count, size_t words_per,
                          uint64_t* sum_k_device) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  size_t fb = 0;
  return evaluate_dev(c, bitsets_device, count, words_per, reinterpret_cast<int64_t*>(sum_k_device), &fb, 2);
}

int pm_scan_walks_device(pm_ctx* c, const uint64_t* bitsets_device, size_t count, size_t words_per,
                         uint64_t* group_walk_sum_device, uint32_t* client_max_walk_device) {
  if (!c) return PM_STRUCTURAL;
  if (!c->has_instance) return c->fail(PM_CONTRACT, "no instance set");
  if (words_per != (size_t)(c->t.m + 63) / 64) return c->fail(PM_STRUCTURAL, kMsgLength);
  if (count == 0) return PM_OK;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t groups = (count + 63) / 64;
  PM_CUDA_TRY(c, c->T.ensure(groups * scan_t_stride(c->t.m) * 8));
  PM_CUDA_TRY(c, c->scal.ensure(std::max<size_t>(16, count * 8)));
  PM_CUDA_TRY(c, launch_transpose_population(bitsets_device, count, (int)words_per, c->t.m, c->T.as<uint64_t>(),
                                             c->scal.as<unsigned long long>(), nullptr, c->stream));
  PM_CUDA_TRY(c, cudaMemsetAsync(group_walk_sum_device, 0, (count + 31) / 32 * 8, c->stream));
  PM_CUDA_TRY(c, cudaMemsetAsync(client_max_walk_device, 0, (size_t)c->t.n * 4, c->stream));
  PM_CUDA_TRY(c, launch_walks(c->t, c->T.as<uint64_t>(), count,
                              reinterpret_cast<unsigned long long*>(group_walk_sum_device),
                              client_max_walk_device, c->stream));
  c->launches += 2;
  PM_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PM_OK;
}

int pm_set_profiling(pm_ctx* c, int enabled) {
  if (!c) return PM_STRUCTURAL;
  c->profiling = enabled != 0;
  return PM_OK;
}

int pm_profile_read(pm_ctx* c, double* kernel_ms, uint64_t* kernel_launches) {
  if (!c) return PM_STRUCTURAL;
  PM_CUDA_TRY(c, cudaSetDevice(c->device));
  double total = 0;
  uint64_t cnt = 0;
  for (auto& e : c->ev_used) {
    PM_CUDA_TRY(c, cudaEventSynchronize(e.second));
    float ms = 0;
    PM_CUDA_TRY(c, cudaEventElapsedTime(&ms, e.first, e.second));
    total += ms;
    ++cnt;
    c->ev_free.push_back(e);
  }
  c->ev_used.clear();
  if (kernel_ms) *kernel_ms = total;
  if (kernel_launches) *kernel_launches = cnt;
  return PM_OK;
}

int pm_min_cost_sum(pm_ctx* c, const uint64_t* bitsets, size_t count, size_t words_per,
                    int64_t* costs_out, size_t* first_bad) {
  return evaluate_host(c, bitsets, count, words_per, costs_out, first_bad, 1);
}

}  // extern "C"
