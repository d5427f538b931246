/*
 * pmedian_b200.h -- C ABI of the B200-native HBP fitness path.
 *
 * The reference (arXiv 1610.10061's `pmedian` C++ library, /root/reference/proj)
 * has no FFI: its boundary is the C++ API in proj/include/pmedian/.  This ABI
 * is what a maintainer binds underneath that API; every
 * entry point names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "host" buffers are ordinary CPU memory;
 *    "_device" entry points take CUDA device pointers and run on the context's
 *    stream without synchronising unless stated.
 *  - Chromosome wire format = the reference's Chromosome words
 *    (proj/include/pmedian/chromosome.hpp:24,43): m bits per chromosome packed
 *    into words_per = ceil(m/64) uint64 words, site j = bit (j & 63) of word
 *    (j >> 6).  A population is count x words_per, row-major.  Bits at
 *    positions >= m are ignored.
 *  - Every call returns a pm_status.  The message of the last failure is kept
 *    per context (pm_last_error).  Status codes map one-to-one onto the
 *    reference's exception types (proj/include/pmedian/errors.hpp:8-25) and
 *    the message texts are the reference's.
 *  - A context is not thread-safe: one context per host thread.
 */
#ifndef PMEDIAN_B200_H_
#define PMEDIAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pm_status {
  PM_OK = 0,
  PM_STRUCTURAL = 1, /* pmedian::StructuralError (errors.hpp:8-10) */
  PM_CONTRACT = 2,   /* pmedian::ContractError   (errors.hpp:13-15) */
  PM_DOMAIN = 3,     /* pmedian::DomainError     (errors.hpp:18-20) */
  PM_BUDGET = 4,     /* pmedian::BudgetError     (errors.hpp:23-25) */
  PM_CUDA = 5,       /* CUDA runtime failure (no reference equivalent) */
  PM_NCCL = 6        /* collective failure (no reference equivalent) */
} pm_status;

/* Fitness kernel selection (SURVEY.md 8(d) "scan vs gather crossover"). */
typedef enum pm_eval_kernel {
  PM_EVAL_AUTO = 0,   /* measured crossover table picks scan or gather */
  PM_EVAL_SCAN = 1,   /* K2: bit-sliced scan of Pi'/D' to the first open site */
  PM_EVAL_GATHER = 2  /* K2b: gather-min over the open sites, site-major costs */
} pm_eval_kernel;

typedef struct pm_ctx pm_ctx;

typedef struct pm_table_info {
  size_t clients;     /* n                       (OrderingTables::clients, ordering.hpp:18) */
  size_t sites;       /* m                       (OrderingTables::sites, ordering.hpp:19) */
  size_t open_count;  /* p                       (OrderingTables::open_count, ordering.hpp:20) */
  size_t width;       /* W = m - p + 1           (OrderingTables::width, ordering.hpp:21) */
  size_t row_stride;  /* padded device row length in elements (>= width, multiple of 16) */
  int site_bytes;     /* device Pi' element width: 2 (m < 65535) or 4 */
  int dist_bytes;     /* device sorted-distance element width: 2, 4 or 8 */
  int64_t max_cost;   /* largest cost in the matrix */
} pm_table_info;

/* ---- context ----------------------------------------------------------- */

/* Initialises the CUDA runtime on `device` (the one-time context creation,
 * hundreds of milliseconds) without creating a pm_ctx; PM_CUDA without a device.
 * As the process's first CUDA call it also selects eager module loading
 * (CUDA_MODULE_LOADING=EAGER unless the caller set it), so no kernel pays its
 * load time inside a timed call. */
int pm_warmup(int device);
/* Creates a context on CUDA device `device` with its own non-blocking stream. */
int pm_create(int device, pm_ctx** out);
void pm_destroy(pm_ctx* ctx);
/* Text of the last failure on this context ("" if none).  Valid until the next call. */
const char* pm_last_error(const pm_ctx* ctx);
/* Routes all later work to `stream` (a cudaStream_t; NULL restores the context's own).
 * Device buffers passed to the *_device entry points are read in order on this
 * stream: a producer on another stream must be complete (or joined with an
 * event) first.  The context's own stream is non-blocking, i.e. it does not
 * order against the legacy default stream. */
int pm_set_stream(pm_ctx* ctx, void* stream);
/* Number of kernels this context has launched so far (evidence counter for bench/tests). */
uint64_t pm_kernel_launches(const pm_ctx* ctx);

/* ---- instance + ordering tables (K1) ------------------------------------
 * Replaces pmedian::Instance::Instance (instance.cpp:10-30) validation and
 * pmedian::build_ordering (ordering.hpp:33, ordering.cpp:10-38).  Validates
 * exactly as the Instance constructor does (same errors, same texts), then
 * builds Pi' and the sorted distances on the device and keeps them resident
 * together with the site-major cost matrix used by the gather kernel.
 * `costs` is n x m row-major int64, caller-owned, read during the call only. */
int pm_set_instance(pm_ctx* ctx, const int64_t* costs, size_t n, size_t m, size_t p);
/* Same with `costs` already in device memory (no host copy). */
int pm_set_instance_device(pm_ctx* ctx, const int64_t* costs_device, size_t n, size_t m, size_t p);
int pm_table_info_get(pm_ctx* ctx, pm_table_info* out);
/* Copies the tables back in the reference's own layout (OrderingTables::site_order
 * uint32 and ::increments int64, clients x width row-major, ordering.hpp:22-23).
 * For parity checks; synchronises. */
int pm_get_tables(pm_ctx* ctx, uint32_t* site_order, int64_t* increments);

/* ---- population evaluation (K2 / K2b) -----------------------------------
 * Replaces one pmedian::fitness(tables, c) call per chromosome
 * (ordering.hpp:39, ordering.cpp:40-59) as called by evolve_block
 * (ga.cpp:147,166,183).  costs_out[c] is bit-identical to fitness().
 * Errors: words_per != ceil(m/64) -> PM_STRUCTURAL with the text of
 * ordering.cpp:42; a chromosome with no open site inside the scan width ->
 * PM_CONTRACT with the text of ordering.cpp:51 and *first_bad = the LOWEST such
 * chromosome index (what a sequential loop of fitness() calls throws first).
 * Host-buffer form: copies in, evaluates, copies out, synchronises. */
int pm_evaluate(pm_ctx* ctx, const uint64_t* bitsets, size_t count, size_t words_per,
                int64_t* costs_out, size_t* first_bad);
/* Device-buffer form.  If first_bad is NULL the call is fully asynchronous on
 * the context stream and errors are reported by pm_check_errors; otherwise it
 * synchronises and reports as pm_evaluate. */
int pm_evaluate_device(pm_ctx* ctx, const uint64_t* bitsets_device, size_t count,
                       size_t words_per, int64_t* costs_out_device, size_t* first_bad);
/* Synchronises and reports any contract failure recorded by asynchronous calls
 * since the last check. */
int pm_check_errors(pm_ctx* ctx, size_t* first_bad);
/* Chooses the evaluation kernel (default PM_EVAL_AUTO). */
int pm_set_eval_kernel(pm_ctx* ctx, int kind);
/* Kernel PM_EVAL_AUTO would pick for the current instance (1 = scan, 2 = gather). */
int pm_auto_eval_kernel(pm_ctx* ctx);

/* Gather-min without the scan-width contract: replaces pmedian::min_cost_sum
 * (instance.hpp:39, instance.cpp:32-48) per chromosome; a chromosome with no
 * open site -> PM_CONTRACT "at least one site must be open". */
int pm_min_cost_sum(pm_ctx* ctx, const uint64_t* bitsets, size_t count, size_t words_per,
                    int64_t* costs_out, size_t* first_bad);

/* ---- measurement hooks -----------------------------------------------------
 * Per chromosome, the sum over clients of the 1-based stopping column k*_i of
 * the reference scan (ordering.cpp:49-55) -- the work measure of the roofline
 * (B_eval = 12 * sum_i k*_i + 8 * ceil(m/64)).  Device
 * buffers; synchronises; PM_CONTRACT as pm_evaluate on a runoff. */
int pm_scan_depths_device(pm_ctx* ctx, const uint64_t* bitsets_device, size_t count,
                          size_t words_per, uint64_t* sum_k_device);
/* The scan's reuse-aware work (measurement only): per 32-chromosome group g
 * (ceil(count/32) entries) the sum over clients of walk_gi = max_{c in g} k*_ic
 * -- the columns K2 walks once for the whole group -- and per client the
 * maximum walk over all groups (n entries), i.e. the row prefix that must be
 * read from DRAM at least once.  Device buffers; synchronises. */
int pm_scan_walks_device(pm_ctx* ctx, const uint64_t* bitsets_device, size_t count, size_t words_per,
                         uint64_t* group_walk_sum_device, uint32_t* client_max_walk_device);
/* When enabled, CUDA events on the context stream bracket every launch of the
 * dominant evaluation kernel (K2 scan or K2b gather). */
int pm_set_profiling(pm_ctx* ctx, int enabled);
/* Synchronises, returns the summed duration (ms) and count of the bracketed
 * launches since the last read, and resets. */
int pm_profile_read(pm_ctx* ctx, double* kernel_ms, uint64_t* kernel_launches);

/* ---- instance ingestion (proj/src/bench.cpp:65-168) ---------------------------
 * OR-Library graph text ("n edges p" + "u v cost" triples): the reference's
 * parse_orlib diagnostics (same texts), then the all-pairs shortest-path closure
 * on the device (blocked Floyd-Warshall) and pm_set_instance_device on it.
 * p_override != 0 replaces the file's p (run_benchmark's --p). */
int pm_set_instance_orlib(pm_ctx* ctx, const char* text, size_t len, size_t p_override);
/* The closure alone, copied to the host (n*n int64 into costs_out, capacity entries). */
int pm_orlib_closure(pm_ctx* ctx, const char* text, size_t len, int64_t* costs_out, size_t capacity,
                     size_t* n_out, size_t* p_out);
/* Dense text ("n m p" + n rows of m costs): parse_dense diagnostics, then pm_set_instance. */
int pm_set_instance_dense(pm_ctx* ctx, const char* text, size_t len, size_t p_override);
/* parse_dense alone (bench.cpp:65-104): n, m, p and the n*m costs (costs_out may be
 * NULL to query the sizes; capacity in entries).  Same diagnostics. */
int pm_parse_dense(pm_ctx* ctx, const char* text, size_t len, int64_t* costs_out, size_t capacity, size_t* n_out,
                   size_t* m_out, size_t* p_out);

/* ---- genetic algorithm (K3 evolve, K4 islands) ------------------------------ */

enum { PM_MIGRATE_BLOCK = 0, PM_MIGRATE_TEAM = 1 }; /* MigrationMode, ga.hpp:22 */
enum {
  /* the reference's exact draw: one host stream derive(seed, {1}), BigInt
   * unranking of a uniform rank (combinatorics.cpp:54-75, ga.cpp:226-235) --
   * run_ga results equal the reference's bit for bit */
  PM_POPULATION_REFERENCE = 0,
  /* device draw: Floyd's algorithm per chromosome from derive(seed, {4,
   * generation, global index}); same distribution, not the same sequence */
  PM_POPULATION_DEVICE = 1
};

/* GaConfig (ga.hpp:24-38).  crossover_iters / mutation_iters < 0 mean "lg(nt)". */
typedef struct pm_ga_config {
  size_t nb;
  size_t nt;
  size_t evolve_limit;
  size_t saturation;
  uint64_t seed;
  long long crossover_iters;
  long long mutation_iters;
  int migration;
  int population;
} pm_ga_config;

/* RunResult (ga.hpp:49-56) plus work counters. */
typedef struct pm_run_result {
  int64_t best_cost;
  size_t kernels_executed;
  size_t kernel_of_best; /* 1-based */
  double wall_time_s;
  double evolve_time_s;        /* host time spent in the generation loop */
  uint64_t evaluations;        /* fitness calls the reference run would make (this island) */
  uint64_t device_evaluations; /* chromosomes evaluated on the device (includes skipped attempts) */
} pm_run_result;

/* Replaces pmedian::evolve_block (ga.hpp:100-102) for nb consecutive blocks at
 * once: blocks = nb x cfg->nt chromosomes (host, words_per words each, block
 * major), evolved in place with kernel index `kernel_index` and block indices
 * first_block .. first_block+nb-1; best_cost/best_thread (nb entries) receive
 * each block's BlockResult (the best chromosome is blocks[b][best_thread]).
 * Every chromosome must open exactly p sites (PM_DOMAIN otherwise) -- the GA
 * invariant; the reference only fails later, inside crossover or fitness. */
int pm_evolve_blocks(pm_ctx* ctx, uint64_t* blocks, size_t nb, size_t words_per, const pm_ga_config* cfg,
                     uint64_t kernel_index, size_t first_block, int64_t* best_cost, size_t* best_thread);

/* Replaces pmedian::run_ga (ga.hpp:109) on the context's instance.  best_words
 * (ceil(m/64) words) receives RunResult::best; per_kernel_best, if not NULL,
 * receives RunResult::per_kernel_best_costs (kernels_executed <= evolve_limit
 * entries).  A caller that cannot size a buffer by evolve_limit (a large limit
 * that relies on saturation) passes NULL and reads them afterwards with
 * pm_last_per_kernel_best.  The generation step -- global best, stop rule,
 * migration (ga.cpp:279-297) -- runs on the device; the host reads one stop
 * word per generation. */
int pm_run_ga(pm_ctx* ctx, const pm_ga_config* cfg, uint64_t* best_words, int64_t* per_kernel_best,
              pm_run_result* result);

/* Islands over processes/GPUs: this rank evolves blocks
 * [rank*nb/world, (rank+1)*nb/world) (nb must divide evenly) and every
 * generation exchanges its block bests through `allgather` (send `bytes`,
 * receive world*bytes in rank order; return 0 on success), so every rank
 * computes the same global best, stop decision and RunResult.  RNG keys use
 * global block indices: any world size gives the identical RunResult. */
typedef int (*pm_allgather_fn)(const void* send, size_t bytes, void* recv, void* user);
int pm_run_ga_islands(pm_ctx* ctx, const pm_ga_config* cfg, int rank, int world, pm_allgather_fn allgather,
                      void* user, uint64_t* best_words, int64_t* per_kernel_best, pm_run_result* result);

/* The same with a DEVICE collective: `allgather` enqueues the gather of the
 * device buffer `send_device` (bytes) into `recv_device` (world * bytes, rank
 * order) on `stream` (a cudaStream_t, the context's) and returns 0 -- e.g.
 * pm_nccl_allgather_device.  The block records, the exchange and the
 * generation step stay on the device: no host staging. */
typedef int (*pm_allgather_device_fn)(const void* send_device, size_t bytes, void* recv_device, void* stream,
                                      void* user);
int pm_run_ga_islands_device(pm_ctx* ctx, const pm_ga_config* cfg, int rank, int world,
                             pm_allgather_device_fn allgather, void* user, uint64_t* best_words,
                             int64_t* per_kernel_best, pm_run_result* result);

/* RunResult::per_kernel_best_costs of the last pm_run_ga* call on this
 * context: *count = kernels executed; min(count, capacity) entries copied. */
int pm_last_per_kernel_best(pm_ctx* ctx, int64_t* out, size_t capacity, size_t* count);

/* Native island exchange over NCCL (NVLink/NVSwitch on one node) for C/C++
 * hosts without torch.distributed: one communicator per rank, created from a
 * unique id that rank 0 generates and the launcher distributes (file, MPI,
 * socket ...).  pm_nccl_allgather has the pm_allgather_fn shape; pass the
 * pm_nccl* as `user`.  The record travels through device memory and one
 * ncclAllGather on the communicator's stream.  PM_NCCL on failure. */
#define PM_NCCL_ID_BYTES 128
typedef struct pm_nccl pm_nccl;
int pm_nccl_unique_id(char id[PM_NCCL_ID_BYTES]);
int pm_nccl_create(const char id[PM_NCCL_ID_BYTES], int rank, int world, int device, pm_nccl** out);
void pm_nccl_destroy(pm_nccl* comm);
int pm_nccl_allgather(const void* send, size_t bytes, void* recv, void* user);
/* pm_allgather_device_fn over the communicator: one ncclAllGather of device
 * buffers enqueued on `stream` (asynchronous).  pass the pm_nccl* as `user`. */
int pm_nccl_allgather_device(const void* send_device, size_t bytes, void* recv_device, void* stream, void* user);
/* rank / world size of a communicator */
int pm_nccl_rank(const pm_nccl* comm, int* rank, int* world);

#ifdef __cplusplus
}
#endif

#endif /* PMEDIAN_B200_H_ */
