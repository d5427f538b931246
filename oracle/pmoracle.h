/* pmoracle.h -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference's
 * fitness path (see pmoracle.c).  Never linked by the product. */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the product C-ABI (include/pmedian_b200.h) */
enum { OR_OK = 0, OR_STRUCTURAL = 1, OR_CONTRACT = 2, OR_DOMAIN = 3, OR_BUDGET = 4 };

uint64_t or_mix64(uint64_t z);
uint64_t or_rs_derive(uint64_t master, const uint64_t* key, size_t nkey);
uint64_t or_rs_next(uint64_t* state);
uint64_t or_rs_below(uint64_t* state, uint64_t bound);
int or_rs_coin(uint64_t* state);

void or_synth_euclid(uint64_t seed, size_t npts, int64_t* costs);
void or_random_costs(uint64_t seed, size_t n, size_t m, int64_t max_cost, int64_t* costs);
void or_random_population(uint64_t seed, size_t m, size_t p, size_t count, uint64_t* words);

int or_validate_instance(size_t n, size_t m, size_t p, const int64_t* costs, size_t ncosts);
void or_build_ordering(size_t n, size_t m, size_t p, const int64_t* costs, uint32_t* site_order,
                       int64_t* increments);
int or_fitness(size_t n, size_t width, const uint32_t* site_order, const int64_t* increments,
               const uint64_t* words, int64_t* out);
int or_evaluate_population(size_t n, size_t m, size_t width, const uint32_t* site_order,
                           const int64_t* increments, const uint64_t* words, size_t words_per,
                           size_t count, int64_t* costs_out, uint64_t* sum_k_out,
                           size_t* first_bad);
int or_min_cost_sum(size_t n, size_t m, const int64_t* costs, const uint64_t* words,
                    int64_t* out);
int or_direct_cost(size_t n, size_t m, size_t p, const int64_t* costs, const uint64_t* words,
                   int64_t* out);

int or_orlib_closure(size_t n, size_t edges, const int64_t* uv, const int64_t* w, int64_t* out,
                     size_t* bad);

#ifdef __cplusplus
}
#endif
