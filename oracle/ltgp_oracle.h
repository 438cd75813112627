/*
 * ltgp_oracle.h — C interface of the CPU ORACLE (test infrastructure only).
 *
 * This library is the parity checker for the B200 engine. It restates, on
 * the CPU, the algorithms the reference declares in
 * /root/reference/proj/include/ltgp/ (the *.hpp headers) and specifies in
 * /root/reference/SPEC.md. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * (paper_1902_09215_b200/) never links, imports or calls it.
 *
 * Parity pins: SPEC examples, the paper's
 * Table 1 protected-division footnote and known-answer
 * values computed from the reference's inline code (rng.hpp:9-51,
 * eval.hpp:54-63, eval.hpp:89-98). The reference has no implementation
 * bodies, so nothing else can be pinned.
 */
#ifndef LTGP_ORACLE_H
#define LTGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    float fitness;
    int32_t hits;
    uint32_t size;
    uint32_t depth;
} orc_record;

typedef struct {
    uint32_t mum_index, dad_index, mum_pt, dad_pt;
} orc_plan;

/* rng.hpp:9-51 */
uint64_t orc_splitmix64(uint64_t x);
void orc_rng_below_seq(uint64_t seed, uint64_t n, uint32_t count, uint64_t* out);
void orc_rng_uniform_seq(uint64_t seed, uint32_t count, float* out);
/* eval.hpp:54-63, 89-98, 100-102 */
float orc_protected_div(float a, float b);
int orc_fitness_better(float a, float b);
int orc_fitness_tied(float a, float b);
double orc_flajolet_stack_bound(uint64_t capacity, double safety);
/* genome.hpp:40-57, 71-84 */
int orc_validate(const uint8_t* ops, uint64_t n);
uint64_t orc_depth(const uint8_t* ops, uint64_t n);
int orc_subtree_extent(const uint8_t* ops, uint64_t n, uint64_t idx, uint64_t* start, uint64_t* end);
uint64_t orc_crossover_child_size(const uint8_t* mum, uint64_t mn, const uint8_t* dad, uint64_t dn,
                                  uint64_t mum_pt, uint64_t dad_pt);
/* returns child size; writes child to out when size < capacity and out_cap is big enough;
   *size_limit_hit = 1 (nothing written) when child >= capacity */
uint64_t orc_crossover(const uint8_t* mum, uint64_t mn, const uint8_t* dad, uint64_t dn,
                       uint64_t mum_pt, uint64_t dad_pt, uint64_t capacity, uint8_t* out,
                       uint64_t out_cap, int* size_limit_hit);
/* sextic.hpp:33-51, driver.hpp:17-19 */
float orc_target(float x);
uint64_t orc_suite_seed(uint64_t run_seed);
void orc_make_suite(uint64_t seed, float* inputs48, float* targets48, float* consts250);
/* genome.hpp:59-69, bench.hpp:13-15: generators. Return size, or 0 when the
   tree exceeds capacity/out_cap (gen_* throw std::length_error there). */
uint64_t orc_gen_full(uint64_t* rng_state_seed, int depth, uint64_t capacity, uint8_t* out,
                      uint64_t out_cap);
/* Ramped half-and-half for `count` genomes from Rng(seed): writes all genomes
   back to back into out, sizes into sizes. Returns total bytes or 0. */
uint64_t orc_ramped_half_and_half(uint64_t seed, uint32_t count, uint64_t capacity, int min_depth,
                                  int max_depth, uint8_t* out, uint64_t out_cap, uint64_t* sizes);
/* random_tree_of_size from Rng(seed) (one tree per call). */
int orc_random_tree_of_size(uint64_t seed, uint64_t n, uint8_t* out);
/* BASELINE.json configs[2] corpus (same bytes as the product's generator):
   sizes[M] always; with buf/offsets, trees [first, first+count) packed
   16-byte aligned. Returns the packed byte count. */
uint64_t orc_corpus(uint64_t seed, uint32_t M, double lg_lo, double lg_hi, uint32_t first, uint32_t count,
                    uint8_t* buf, uint64_t* offsets, uint64_t* sizes, int threads);
/* eval.hpp:65-87 */
float orc_eval_scalar(const uint8_t* ops, uint64_t n, float x, const float* consts250);
/* 0 ok, <0 malformed; out48 receives the result frame; peak receives peak frames */
int orc_eval_batch(const uint8_t* ops, uint64_t n, const float* inputs48, const float* consts250,
                   float* out48, uint64_t* peak_frames);
float orc_fitness(const float* out48, const float* targets48);
int32_t orc_hits(const float* out48, const float* targets48, float threshold);
/* evolve.hpp:106-109: evaluate M genomes stored at ops+offsets[i] with sizes[i];
   threads = worker count (0 = hardware concurrency). Returns node count. */
uint64_t orc_evaluate_population(uint32_t M, const uint8_t* ops, const uint64_t* offsets,
                                 const uint64_t* sizes, const float* inputs48,
                                 const float* targets48, const float* consts250, int threads,
                                 orc_record* out);
/* evolve.hpp:79-87 */
uint32_t orc_tournament_seq(uint64_t seed, uint32_t M, const float* fitness, uint32_t k,
                            uint32_t count, uint32_t* out);
void orc_plan_generation(uint64_t seed, uint32_t M, const orc_record* pop, uint32_t k,
                         orc_plan* out);
/* run.hpp:33-36 — full generational loop. Writes a population dump (one
   line per individual per generation, stats.hpp:104-107) into dump_path
   (NULL = none). Returns generations completed; *reason: 0 MaxGenerations,
   1 SizeLimitHit, 2 MemoryBudgetExceeded. grow_mode: 0 = SPEC grow (uniform
   over the 255 primitives), 1 = 50/50 function-vs-terminal grow.
   memory_budget (RunConfig::memory_budget_bytes, evolve.hpp:44; 0 = off):
   before a generation is materialized, planned_generation_bytes (parents
   plus every planned child, child sizes from the crossover algebra;
   evolve.hpp:89-93) must not exceed it. */
int64_t orc_run(uint32_t M, uint32_t max_generations, uint64_t node_limit, uint32_t k,
                uint64_t seed, int threads, const char* dump_path, int* reason,
                uint64_t* nodes_evaluated, int grow_mode, uint64_t memory_budget);

#ifdef __cplusplus
}
#endif
#endif
