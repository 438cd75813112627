/*
 * ltgp_host.h — C entry points of libltgp_host.so, the C++ host side that
 * keeps the reference's population, selection and crossover API
 * (/root/reference/proj/include/ltgp/{rng,genome,sextic,evolve,run,bench}.hpp)
 * and drives the B200 engine through include/ltgp_cuda.h.
 *
 * The C++ API itself is paper_1902_09215_b200/host/ltgp/ltgp.hpp (namespace
 * ltgp, the reference's names and signatures); these C wrappers exist for
 * bench.py and the Python tests (ctypes).
 */
#ifndef LTGP_HOST_H
#define LTGP_HOST_H

#include <stdint.h>

#include "ltgp_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:9-51 */
uint64_t ltgp_host_splitmix64(uint64_t x);
/* driver.hpp:17-19 + sextic.hpp:50-51 */
uint64_t ltgp_host_suite_seed(uint64_t run_seed);
void ltgp_host_make_suite(uint64_t seed, float* inputs48, float* targets48, float* consts250);

/* Evaluation-only corpus (BASELINE config 3 and the bench harness of
   bench.hpp:13-15 / driver.hpp:44-51): M trees, tree i of size
   odd(floor(10^(lg_lo + (lg_hi-lg_lo) u_i))) with u_i uniform from
   Rng(seed), shape from random_tree_of_size(Rng(tree_seed(seed, i)), n_i).
   sizes[M] always receives every tree size. Trees [first, first+count) are
   packed (16-byte aligned offsets relative to buf, offsets[count]); with
   buf == NULL only the layout is computed. Returns the packed byte count of
   the range. threads: 0 = all hardware threads. */
uint64_t ltgp_host_corpus(uint64_t seed, uint32_t M, double lg_lo, double lg_hi, uint32_t first,
                          uint32_t count, uint8_t* buf, uint64_t* offsets, uint64_t* sizes, int threads);
/* The host's bulk std::mt19937_64 engine against the standard library's:
   outputs and text state (0 = identical). */
int ltgp_host_rng_selftest(void);
uint64_t ltgp_host_tree_seed(uint64_t seed, uint32_t i);
/* random_tree_of_size (bench.hpp:15) from Rng(seed). 0 ok. */
int ltgp_host_random_tree_of_size(uint64_t seed, uint64_t n, uint8_t* out);
/* Random uniform binary tree shape by Remy's repeated random insertion
   (BASELINE config 4), n odd; labels as in config 3. 0 ok. */
int ltgp_host_remy_tree(uint64_t seed, uint64_t n, uint8_t* out);
/* ramped_half_and_half (genome.hpp:66-69) from Rng(seed), packed back to back. */
uint64_t ltgp_host_ramped(uint64_t seed, uint32_t count, uint64_t capacity, int min_depth,
                          int max_depth, uint8_t* out, uint64_t out_cap, uint64_t* sizes);
/* plan_generation (evolve.hpp:84-87) from Rng(seed) over M records. */
void ltgp_host_plan_generation(uint64_t seed, uint32_t M, const ltgp_record* pop, uint32_t k,
                               ltgp_plan* out);

/* run() (run.hpp:33-36) on the engine: ramped init, generation-0
   evaluation, plan/execute until max_generations, SizeLimitHit or (with a
   non-zero memory_budget = RunConfig::memory_budget_bytes) MemoryBudgetExceeded.
   *reason: 0 MaxGenerations, 1 SizeLimitHit, 2 MemoryBudgetExceeded
   (TerminationReason, evolve.hpp:34). Writes the determinism dump
   (stats.hpp:104-107) to dump_path (NULL: none) and returns generations
   completed (< 0: error, see ltgp_last_error()). grow_mode: 0 = SPEC grow
   (uniform over the 255 primitives), 1 = 50/50 function-vs-terminal grow
   (SPEC.md:148 open question; the variant whose runs bloat). */
int64_t ltgp_host_run(ltgp_engine* e, uint32_t M, uint32_t max_generations, uint64_t node_limit,
                      uint32_t k, uint64_t seed, int grow_mode, uint64_t memory_budget,
                      const char* dump_path, int* reason, uint64_t* nodes_evaluated, double* eval_seconds);

/* ltgp_host_run with checkpoint/resume: when
   ckpt_every > 0, after generation 0 and every ckpt_every-th generation (and
   the last) the population's genomes (downloaded from the device), records,
   Rng stream position and run counters are written to ckpt_path (atomically,
   via ckpt_path.tmp). resume_path (NULL: fresh start) continues a run from
   such a file: the parameters must equal the checkpointed run's (else error),
   the parents are re-uploaded with their records restored, the dump is
   appended to, and the return value and *nodes_evaluated / *eval_seconds
   count the whole run. A resumed run's dump equals the uninterrupted run's. */
int64_t ltgp_host_run_checkpointed(ltgp_engine* e, uint32_t M, uint32_t max_generations, uint64_t node_limit,
                                   uint32_t k, uint64_t seed, int grow_mode, uint64_t memory_budget,
                                   const char* dump_path, const char* ckpt_path, uint32_t ckpt_every,
                                   const char* resume_path, int* reason, uint64_t* nodes_evaluated,
                                   double* eval_seconds);

/* BenchCell (bench.hpp:17-27) of run_bench on the engine: workers = GPUs
   (devices 0..workers-1); batch_gpops = one GPU, parallel_gpops = `workers`
   GPUs, device-timed, best of `repeats`. The engine has no CPU interpreter:
   scalar_gpops and vector_speedup are 0. */
typedef struct {
    uint64_t tree_size;
    uint32_t workers;
    uint64_t nodes;
    double scalar_gpops, batch_gpops, parallel_gpops, vector_speedup, parallel_speedup;
    int counters_consistent;
} ltgp_bench_cell;

/* run_bench (bench.hpp:33-35): for each tree size (made odd) a corpus of
   ceil(min_corpus_nodes / size) random_tree_of_size trees (tree i from
   Rng(tree_seed(seed, i))), the Sextic suite of suite_seed(seed), one cell
   per (size, worker count) in that order into out[n_sizes * n_workers].
   0 ok, -1 on invalid arguments or an engine error. */
int ltgp_host_run_bench(const uint64_t* tree_sizes, uint32_t n_sizes, const uint32_t* worker_counts,
                        uint32_t n_workers, uint64_t seed, uint64_t min_corpus_nodes, int repeats,
                        ltgp_bench_cell* out);

#ifdef __cplusplus
}
#endif
#endif
