/*
 * ltgp_cuda.h — C ABI of the B200 fitness-evaluation engine (libltgp_cuda.so).
 *
 * This is the drop-in boundary for the reference's population API
 * (/root/reference/proj/include/ltgp/evolve.hpp:95-117 and eval.hpp:65-87).
 * Every entry point below names the reference declaration it replaces.
 * Plain C types only: no exceptions, no C++ or torch types cross it.
 *
 * Conventions:
 *  - every call returns int status: 0 = ok, < 0 = error (ltgp_last_error()
 *    has the message). A crossover reaching the node limit is NOT an error:
 *    it is reported through an out-flag, like CrossoverResult::size_limit_hit
 *    (genome.hpp:71-74) and ExecOutcome::size_limit_hit (evolve.hpp:102-104).
 *  - the caller owns host arrays; the engine owns device arenas and genomes
 *    by population slot.
 *  - one coordinator thread per engine handle (the reference's sequential
 *    coordinator). Shards of the population may live on
 *    several GPUs (devices[]); the engine uses one CUDA stream per shard.
 */
#ifndef LTGP_CUDA_H
#define LTGP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTGP_LANES 48       /* kLaneWidth, common.hpp:10-11 */
#define LTGP_CONSTANTS 250  /* kConstantCount, opcodes.hpp:18 */
#define LTGP_MAX_SHARDS 16

typedef struct ltgp_engine ltgp_engine;

/* Per-individual record: Individual minus the genome (evolve.hpp:17-23). */
typedef struct {
    float fitness;  /* MAE, sequential lane order (eval.hpp:81-84); NaN possible */
    int32_t hits;   /* lanes with |o-t| <= 0.01f (eval.hpp:86-87) */
    uint32_t size;  /* nodes */
    uint32_t depth; /* single node = 1 (genome.hpp:45-46) */
} ltgp_record;

/* CrossoverPlan (evolve.hpp:25-32). */
typedef struct {
    uint32_t mum_index, dad_index, mum_pt, dad_pt;
} ltgp_plan;

typedef struct {
    int n_shards;                     /* 1..LTGP_MAX_SHARDS */
    int devices[LTGP_MAX_SHARDS];     /* CUDA ordinal per shard (may repeat) */
    uint64_t node_limit;              /* RunConfig::node_limit (evolve.hpp:40) */
    uint64_t arena_bytes;             /* per shard and buffer; 0 = grow on demand */
    uint32_t chunk_nodes;             /* intra-tree chunk length; 0 = default */
    int use_nccl;                     /* 1: NCCL all-gather when devices are distinct */
} ltgp_config;

/* Counters (GpopsCounter, eval.hpp:14-25, plus device timings). */
typedef struct {
    uint64_t nodes_evaluated;   /* sum of sizes over all evaluations */
    double eval_seconds;        /* device time of the last evaluation (CUDA events) */
    double eval_kernel_seconds; /* of which the scan pass: k_decode + k_plan + k_eval (+ overflow re-runs) */
    double combine_seconds;     /* of which the spine combine kernel (k_combine) */
    double splice_seconds;      /* device time of the last splice (k_splice) */
    double gather_seconds;      /* device time of the last record all-gather */
    uint64_t arena_high_water;  /* bytes, max over shards */
    uint64_t last_chunks;       /* chunk work items of the last evaluation */
    uint64_t last_fallback_items; /* items re-run with worst-case capacities */
    uint64_t last_exits;        /* packets the fast path handed to the checked / window path */
    uint64_t last_window_adjusts; /* of which needed a stack window spill or refill */
    uint64_t last_spine_steps;  /* spine steps the chunk summaries of the last evaluation hold */
    uint32_t kernel_launches;   /* engine kernels launched by the last call */
    uint32_t gather_nccl;       /* 1: records are all-gathered by NCCL (distinct devices, use_nccl);
                                   2: across processes (ltgp_nccl_attach) */
    double keval_seconds;       /* k_eval alone, max over shards (resident evaluations; 0 when streamed) */
    uint64_t live_genomes_high_water; /* streaming memory mode: most live genomes (parents not yet
                                         retired + children built) seen at a wave boundary */
    uint64_t arena_used_high_water;   /* streaming memory mode: most arena bytes holding live genomes */
    uint64_t last_h2d_bytes;    /* host-to-device bytes of the last ltgp_evaluate_packed (packed slices,
                                   ltgp_pack.h; the raw bytes with LTGP_PACK=0) */
} ltgp_stats;

/* Generation statistics of the current population (GenerationStats,
   stats.hpp:14-27; best_index / convergence, stats.hpp:36-40), reduced on the
   device from the records of the last evaluation. */
typedef struct {
    uint32_t best_index;    /* first slot holding the best fitness (NaN is worst) */
    float best_fitness;
    int32_t best_hits;
    uint32_t best_size;
    uint32_t best_depth;
    uint32_t convergence;   /* slots whose fitness is bit-equal to the best's */
    uint32_t max_size;
    uint32_t pad;
    uint64_t sum_size;      /* mean_size = sum_size / M (exact) */
    uint64_t sum_depth;     /* mean_depth = sum_depth / M (exact) */
    double sum_fitness;     /* in slot order, double accumulation (mean_fitness = sum / M) */
} ltgp_gen_stats;

const char* ltgp_last_error(void);
/* Visible CUDA devices (for callers that map workers to GPUs). */
int ltgp_device_count(int* n);
const char* ltgp_version(void);

int ltgp_engine_create(const ltgp_config* cfg, ltgp_engine** out);
int ltgp_engine_destroy(ltgp_engine* e);

/* TestSuite (sextic.hpp:25-31): 48 inputs, 48 targets, 250 constants. */
int ltgp_set_suite(ltgp_engine* e, const float* inputs48, const float* targets48,
                   const float* consts250);

/* Replace the current population by M host genomes (pointer per genome),
   e.g. the ramped_half_and_half output (genome.hpp:66-69). */
int ltgp_upload_population(ltgp_engine* e, uint32_t M, const uint8_t* const* ops,
                           const uint64_t* sizes);

/* Same, from one packed host buffer: genome i at buf + offsets[i]. Offsets
   must be multiples of 16 and buf must hold ceil16(offsets[i]+sizes[i])
   bytes; one host-to-device copy per shard (pinned buf recommended). */
int ltgp_upload_packed(ltgp_engine* e, uint32_t M, const uint8_t* buf, uint64_t buf_bytes,
                       const uint64_t* offsets, const uint64_t* sizes);

/* evaluate_population (evolve.hpp:108-109) + evaluate_individual
   (evolve.hpp:106): eval_batch_raw + fitness + hits + size + depth of every
   slot. out: M records in slot order (may be NULL to keep them on device);
   nodes: sum of sizes (may be NULL). */
int ltgp_evaluate_population(ltgp_engine* e, ltgp_record* out, uint64_t* nodes);

/* evaluate_population plus the 48 per-case outputs of every slot
   (eval_batch_raw's result frame, eval.hpp:73-74) into outs48[M*48]. */
int ltgp_evaluate_outputs(ltgp_engine* e, ltgp_record* out, float* outs48);

/* evaluate_population (evolve.hpp:108-109) on host genomes in one call:
   the packed buffer (same layout rules as ltgp_upload_packed) becomes the
   population and is evaluated while it uploads. The buffer goes over in
   slices (16 MB target, at most 48), each packed on the host first
   (ltgp_pack_host: ~0.63 B per node instead of 1, host threads;
   LTGP_PACK=0 sends the raw bytes); one persistent kernel rebuilds, decodes,
   plans and evaluates every slice as it lands (LTGP_XSLICE=0: per-slice
   launches; also the case under launch-serialising tools). out: M records;
   outs48: per-case outputs or NULL. */
int ltgp_evaluate_packed(ltgp_engine* e, uint32_t M, const uint8_t* buf, uint64_t buf_bytes,
                         const uint64_t* offsets, const uint64_t* sizes, ltgp_record* out,
                         float* outs48);

/* Same work, split in two halves so callers can time the device part
   alone: launch (async) then collect (waits, copies records). */
int ltgp_evaluate_launch(ltgp_engine* e);
int ltgp_evaluate_collect(ltgp_engine* e, ltgp_record* out, uint64_t* nodes);

/* execute_generation (evolve.hpp:111-117): for every plan, crossover
   (genome.hpp:80-84) mum[0,ms) ++ dad[ds,de) ++ mum[me,n) on device, then
   evaluate the child. On success the children become the population
   (double buffering, evolve.hpp:45). The run-ending outcomes leave the
   population unchanged and are reported in *size_limit_hit (0 otherwise):
   2 = MemoryBudgetExceeded, checked first, before anything is built: the
   planned generation bytes (parents plus every child, child sizes from the
   crossover algebra; evolve.hpp:89-93) exceed the budget set with
   ltgp_set_memory_budget; 1 = SizeLimitHit, some child would reach
   node_limit (evolve.hpp:102-104). */
int ltgp_execute_generation(ltgp_engine* e, const ltgp_plan* plans, uint32_t M,
                            ltgp_record* out, int* size_limit_hit);

/* ltgp_execute_generation in two halves, so the caller's host work overlaps
   the device's: launch validates the plans and, on a single-shard
   double-buffered engine, issues the whole generation (one CUDA graph:
   directory, extents, child layout and limit checks, work list, splice,
   evaluation, readback) without waiting; finish waits once and reports
   exactly what ltgp_execute_generation reports. No other call on the engine
   between the two. (Multi-shard and streaming engines run the generation
   inside finish.) */
int ltgp_execute_generation_launch(ltgp_engine* e, const ltgp_plan* plans, uint32_t M);
int ltgp_execute_generation_finish(ltgp_engine* e, ltgp_record* out, int* size_limit_hit);

/* Generation statistics of the current population (after an evaluation or
   execute_generation): no host pass over the records. */
int ltgp_generation_stats(ltgp_engine* e, ltgp_gen_stats* out);

/* RunConfig::streaming_memory (evolve.hpp:45; execute_generation's "in
   streaming mode parents are retired as their last planned use completes",
   evolve.hpp:111-114): on = 1 splices each generation's children, in plan
   order and waves of `wave` children (0 = keep the current, default 256), into
   the parents' own arena by first fit, releasing a parent's bytes after the
   wave of its last planned use. Results are identical to the default
   double-buffered mode (2M); single-shard engines only. */
int ltgp_set_streaming(ltgp_engine* e, int on, uint32_t wave);

/* RunConfig::memory_budget_bytes (evolve.hpp:44): genome bytes a generation
   may plan (parents + children); 0 (the default) disables the check. */
int ltgp_set_memory_budget(ltgp_engine* e, uint64_t bytes);

/* Genome bytes of slot idx (for dumps, to_text, parity). *size is always set. */
int ltgp_download_genome(ltgp_engine* e, uint32_t idx, uint8_t* buf, uint64_t cap,
                         uint64_t* size);

/* eval_batch (eval.hpp:78-79) of one genome: the 48 per-case outputs. */
int ltgp_eval_one(ltgp_engine* e, const uint8_t* ops, uint64_t n, float* out48);

/* ltgp_eval_one plus the individual's record (evaluate_individual,
   evolve.hpp:106: fitness, hits, size, depth computed on the device). */
int ltgp_eval_one_record(ltgp_engine* e, const uint8_t* ops, uint64_t n, float* out48, ltgp_record* rec);

/* subtree_extent (genome.hpp:56-57) of `count` (slot, point) queries on
   device; out holds [start, end) pairs. */
int ltgp_subtree_extents(ltgp_engine* e, uint32_t count, const uint32_t* slots,
                         const uint32_t* points, uint64_t* out_start_end);

int ltgp_get_stats(ltgp_engine* e, ltgp_stats* out);
uint32_t ltgp_population_size(ltgp_engine* e);

/* Device address of the record array of shard s (M_s records, slots
   [first, first + count)) and the CUDA stream it is produced on, for
   callers that run their own collective (e.g. torch.distributed NCCL). */
int ltgp_shard_records(ltgp_engine* e, int s, void** dev_records, uint32_t* first,
                       uint32_t* count, void** stream);

/* One process per GPU (torchrun / bench.py --gpus N): the engine (one shard)
   joins an NCCL communicator across processes and every evaluation
   all-gathers the ranks' 16-byte records (tournament selection needs every
   fitness), over NVLink. ltgp_nccl_unique_id makes the
   communicator id on one rank (128 bytes, to be broadcast by the caller);
   ltgp_nccl_attach joins with it (equal population sizes per rank);
   ltgp_gathered_records returns the last gather: nranks x M records, rank r's
   at r x M (*n = their count; out may be NULL to query it). */
int ltgp_nccl_unique_id(uint8_t* out128);
int ltgp_nccl_attach(ltgp_engine* e, const uint8_t* id128, int nranks, int rank);
int ltgp_gathered_records(ltgp_engine* e, ltgp_record* out, uint32_t cap, uint32_t* n);

/* The packed form a streamed evaluation sends over PCIe (ltgp_pack.h:
   3-bit codes for opcodes 0-4 and 0xFF, literal bytes for the rest), exposed
   for tests and tools. ltgp_pack_bound: the buffer size packing `len` bytes
   may need. ltgp_pack_host packs src[0, len) into dst with `threads` host
   threads and returns the packed size (0 on error). */
uint64_t ltgp_pack_bound(uint64_t len);
uint64_t ltgp_pack_host(const uint8_t* src, uint64_t len, uint8_t* dst, int threads);

#ifdef __cplusplus
}
#endif
#endif
