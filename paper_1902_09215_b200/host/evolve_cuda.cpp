// evolve_cuda.cpp — libltgp_refabi.so: the B200 engine behind the reference's
// OWN declarations, compiled against its unmodified headers
// (/root/reference/proj/include/ltgp/evolve.hpp, eval.hpp; see
// include/ltgp_refabi.h and INTEGRATION.md).
//
// Definitions provided (everything else of the reference API is the
// caller's, unchanged):
//   evaluate_population  evolve.hpp:108-109  upload + device evaluation
//   execute_generation   evolve.hpp:111-117  device extents, splice, evaluation
//   evaluate_individual  evolve.hpp:106      one genome on a per-thread engine
//   eval_batch_raw       eval.hpp:73-74      48 per-case outputs into the EvalStack
//   eval_batch           eval.hpp:78-79
//   EvalStack::reserve_frames / grow         eval.hpp:34-40 (host frame storage)
// Every node is evaluated on the GPU through the C ABI (ltgp_cuda.h); this
// file holds no arithmetic of the path.
//
// Engine lookup: ExecContext (evolve.hpp:95-100) carries no engine, so the
// engine is keyed by the address of ExecContext::pool, the caller's worker
// pool, which lives for the whole run (ltgp_ref_bind_engine; otherwise one is
// created on first use). The engine keeps the population device-resident:
// after evaluate_population(pop) or execute_generation(..., children) it
// remembers which vector it holds (buffer address and size). A later
// execute_generation whose `parents` is that vector (the caller's swap of
// parents and children swaps the buffers) splices on the device; any other
// parents vector is uploaded from its host genomes first.
//
// Error conventions: engine failures throw
// std::runtime_error, bad arguments std::invalid_argument; SizeLimitHit is
// the ExecOutcome value, not an error.
#include "ltgp/eval.hpp"
#include "ltgp/evolve.hpp"

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "ltgp_refabi.h"

static_assert(sizeof(ltgp::CrossoverPlan) == sizeof(ltgp_plan), "CrossoverPlan and ltgp_plan differ");
static_assert(offsetof(ltgp::CrossoverPlan, mum_index) == offsetof(ltgp_plan, mum_index) &&
                  offsetof(ltgp::CrossoverPlan, dad_index) == offsetof(ltgp_plan, dad_index) &&
                  offsetof(ltgp::CrossoverPlan, mum_pt) == offsetof(ltgp_plan, mum_pt) &&
                  offsetof(ltgp::CrossoverPlan, dad_pt) == offsetof(ltgp_plan, dad_pt),
              "CrossoverPlan field layout");
static_assert(ltgp::kLaneWidth == LTGP_LANES && ltgp::kConstantCount == LTGP_CONSTANTS, "lane / constant counts");

namespace {

void check(int status) {
    if (status != 0) throw std::runtime_error(std::string("ltgp engine: ") + ltgp_last_error());
}

struct Binding {
    ltgp_engine* e = nullptr;
    bool owned = false;
    int flags = 0;
    const void* resident = nullptr;  // data() of the vector whose genomes the engine holds
    std::size_t resident_n = 0;
    ~Binding() {
        if (owned && e) ltgp_engine_destroy(e);
    }
};

std::mutex g_mu;
std::map<const void*, std::unique_ptr<Binding>>& registry() {
    static auto* r = new std::map<const void*, std::unique_ptr<Binding>>();  // outlives static teardown
    return *r;
}

// The binding of this context's worker pool; created with a default engine
// on first use (one shard per RunConfig::worker_count, round robin over the
// visible GPUs: the reference's workers become GPUs).
Binding& binding(const ltgp::ExecContext& ctx) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = registry()[static_cast<const void*>(&ctx.pool)];
    if (!slot) {
        slot = std::make_unique<Binding>();
        ltgp_config cfg{};
        int ndev = 0;
        check(ltgp_device_count(&ndev));
        if (ndev == 0) throw std::runtime_error(std::string("ltgp engine: no usable GPU: ") + ltgp_last_error());
        const std::uint32_t w = std::max<std::uint32_t>(1, std::min<std::uint32_t>(ctx.config.worker_count, LTGP_MAX_SHARDS));
        cfg.n_shards = static_cast<int>(w);
        for (std::uint32_t i = 0; i < w; ++i) cfg.devices[i] = static_cast<int>(i % static_cast<std::uint32_t>(ndev));
        cfg.node_limit = ctx.config.node_limit;
        cfg.use_nccl = 1;
        check(ltgp_engine_create(&cfg, &slot->e));
        slot->owned = true;
    }
    return *slot;
}

void set_suite(ltgp_engine* e, const ltgp::TestSuite& suite) {
    check(ltgp_set_suite(e, suite.inputs.data(), suite.targets.data(), suite.constants.data()));
}

void account(ltgp::ExecContext& ctx, ltgp_engine* e, std::uint64_t nodes) {
    if (ctx.pool.empty()) return;
    ltgp_stats st{};
    check(ltgp_get_stats(e, &st));
    ctx.pool[0].counter.nodes_evaluated += nodes;  // GpopsCounter (eval.hpp:14-25)
    ctx.pool[0].counter.elapsed_seconds += st.eval_seconds;
}

// A per-thread one-shard engine for the single-genome entry points
// (evaluate_individual, eval_batch_raw): they take no ExecContext.
ltgp_engine* thread_engine() {
    struct Holder {
        ltgp_engine* e = nullptr;
        ~Holder() {
            if (e) ltgp_engine_destroy(e);
        }
    };
    thread_local Holder h;
    if (!h.e) {
        ltgp_config cfg{};
        cfg.n_shards = 1;
        cfg.devices[0] = 0;
        cfg.node_limit = ~0ull;
        check(ltgp_engine_create(&cfg, &h.e));
    }
    return h.e;
}

void fill(ltgp::Individual& ind, const ltgp_record& r) {
    ind.fitness = r.fitness;
    ind.hits = r.hits;
    ind.size = r.size;
    ind.depth = r.depth;
}

}  // namespace

extern "C" {

int ltgp_ref_bind_engine(const void* pool_key, ltgp_engine* e, int flags) {
    if (!pool_key || !e) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    auto b = std::make_unique<Binding>();
    b->e = e;
    b->flags = flags;
    registry()[pool_key] = std::move(b);
    return 0;
}

int ltgp_ref_unbind(const void* pool_key) {
    std::lock_guard<std::mutex> lk(g_mu);
    registry().erase(pool_key);
    return 0;
}

ltgp_engine* ltgp_ref_engine(const void* pool_key) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = registry().find(pool_key);
    return it == registry().end() ? nullptr : it->second->e;
}

}  // extern "C"

namespace ltgp {

// evolve.hpp:108-109 — every slot's eval_batch_raw + fitness + hits + size +
// depth (evaluate_individual, evolve.hpp:106), on the device.
void evaluate_population(std::vector<Individual>& population, ExecContext ctx) {
    Binding& b = binding(ctx);
    const std::size_t M = population.size();
    if (M == 0) return;
    if (M > 0xffffffffull) throw std::invalid_argument("evaluate_population: population too large");
    std::vector<const std::uint8_t*> ptrs(M);
    std::vector<std::uint64_t> sizes(M);
    for (std::size_t i = 0; i < M; ++i) {
        if (population[i].genome.empty()) throw std::invalid_argument("evaluate_population: empty genome");
        ptrs[i] = population[i].genome.data();
        sizes[i] = population[i].genome.size();
    }
    set_suite(b.e, ctx.suite);
    check(ltgp_upload_population(b.e, static_cast<std::uint32_t>(M), ptrs.data(), sizes.data()));
    std::vector<ltgp_record> rec(M);
    std::uint64_t nodes = 0;
    check(ltgp_evaluate_population(b.e, rec.data(), &nodes));
    for (std::size_t i = 0; i < M; ++i) fill(population[i], rec[i]);
    b.resident = population.data();
    b.resident_n = M;
    account(ctx, b.e, nodes);
}

// evolve.hpp:111-117 — per plan crossover(mum, dad, mum_pt, dad_pt,
// node_limit) (genome.hpp:80-84) then evaluation, every child on the device.
// size_limit_hit: some child would reach node_limit; nothing is built and
// `children` is left as it was (genome.hpp:71-74).
ExecOutcome execute_generation(std::span<const CrossoverPlan> plans, std::vector<Individual>& parents,
                               std::vector<Individual>& children, ExecContext ctx) {
    Binding& b = binding(ctx);
    const std::size_t M = plans.size();
    ExecOutcome out;
    if (M == 0) {
        children.clear();
        return out;
    }
    if (M != parents.size()) throw std::invalid_argument("execute_generation: one plan per parent slot expected");
    if (b.resident != parents.data() || b.resident_n != parents.size()) {
        // the engine holds another population: upload these parents
        std::vector<const std::uint8_t*> ptrs(parents.size());
        std::vector<std::uint64_t> sizes(parents.size());
        for (std::size_t i = 0; i < parents.size(); ++i) {
            if (parents[i].genome.empty())
                throw std::invalid_argument("execute_generation: parents are neither device-resident nor on the host");
            ptrs[i] = parents[i].genome.data();
            sizes[i] = parents[i].genome.size();
        }
        check(ltgp_upload_population(b.e, static_cast<std::uint32_t>(parents.size()), ptrs.data(), sizes.data()));
    }
    set_suite(b.e, ctx.suite);
    if (ctx.config.streaming_memory) check(ltgp_set_streaming(b.e, 1, 0));  // evolve.hpp:45, :111-114
    std::vector<ltgp_record> rec(M);
    int flag = 0;
    check(ltgp_execute_generation(b.e, reinterpret_cast<const ltgp_plan*>(plans.data()),
                                  static_cast<std::uint32_t>(M), rec.data(), &flag));
    if (flag == 1) {
        out.size_limit_hit = true;
        return out;
    }
    if (flag != 0) throw std::runtime_error("execute_generation: unexpected engine outcome");
    children.resize(M);
    std::uint64_t nodes = 0;
    for (std::size_t i = 0; i < M; ++i) {
        fill(children[i], rec[i]);
        nodes += rec[i].size;
        if (b.flags & LTGP_REF_MATERIALIZE_GENOMES) {
            std::vector<std::uint8_t> g(rec[i].size);
            std::uint64_t n = 0;
            check(ltgp_download_genome(b.e, static_cast<std::uint32_t>(i), g.data(), g.size(), &n));
            children[i].genome = Genome(std::move(g));
        } else {
            children[i].genome.release();
        }
    }
    ctx.gauge.add(static_cast<std::int64_t>(M));  // the children are live genomes
    b.resident = children.data();
    b.resident_n = M;
    account(ctx, b.e, nodes);
    return out;
}

// evolve.hpp:106 — one individual (gen-0 style), on this thread's engine.
void evaluate_individual(Individual& ind, const TestSuite& suite, WorkerState& worker) {
    if (ind.genome.empty()) throw std::invalid_argument("evaluate_individual: empty genome");
    ltgp_engine* e = thread_engine();
    set_suite(e, suite);
    float out[kLaneWidth];
    ltgp_record r{};
    check(ltgp_eval_one_record(e, ind.genome.data(), ind.genome.size(), out, &r));
    fill(ind, r);
    ltgp_stats st{};
    check(ltgp_get_stats(e, &st));
    worker.counter.nodes_evaluated += ind.genome.size();
    worker.counter.elapsed_seconds += st.eval_seconds;
}

// eval.hpp:73-74 — the 48 per-case outputs of g for these inputs and
// constants, written to frame 0 of `stack` (valid until the stack's next use).
const float* eval_batch_raw(const Genome& g, const float* inputs, std::span<const float> constants,
                            EvalStack& stack, GpopsCounter* counter) {
    if (g.empty()) throw std::invalid_argument("eval_batch_raw: empty genome");
    if (constants.size() != static_cast<std::size_t>(kConstantCount))
        throw std::invalid_argument("eval_batch_raw: the constant table has 250 entries");
    if (stack.frame_capacity() < 1) stack.reserve_frames(1);
    ltgp_engine* e = thread_engine();
    static const float zeros[kLaneWidth] = {};
    check(ltgp_set_suite(e, inputs, zeros, constants.data()));
    check(ltgp_eval_one(e, g.data(), g.size(), stack.data()));
    stack.note_frames(1);
    if (counter) {
        ltgp_stats st{};
        check(ltgp_get_stats(e, &st));
        counter->nodes_evaluated += g.size();
        counter->elapsed_seconds += st.eval_seconds;
    }
    return stack.data();
}

// eval.hpp:78-79
LaneResult eval_batch(const Genome& g, const LaneResult& inputs, std::span<const float> constants,
                      EvalStack& stack, GpopsCounter* counter) {
    const float* r = eval_batch_raw(g, inputs.data(), constants, stack, counter);
    LaneResult out;
    std::memcpy(out.data(), r, sizeof(float) * kLaneWidth);
    return out;
}

// eval.hpp:34-40 — host frame storage of the EvalStack (the device keeps its
// own stacks; the host stack receives the result frame).
void EvalStack::reserve_frames(std::size_t frames) {
    if (frames <= frames_ && data_) return;
    data_ = alloc_lane_frames(frames);
    frames_ = frames;
}

void EvalStack::grow(std::size_t live, std::size_t min_frames) {
    if (min_frames <= frames_ && data_) return;
    if (live > frames_) throw std::invalid_argument("EvalStack::grow: more live frames than capacity");
    AlignedFloats fresh = alloc_lane_frames(min_frames);
    if (live) std::memcpy(fresh.get(), data_.get(), live * kLaneWidth * sizeof(float));
    data_ = std::move(fresh);
    frames_ = min_frames;
}

}  // namespace ltgp
