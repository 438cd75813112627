// ref_run.cpp — TEST HARNESS (test infrastructure, not product): the
// reference's generational loop written against the reference's UNMODIFIED
// headers (/root/reference/proj/include/ltgp/*.hpp, run.hpp:33-36 order:
// ramped init, generation-0 evaluate_population, then plan_generation /
// execute_generation), linked against libltgp_refabi.so, which supplies
// evaluate_population / execute_generation (evolve.hpp:106-117) on the B200
// engine. Writes the determinism dump (stats.hpp:104-107 format) so
// tests/test_refabi.py can compare it with the CPU oracle's run().
//
// The reference declares, but does not define, ramped_half_and_half,
// tournament, plan_generation and make_suite; this harness restates them
// exactly as the oracle does (oracle/ltgp_oracle.cpp: gen_node, ramped,
// tournament, plan_generation; SURVEY App. A #3,
// #4, #7, #10) on the reference's own inline Rng (rng.hpp:9-51), and takes
// the suite from the oracle's make_suite (C ABI).
//
//   ref_run M G node_limit k seed grow_mode dump_path [bind_flags|default]
#include "ltgp/evolve.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ltgp_refabi.h"

extern "C" {
uint64_t orc_suite_seed(uint64_t run_seed);
void orc_make_suite(uint64_t seed, float* inputs48, float* targets48, float* consts250);
}

using namespace ltgp;

namespace {

// oracle gen_node: prefix-order draws (functions below(4), terminals
// 4+below(251); grow below the cap: below(255) in SPEC mode, 50/50 in mode 1)
std::vector<std::uint8_t> gen_tree(Rng& rng, int target, bool full, int grow_mode) {
    std::vector<std::uint8_t> out;
    std::vector<int> todo{1};
    while (!todo.empty()) {
        const int dep = todo.back();
        todo.pop_back();
        std::uint8_t op;
        if (dep >= target) op = static_cast<std::uint8_t>(4 + rng.below(251));
        else if (full) op = static_cast<std::uint8_t>(rng.below(4));
        else if (grow_mode == 0) op = static_cast<std::uint8_t>(rng.below(255));
        else op = rng.below(2) == 0 ? static_cast<std::uint8_t>(rng.below(4)) : static_cast<std::uint8_t>(4 + rng.below(251));
        out.push_back(op);
        if (is_function(op)) {
            todo.push_back(dep + 1);
            todo.push_back(dep + 1);
        }
    }
    return out;
}

std::size_t tournament_(Rng& rng, const std::vector<Individual>& pop, std::uint32_t k) {
    const std::size_t M = pop.size();
    std::size_t best = rng.below(M);
    std::uint64_t ties = 1;
    for (std::uint32_t i = 1; i < k; ++i) {
        const std::size_t idx = rng.below(M);
        if (fitness_better(pop[idx].fitness, pop[best].fitness)) {  // eval.hpp:89-98 (reference inline)
            best = idx;
            ties = 1;
        } else if (fitness_tied(pop[idx].fitness, pop[best].fitness)) {
            if (rng.below(ties + 1) == 0) best = idx;
            ++ties;
        }
    }
    return best;
}

std::vector<CrossoverPlan> plan_(Rng& rng, const std::vector<Individual>& pop, std::uint32_t k) {
    std::vector<CrossoverPlan> plans(pop.size());
    for (auto& p : plans) {
        p.mum_index = static_cast<std::uint32_t>(tournament_(rng, pop, k));
        p.dad_index = static_cast<std::uint32_t>(tournament_(rng, pop, k));
        p.mum_pt = static_cast<std::uint32_t>(rng.below(pop[p.mum_index].size));  // Individual::size (App. A #10)
        p.dad_pt = static_cast<std::uint32_t>(rng.below(pop[p.dad_index].size));
    }
    return plans;
}

void dump(std::FILE* f, std::uint32_t gen, const std::vector<Individual>& pop) {
    for (std::size_t i = 0; i < pop.size(); ++i) {
        std::uint32_t bits;
        std::memcpy(&bits, &pop[i].fitness, 4);
        if (std::isnan(pop[i].fitness)) bits = 0x7fc00000u;
        std::fprintf(f, "%u %zu %u %u %d %08x\n", gen, i, pop[i].size, pop[i].depth, pop[i].hits, bits);
    }
}

}  // namespace

// `ref_run eval SEED COUNT`: evaluate_individual (evolve.hpp:106) and
// eval_batch_raw / eval_batch (eval.hpp:73-79) on COUNT random genomes of the
// suite of SEED; prints per genome: fitness bits, hits, size, depth, then the
// 48 eval_batch_raw output bits, then whether eval_batch matched them; next
// line: '#' + the genome in hex (the test re-evaluates it with the oracle).
static int eval_mode(std::uint64_t seed, int count) {
    TestSuite suite;
    orc_make_suite(orc_suite_seed(seed), suite.inputs.data(), suite.targets.data(), suite.constants.data());
    Rng rng(seed * 7919 + 1);
    WorkerState worker;
    EvalStack stack;
    GpopsCounter counter;
    for (int g = 0; g < count; ++g) {
        Individual ind;
        ind.genome = Genome(gen_tree(rng, 2 + g % 7, g % 2 == 0, 1));
        evaluate_individual(ind, suite, worker);
        const float* raw = eval_batch_raw(ind.genome, suite.inputs.data(), suite.constants, stack, &counter);
        float out[kLaneWidth];  // the raw frame is valid only until the stack's next use
        std::memcpy(out, raw, sizeof out);
        std::uint32_t fb;
        std::memcpy(&fb, &ind.fitness, 4);
        std::printf("%zu %08x %d %u %u", ind.genome.size(), fb, ind.hits, ind.size, ind.depth);
        for (std::size_t l = 0; l < kLaneWidth; ++l) {
            std::uint32_t b;
            std::memcpy(&b, out + l, 4);
            std::printf(" %08x", b);
        }
        LaneResult in;
        std::copy(suite.inputs.begin(), suite.inputs.end(), in.begin());
        const LaneResult r = eval_batch(ind.genome, in, suite.constants, stack, nullptr);
        const bool same = std::memcmp(r.data(), out, sizeof out) == 0;
        std::printf(" %d\n", same ? 1 : 0);
        std::printf("#");  // the genome, hex, for the test's oracle check
        for (std::size_t k = 0; k < ind.genome.size(); ++k) std::printf("%02x", (unsigned)ind.genome[k]);
        std::printf("\n");
    }
    std::printf("counter %llu %.9f peak %zu\n", (unsigned long long)counter.nodes_evaluated, counter.elapsed_seconds,
                stack.peak_frames());
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 4 && std::string(argv[1]) == "eval") {
        try {
            return eval_mode(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]));
        } catch (const std::exception& ex) {
            std::fprintf(stderr, "error: %s\n", ex.what());
            return 6;
        }
    }
    if (argc < 8) {
        std::fprintf(stderr, "usage: ref_run M G node_limit k seed grow_mode dump [bind_flags|default]\n");
        return 2;
    }
    RunConfig cfg;
    cfg.population_size = static_cast<std::uint32_t>(std::strtoul(argv[1], nullptr, 10));
    cfg.max_generations = static_cast<std::uint32_t>(std::strtoul(argv[2], nullptr, 10));
    cfg.node_limit = std::strtoull(argv[3], nullptr, 10);
    cfg.tournament_size = static_cast<std::uint32_t>(std::strtoul(argv[4], nullptr, 10));
    cfg.seed = std::strtoull(argv[5], nullptr, 10);
    const int grow_mode = std::atoi(argv[6]);
    const std::string mode = argc > 8 ? argv[8] : "0";
    TestSuite suite;
    orc_make_suite(orc_suite_seed(cfg.seed), suite.inputs.data(), suite.targets.data(), suite.constants.data());
    std::vector<WorkerState> pool(1);
    MemoryGauge gauge;
    ExecContext ctx{suite, cfg, pool, gauge};
    ltgp_engine* e = nullptr;
    if (mode != "default") {  // bind our own engine (else the adapter creates one on first use)
        ltgp_config ec{};
        ec.n_shards = 1;
        ec.node_limit = cfg.node_limit;
        if (ltgp_engine_create(&ec, &e) != 0 || ltgp_ref_bind_engine(&pool, e, std::atoi(mode.c_str())) != 0) {
            std::fprintf(stderr, "engine: %s\n", ltgp_last_error());
            return 3;
        }
    }
    std::FILE* f = std::fopen(argv[7], "w");
    if (!f) return 4;
    try {
        Rng rng(cfg.seed);
        std::vector<Individual> pop(cfg.population_size), next;
        for (std::uint32_t i = 0; i < cfg.population_size; ++i) {  // App. A #3: depth 2 + (i/2) % 5, even full
            const int d = 2 + static_cast<int>((i / 2) % 5);
            pop[i].genome = Genome(gen_tree(rng, d, i % 2 == 0, grow_mode));
        }
        gauge.add(cfg.population_size);
        evaluate_population(pop, ctx);
        dump(f, 0, pop);
        std::uint32_t gen = 1;
        int reason = 0;
        for (; gen <= cfg.max_generations; ++gen) {
            const auto plans = plan_(rng, pop, cfg.tournament_size);
            const ExecOutcome o = execute_generation(plans, pop, next, ctx);
            if (o.size_limit_hit) { reason = 1; break; }
            std::swap(pop, next);
            gauge.sub(cfg.population_size);  // the parents are retired
            dump(f, gen, pop);
            if (mode == "1")  // materialized children: the host genomes match the sizes
                for (const auto& ind : pop)
                    if (ind.genome.size() != ind.size) {
                        std::fprintf(stderr, "materialized genome mismatch\n");
                        return 5;
                    }
        }
        std::fclose(f);
        std::printf("generations %u reason %d nodes %llu elapsed %.6f live %lld high %lld\n", gen - 1, reason,
                    (unsigned long long)pool[0].counter.nodes_evaluated, pool[0].counter.elapsed_seconds,
                    (long long)gauge.live(), (long long)gauge.high_water());
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "error: %s\n", ex.what());
        return 6;
    }
    if (e) {
        ltgp_ref_unbind(&pool);
        ltgp_engine_destroy(e);
    }
    return 0;
}
