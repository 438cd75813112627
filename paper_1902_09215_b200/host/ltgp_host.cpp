// ltgp_host.cpp — libltgp_host.so: the reference's host-side population API
// (ltgp/ltgp.hpp) on top of the B200 engine (include/ltgp_cuda.h).
//
// Everything here is the *caller* side of the hot path that the reference
// keeps sequential on the host: the RNG stream, tree
// construction, tournament selection and crossover planning. Evaluation and
// splicing go through the C ABI to the GPU.

#include "ltgp/ltgp.hpp"

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <random>
#include <sstream>
#include <thread>

#include <unistd.h>

#include "../../include/ltgp_host.h"

namespace ltgp {

void check(int status) {
    if (status != 0) throw std::runtime_error(std::string("ltgp engine: ") + ltgp_last_error());
}

// sextic.hpp:33-35: y = x*x*(x-1)*(x-1)*(x+1)*(x+1), left to right, float.
float target(float x) {
    float y = x * x;
    y *= (x - 1.0f);
    y *= (x - 1.0f);
    y *= (x + 1.0f);
    y *= (x + 1.0f);
    return y;
}

namespace {
// sextic.hpp:37-40: 9 significant digits (lossless for float).
float canonical(float v) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%.9g", static_cast<double>(v));
    return std::strtof(buf, nullptr);
}
}  // namespace

// sextic.hpp:42-51: 48 cases first (x, y after the text round trip), then
// 250 distinct millesimal-grid constants by partial Fisher-Yates
// (below(2001 - j)), each parsed from its 3-decimal text, sorted.
TestSuite make_suite(Rng& rng) {
    TestSuite s;
    for (std::size_t l = 0; l < kLaneWidth; ++l) {
        const float x = canonical(rng.uniform_pm1());
        s.inputs[l] = x;
        s.targets[l] = canonical(target(x));
    }
    int grid[2001];
    for (int k = 0; k < 2001; ++k) grid[k] = k;
    for (int j = 0; j < kConstantCount; ++j) {
        const auto k = static_cast<std::size_t>(j) + rng.below(static_cast<std::uint64_t>(2001 - j));
        std::swap(grid[j], grid[k]);
    }
    for (int j = 0; j < kConstantCount; ++j) {
        const int m = grid[j] - 1000;
        char buf[32];
        std::snprintf(buf, sizeof buf, "%s%d.%03d", m < 0 ? "-" : "", std::abs(m) / 1000, std::abs(m) % 1000);
        s.constants[j] = std::strtof(buf, nullptr);
    }
    std::sort(s.constants, s.constants + kConstantCount);
    return s;
}

TestSuite make_suite(std::uint64_t seed) {
    Rng rng(seed);
    return make_suite(rng);
}

std::uint64_t suite_seed(std::uint64_t run_seed) { return splitmix64(run_seed ^ 0x53554954ull); }

namespace {
// Prefix-order construction shared by gen_full / gen_grow (genome.hpp:59-64,
// SPEC.md:72-89): function draws below(4), terminal draws 4+below(251), a
// grow node above the cap draws below(255) (one draw per opcode) with
// GrowMode::kUniformPrimitive, or below(2) function-vs-
// terminal first with GrowMode::kHalfFunctions (the alternative SPEC.md:148
// leaves open; GPquick-style, and the one whose runs bloat like the paper's).
Genome build(Rng& rng, int cap_depth, bool full, std::size_t capacity, GrowMode mode) {
    std::vector<std::uint8_t> ops;
    std::vector<int> todo{1};
    while (!todo.empty()) {
        const int d = todo.back();
        todo.pop_back();
        std::uint8_t op;
        if (d >= cap_depth) op = static_cast<std::uint8_t>(4 + rng.below(251));
        else if (full) op = static_cast<std::uint8_t>(rng.below(4));
        else if (mode == GrowMode::kUniformPrimitive) op = static_cast<std::uint8_t>(rng.below(255));
        else op = rng.below(2) == 0 ? static_cast<std::uint8_t>(rng.below(4))
                                    : static_cast<std::uint8_t>(4 + rng.below(251));
        ops.push_back(op);
        if (ops.size() > capacity) throw std::length_error("tree exceeds capacity");
        if (is_function(op)) {
            todo.push_back(d + 1);
            todo.push_back(d + 1);
        }
    }
    return Genome(std::move(ops));
}
}  // namespace

Genome gen_full(Rng& rng, int target_depth, std::size_t capacity) {
    if (target_depth < 1) throw std::invalid_argument("depth < 1");
    if (target_depth >= 64 || ((std::size_t{1} << target_depth) - 1) > capacity)
        throw std::length_error("full tree exceeds capacity");
    return build(rng, target_depth, true, capacity, GrowMode::kUniformPrimitive);
}

Genome gen_grow(Rng& rng, int max_depth, std::size_t capacity, GrowMode mode) {
    if (max_depth < 1) throw std::invalid_argument("depth < 1");
    return build(rng, max_depth, false, capacity, mode);
}

// genome.hpp:66-69: depth dmin + (i/2) % span, even i
// full, odd i grow.
std::vector<Genome> ramped_half_and_half(Rng& rng, std::size_t count, std::size_t capacity,
                                         int min_depth, int max_depth, GrowMode mode) {
    std::vector<Genome> out;
    out.reserve(count);
    const std::size_t span = static_cast<std::size_t>(max_depth - min_depth + 1);
    for (std::size_t i = 0; i < count; ++i) {
        const int d = min_depth + static_cast<int>((i / 2) % span);
        out.push_back((i % 2 == 0) ? gen_full(rng, d, capacity) : gen_grow(rng, d, capacity, mode));
    }
    return out;
}

// bench.hpp:13-15: at a function node draw the opcode
// below(4), then the left size uniform over odd values in [1, n-2]; a leaf
// is X or a constant 5+below(250) with equal probability (below(2)).
void random_tree_of_size(Rng& rng, std::size_t n, std::uint8_t* out) {
    if (n == 0 || n % 2 == 0) throw std::invalid_argument("tree size must be odd");
    std::vector<std::uint64_t> todo{n};
    std::size_t pos = 0;
    while (!todo.empty()) {
        const std::uint64_t m = todo.back();
        todo.pop_back();
        if (m == 1) {
            out[pos++] = rng.below(2) == 0 ? kOpX : static_cast<std::uint8_t>(kOpFirstConstant + rng.below(250));
            continue;
        }
        out[pos++] = static_cast<std::uint8_t>(rng.below(4));
        const std::uint64_t left = 2 * rng.below((m - 1) / 2) + 1;
        todo.push_back(m - 1 - left);
        todo.push_back(left);
    }
}

Genome random_tree_of_size(Rng& rng, std::size_t n) {
    std::vector<std::uint8_t> ops(n);
    random_tree_of_size(rng, n, ops.data());
    return Genome(std::move(ops));
}

void validate(const RunConfig& c) {
    if (c.population_size < 2) throw std::invalid_argument("population_size < 2");
    if (c.node_limit < 63) throw std::invalid_argument("node_limit < 63");
    if (c.tournament_size < 1) throw std::invalid_argument("tournament_size < 1");
}

namespace {
// evolve.hpp:79-82 over any fitness accessor: the
// reference's draws and comparisons
template <class Fit>
std::size_t tournament_by(Rng& rng, std::uint64_t M, std::uint32_t k, Fit fit) {
    std::size_t best = static_cast<std::size_t>(rng.below(M));
    std::uint64_t ties = 1;
    for (std::uint32_t i = 1; i < k; ++i) {
        const std::size_t idx = static_cast<std::size_t>(rng.below(M));
        if (fitness_better(fit(idx), fit(best))) {
            best = idx;
            ties = 1;
        } else if (fitness_tied(fit(idx), fit(best))) {
            if (rng.below(ties + 1) == 0) best = idx;
            ++ties;
        }
    }
    return best;
}
}  // namespace

// evolve.hpp:79-82
std::size_t tournament(Rng& rng, std::span<const Individual> pop, std::uint32_t k) {
    return tournament_by(rng, pop.size(), k, [&](std::size_t i) { return pop[i].fitness; });
}

// Mt64's twist + tempering, vectorised per host ISA: the draws that bound
// plan_generation cost 2.7 ns each with SSE2 and 1.2 ns with AVX2 on a Xeon
// host (64K draws per 4000-child generation). Same outputs on every clone.
// Out of place: dst.x[k] from src.x[k], src.x[k+1] and x[k+M] (src's for
// k < N-M, already twisted dst's after).
__attribute__((target_clones("avx512f", "avx2", "default")))
void Mt64::twist(const Block& src, Block& dst) {
    constexpr std::uint64_t kUM = ~0ull << 31, kLM = ~kUM, kA = 0xb5026f5aa96619e9ull;
    const std::uint64_t* x = src.x;
    std::uint64_t* y = dst.x;
    for (int k = 0; k < kN - kM; ++k) {
        const std::uint64_t v = (x[k] & kUM) | (x[k + 1] & kLM);
        y[k] = x[k + kM] ^ (v >> 1) ^ ((0 - (v & 1)) & kA);
    }
    for (int k = kN - kM; k < kN - 1; ++k) {
        const std::uint64_t v = (x[k] & kUM) | (x[k + 1] & kLM);
        y[k] = y[k + kM - kN] ^ (v >> 1) ^ ((0 - (v & 1)) & kA);
    }
    const std::uint64_t v = (x[kN - 1] & kUM) | (y[0] & kLM);
    y[kN - 1] = y[kM - 1] ^ (v >> 1) ^ ((0 - (v & 1)) & kA);
    for (int i = 0; i < kN; ++i) {
        std::uint64_t z = y[i];
        z ^= (z >> 29) & 0x5555555555555555ull;
        z ^= (z << 17) & 0x71d67fffeda60000ull;
        z ^= (z << 37) & 0xfff7eee000000000ull;
        z ^= z >> 43;
        dst.out[i] = z;
    }
}

// evolve.hpp:84-87. The tournaments read fitness from a
// dense copy (4 B per individual, L1-resident) instead of the 40-byte
// Individuals; the draws and comparisons are unchanged.
// Selection key: an unsigned total order equal to fitness_better /
// fitness_tied (eval.hpp:89-98): lower is better, every NaN is the worst and
// ties every NaN, -0 ties +0. Comparing keys is branch-free, so a tournament
// costs its RNG draws, not a mispredicted branch per entrant.
static inline std::uint32_t selection_key(float f) {
    if (f != f) return 0xffffffffu;
    if (f == 0.0f) f = 0.0f;  // -0 ties +0
    std::uint32_t b;
    std::memcpy(&b, &f, 4);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// tournament (evolve.hpp:79-82) on selection keys: the same draws and the
// same winner as tournament_by(fitness_better, fitness_tied). The running
// best is one packed (key << 32 | index) word, so "better" is an unsigned
// min (a cmov). A tie keeps its branch: its draw moves the stream position,
// and a branch-free conditional increment puts every later draw's load
// behind the comparison chain (measured 1.3-3x slower than predicting, even
// on evolved populations where ~3 of 4 entrants tie).
static inline std::size_t tournament_keys(Rng::Cursor& rng, std::uint64_t M, std::uint32_t k, const std::uint32_t* key) {
    const std::uint64_t b0 = rng.below(M);
    std::uint64_t pb = (std::uint64_t)key[b0] << 32 | b0;
    std::uint64_t ties = 1;
    for (std::uint32_t i = 1; i < k; ++i) {
        const std::uint64_t idx = rng.below(M);
        const std::uint64_t pk = (std::uint64_t)key[idx] << 32 | idx;
        if ((pk >> 32) == (pb >> 32)) [[unlikely]] {  // tie: replace with probability 1/(ties + 1)
            if (rng.below(ties + 1) == 0) pb = pk;
            ++ties;
            continue;
        }
        ties = pk < pb ? 1 : ties;
        pb = pk < pb ? pk : pb;
    }
    return static_cast<std::size_t>(pb & 0xffffffffu);
}

std::vector<CrossoverPlan> plan_generation(Rng& rng, std::span<const Individual> pop, std::uint32_t k) {
    // dense keys and sizes: the tournaments' random reads stay in L1
    std::vector<std::uint32_t> key(pop.size()), size(pop.size());
    for (std::size_t i = 0; i < pop.size(); ++i) {
        key[i] = selection_key(pop[i].fitness);
        size[i] = pop[i].size;
    }
    std::vector<CrossoverPlan> plans(pop.size());
    Rng::Cursor cur(rng);
    for (auto& p : plans) {
        p.mum_index = static_cast<std::uint32_t>(tournament_keys(cur, pop.size(), k, key.data()));
        p.dad_index = static_cast<std::uint32_t>(tournament_keys(cur, pop.size(), k, key.data()));
        p.mum_pt = static_cast<std::uint32_t>(cur.below(size[p.mum_index]));
        p.dad_pt = static_cast<std::uint32_t>(cur.below(size[p.dad_index]));
    }
    return plans;
}

namespace {
void fill(Individual& ind, const ltgp_record& r) {
    ind.fitness = r.fitness;
    ind.hits = r.hits;
    ind.size = r.size;
    ind.depth = r.depth;
}
}  // namespace

// evolve.hpp:108-109 on the engine: upload host genomes, evaluate every slot.
void evaluate_population(std::vector<Individual>& population, ExecContext ctx) {
    if (!ctx.engine) throw std::invalid_argument("ExecContext.engine is null");
    check(ltgp_set_suite(ctx.engine, ctx.suite.inputs, ctx.suite.targets, ctx.suite.constants));
    std::vector<const std::uint8_t*> ptrs(population.size());
    std::vector<std::uint64_t> sizes(population.size());
    for (std::size_t i = 0; i < population.size(); ++i) {
        ptrs[i] = population[i].genome.data();
        sizes[i] = population[i].genome.size();
    }
    check(ltgp_upload_population(ctx.engine, static_cast<std::uint32_t>(population.size()), ptrs.data(),
                                 sizes.data()));
    std::vector<ltgp_record> rec(population.size());
    check(ltgp_evaluate_population(ctx.engine, rec.data(), nullptr));
    for (std::size_t i = 0; i < population.size(); ++i) fill(population[i], rec[i]);
}

// evolve.hpp:111-117 on the engine. `parents` must be the engine's current
// population (from evaluate_population or a previous execute_generation).
// execute_generation in two halves (ltgp_execute_generation_launch /
// _finish): the run loop twists the next generation's Rng blocks in between.
static void execute_generation_begin(std::span<const CrossoverPlan> plans, const std::vector<Individual>& parents,
                                     const ExecContext& ctx) {
    if (!ctx.engine) throw std::invalid_argument("ExecContext.engine is null");
    if (plans.size() != parents.size()) throw std::invalid_argument("one plan per child slot");
    check(ltgp_set_memory_budget(ctx.engine, ctx.config.memory_budget_bytes));
    if (ctx.config.streaming_memory) check(ltgp_set_streaming(ctx.engine, 1, 0));  // evolve.hpp:45
    check(ltgp_execute_generation_launch(ctx.engine, plans.data(), static_cast<std::uint32_t>(plans.size())));
}

static ExecOutcome execute_generation_end(std::span<const CrossoverPlan> plans, std::vector<Individual>& parents,
                                          std::vector<Individual>& children, ExecContext ctx) {
    std::vector<ltgp_record> rec(plans.size());
    int hit = 0;
    check(ltgp_execute_generation_finish(ctx.engine, rec.data(), &hit));
    if (hit == 2) return ExecOutcome{false, true};  // MemoryBudgetExceeded: nothing was built
    if (hit) return ExecOutcome{true, false};
    children.resize(plans.size());
    for (std::size_t i = 0; i < plans.size(); ++i) {
        children[i].genome.release();  // device resident (ltgp_download_genome)
        fill(children[i], rec[i]);
    }
    ctx.gauge.add(static_cast<std::int64_t>(plans.size()));
    ctx.gauge.sub(static_cast<std::int64_t>(parents.size()));
    return ExecOutcome{false, false};
}

ExecOutcome execute_generation(std::span<const CrossoverPlan> plans, std::vector<Individual>& parents,
                               std::vector<Individual>& children, ExecContext ctx) {
    execute_generation_begin(plans, parents, ctx);
    return execute_generation_end(plans, parents, children, ctx);
}

namespace {
struct EngineHandle {  // RAII over ltgp_engine_create / destroy
    ltgp_engine* e = nullptr;
    explicit EngineHandle(std::uint32_t gpus) {
        ltgp_config cfg{};
        cfg.n_shards = static_cast<int>(gpus);
        for (std::uint32_t i = 0; i < gpus; ++i) cfg.devices[i] = static_cast<int>(i);
        cfg.node_limit = std::numeric_limits<std::uint64_t>::max();
        cfg.use_nccl = 1;
        check(ltgp_engine_create(&cfg, &e));
    }
    ~EngineHandle() { ltgp_engine_destroy(e); }
    EngineHandle(const EngineHandle&) = delete;
    EngineHandle& operator=(const EngineHandle&) = delete;
};

// Best-of-`repeats` device throughput of one corpus on `gpus` GPUs; sets
// `consistent` if the engine's node counter moved by the corpus size each time.
double corpus_gpops(std::uint32_t gpus, const TestSuite& suite, const std::vector<std::uint8_t>& buf,
                    const std::vector<std::uint64_t>& offs, const std::vector<std::uint64_t>& sizes,
                    std::uint64_t nodes, int repeats, bool& consistent) {
    EngineHandle h(gpus);
    check(ltgp_set_suite(h.e, suite.inputs, suite.targets, suite.constants));
    const auto M = static_cast<std::uint32_t>(sizes.size());
    check(ltgp_upload_packed(h.e, M, buf.data(), buf.size(), offs.data(), sizes.data()));
    std::vector<ltgp_record> rec(M);
    check(ltgp_evaluate_population(h.e, rec.data(), nullptr));  // warm-up
    double best = 0.0;
    for (int r = 0; r < std::max(1, repeats); ++r) {
        ltgp_stats a, b;
        check(ltgp_get_stats(h.e, &a));
        std::uint64_t n = 0;
        check(ltgp_evaluate_population(h.e, rec.data(), &n));
        check(ltgp_get_stats(h.e, &b));
        consistent = consistent && n == nodes && b.nodes_evaluated - a.nodes_evaluated == nodes;
        for (const auto& x : rec) consistent = consistent && x.size > 0;
        if (b.eval_seconds > 0.0) best = std::max(best, static_cast<double>(nodes) * kLaneWidth / b.eval_seconds);
    }
    return best;
}
}  // namespace

BenchReport run_bench(const std::vector<std::size_t>& tree_sizes, const std::vector<std::uint32_t>& worker_counts,
                      std::uint64_t seed, std::size_t min_corpus_nodes, int repeats) {
    if (tree_sizes.empty() || worker_counts.empty()) throw std::invalid_argument("run_bench: empty grid");
    for (const std::uint32_t w : worker_counts)  // more GPUs than present: ltgp_engine_create reports it
        if (w == 0 || w > LTGP_MAX_SHARDS) throw std::invalid_argument("run_bench: worker count (GPUs) out of range");
    BenchReport report;
    const TestSuite suite = make_suite(suite_seed(seed));
    for (const std::size_t size0 : tree_sizes) {
        if (size0 == 0) throw std::invalid_argument("run_bench: tree size 0");
        const std::uint64_t n = size0 | 1u;  // random_tree_of_size needs an odd count
        const std::uint64_t count = std::max<std::uint64_t>(1, (min_corpus_nodes + n - 1) / n);
        std::vector<std::uint64_t> sizes(count, n), offs(count);
        const std::uint64_t stride = (n + 15) & ~std::uint64_t(15);
        std::vector<std::uint8_t> buf(stride * count, 0xff);
        for (std::uint64_t i = 0; i < count; ++i) {
            offs[i] = stride * i;
            Rng r(ltgp_host_tree_seed(seed, static_cast<std::uint32_t>(i)));
            random_tree_of_size(r, n, buf.data() + offs[i]);
        }
        const std::uint64_t nodes = n * count;
        bool c1 = true;
        const double batch = corpus_gpops(1, suite, buf, offs, sizes, nodes, repeats, c1);
        for (const std::uint32_t w : worker_counts) {
            BenchCell cell;
            cell.tree_size = n;
            cell.workers = w;
            cell.nodes = nodes;
            cell.batch_gpops = batch;
            bool cw = c1;
            cell.parallel_gpops = w == 1 ? batch : corpus_gpops(w, suite, buf, offs, sizes, nodes, repeats, cw);
            cell.parallel_speedup = batch > 0.0 ? cell.parallel_gpops / batch : 0.0;
            cell.counters_consistent = cw;
            report.cells.push_back(cell);
        }
    }
    return report;
}

}  // namespace ltgp

using namespace ltgp;

extern "C" {

uint64_t ltgp_host_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ltgp_host_suite_seed(uint64_t s) { return suite_seed(s); }

void ltgp_host_make_suite(uint64_t seed, float* in, float* tg, float* cs) {
    const TestSuite s = make_suite(seed);
    std::memcpy(in, s.inputs, sizeof s.inputs);
    std::memcpy(tg, s.targets, sizeof s.targets);
    std::memcpy(cs, s.constants, sizeof s.constants);
}

// The bulk Mt64 engine against std::mt19937_64 (the engine rng.hpp:50
// names): outputs for several seeds across many twists, and the text state
// both ways (a checkpoint written by one resumes in the other). 0 = equal.
int ltgp_host_rng_selftest(void) {
    for (const uint64_t seed : {0ull, 1ull, 42ull, 0x9e3779b97f4a7c15ull, ~0ull}) {
        ltgp::Mt64 a(seed);
        std::mt19937_64 b(seed);
        for (int i = 0; i < 5000; ++i)
            if (a() != b()) return 1;
        std::ostringstream sa, sb;
        sa << a;
        sb << b;
        if (sa.str() != sb.str()) return 2;
        std::istringstream ia(sb.str());
        ltgp::Mt64 c(7);
        ia >> c;
        std::mt19937_64 d;
        std::istringstream ib(sa.str());
        ib >> d;
        for (int i = 0; i < 2000; ++i) {
            const uint64_t x = a(), y = b(), z = c(), w = d();
            if (x != y || x != z || x != w) return 3;
        }
        // prefill (ring growth included) leaves the stream and its text unchanged
        for (const uint64_t n : {1ull, 311ull, 5000ull, 100000ull}) {
            a.prefill(n);
            for (uint64_t i = 0; i < n / 2 + 7; ++i)
                if (a() != b()) return 4;
            std::ostringstream ta, tb;
            ta << a;
            tb << b;
            if (ta.str() != tb.str()) return 5;
        }
    }
    return 0;
}

uint64_t ltgp_host_tree_seed(uint64_t seed, uint32_t i) {
    return splitmix64(seed ^ (0x7265657274ull + (uint64_t)i * 0x9e3779b97f4a7c15ull));
}

int ltgp_host_random_tree_of_size(uint64_t seed, uint64_t n, uint8_t* out) {
    try {
        Rng rng(seed);
        random_tree_of_size(rng, n, out);
        return 0;
    } catch (...) {
        return -1;
    }
}

uint64_t ltgp_host_corpus(uint64_t seed, uint32_t M, double lg_lo, double lg_hi, uint32_t first,
                          uint32_t count, uint8_t* buf, uint64_t* offsets, uint64_t* sizes, int threads) {
    Rng rng(seed);
    for (uint32_t i = 0; i < M; ++i) {
        const double u = static_cast<double>(rng.below(1ull << 53)) * 0x1.0p-53;
        uint64_t n = static_cast<uint64_t>(std::floor(std::pow(10.0, lg_lo + (lg_hi - lg_lo) * u)));
        sizes[i] = n | 1u;  // odd
    }
    if (first > M) first = M;
    if (count > M - first) count = M - first;
    uint64_t total = 0;
    for (uint32_t j = 0; j < count; ++j) {
        if (offsets) offsets[j] = total;
        total += (sizes[first + j] + 15) & ~uint64_t(15);
    }
    if (!buf || !offsets) return total;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
        for (uint32_t j; (j = next.fetch_add(1)) < count;) {
            const uint32_t i = first + j;
            Rng r(ltgp_host_tree_seed(seed, i));
            random_tree_of_size(r, sizes[i], buf + offsets[j]);
            const uint64_t pad = ((sizes[i] + 15) & ~uint64_t(15)) - sizes[i];
            std::memset(buf + offsets[j] + sizes[i], 0xff, pad);
        }
    };
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) ts.emplace_back(work);
    for (auto& t : ts) t.join();
    return total;
}

// Remy's algorithm: start from one leaf; n_internal times pick a uniform
// node x and replace it by a new function node whose children are x and a
// new leaf (the new leaf left or right with equal probability). Then label
// in prefix order as in config 3.
int ltgp_host_remy_tree(uint64_t seed, uint64_t n, uint8_t* out) {
    if (n == 0 || n % 2 == 0 || n > 0xfffffffeull) return -1;
    Rng rng(seed);
    const uint32_t total = static_cast<uint32_t>(n);
    std::vector<uint32_t> left(total, UINT32_MAX), right(total, UINT32_MAX), parent(total, UINT32_MAX);
    uint32_t root = 0;
    for (uint32_t k = 0; 2 * k + 1 < total; ++k) {
        const uint32_t x = static_cast<uint32_t>(rng.below(2ull * k + 1));
        const uint32_t a = 2 * k + 1, b = 2 * k + 2;
        const uint32_t p = parent[x];
        if (p == UINT32_MAX) root = a;
        else if (left[p] == x) left[p] = a;
        else right[p] = a;
        parent[a] = p;
        if (rng.below(2) == 0) { left[a] = x; right[a] = b; }
        else { left[a] = b; right[a] = x; }
        parent[x] = a;
        parent[b] = a;
    }
    std::vector<uint32_t> todo{root};
    uint64_t pos = 0;
    while (!todo.empty()) {
        const uint32_t v = todo.back();
        todo.pop_back();
        if (left[v] == UINT32_MAX) {
            out[pos++] = rng.below(2) == 0 ? kOpX : static_cast<uint8_t>(kOpFirstConstant + rng.below(250));
        } else {
            out[pos++] = static_cast<uint8_t>(rng.below(4));
            todo.push_back(right[v]);
            todo.push_back(left[v]);
        }
    }
    return pos == n ? 0 : -1;
}

uint64_t ltgp_host_ramped(uint64_t seed, uint32_t count, uint64_t capacity, int dmin, int dmax, uint8_t* out,
                          uint64_t out_cap, uint64_t* sizes) {
    try {
        Rng rng(seed);
        const auto pop = ramped_half_and_half(rng, count, capacity, dmin, dmax, GrowMode::kUniformPrimitive);
        uint64_t pos = 0;
        for (uint32_t i = 0; i < count; ++i) {
            if (pos + pop[i].size() > out_cap) return 0;
            std::memcpy(out + pos, pop[i].data(), pop[i].size());
            sizes[i] = pop[i].size();
            pos += pop[i].size();
        }
        return pos;
    } catch (...) {
        return 0;
    }
}

void ltgp_host_plan_generation(uint64_t seed, uint32_t M, const ltgp_record* rec, uint32_t k, ltgp_plan* out) {
    std::vector<Individual> pop(M);
    for (uint32_t i = 0; i < M; ++i) {
        pop[i].fitness = rec[i].fitness;
        pop[i].size = rec[i].size;
    }
    Rng rng(seed);
    const auto plans = plan_generation(rng, pop, k);
    std::copy(plans.begin(), plans.end(), out);
}

}  // extern "C"

namespace {

// Checkpoint/resume of a run (a SPEC non-goal kept
// as an operational feature): the device-resident population, its records,
// the Rng stream position and the run counters, written after a completed
// generation. Little-endian binary: Header, the Rng text state, M records
// {fitness bits, hits, size, depth}, the M genomes back to back (size bytes
// each, downloaded from the engine), then an FNV-1a 64 of everything before.
constexpr char kCkptMagic[8] = {'L', 'T', 'G', 'P', 'C', 'K', 'P', '1'};

struct CkptHeader {
    char magic[8];
    uint32_t M, k;
    uint64_t node_limit, seed, memory_budget;
    int32_t grow_mode;
    uint32_t rng_len;
    uint64_t gen, nodes;
    double secs;
    int64_t gauge_live, gauge_high;
    uint64_t dump_bytes;  // dump length at this checkpoint: a resume truncates the dump back to it
};

struct Fnv {
    uint64_t h = 0xcbf29ce484222325ull;
    void add(const void* p, size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    }
};

struct CkptWriter {
    FILE* f;
    Fnv fnv;
    void put(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) throw std::runtime_error("checkpoint: write failed");
        fnv.add(p, n);
    }
};

struct CkptReader {
    FILE* f;
    Fnv fnv;
    void get(void* p, size_t n) {
        if (n && std::fread(p, 1, n, f) != n) throw std::invalid_argument("checkpoint: truncated file");
        fnv.add(p, n);
    }
};

void save_checkpoint(const char* path, ltgp_engine* e, const CkptHeader& h0, const Rng& rng,
                     const std::vector<Individual>& pop) {
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) throw std::runtime_error("checkpoint: cannot open " + tmp);
    try {
        CkptWriter w{f, {}};
        CkptHeader h = h0;
        const std::string rs = rng.state();
        h.rng_len = static_cast<uint32_t>(rs.size());
        w.put(&h, sizeof h);
        w.put(rs.data(), rs.size());
        for (const auto& ind : pop) {
            const ltgp_record r{ind.fitness, ind.hits, ind.size, ind.depth};
            w.put(&r, sizeof r);
        }
        std::vector<uint8_t> buf;
        for (uint32_t i = 0; i < h.M; ++i) {  // the genomes live on the device
            buf.resize(pop[i].size);
            uint64_t n = 0;
            check(ltgp_download_genome(e, i, buf.data(), buf.size(), &n));
            if (n != pop[i].size) throw std::runtime_error("checkpoint: genome size mismatch");
            w.put(buf.data(), buf.size());
        }
        const uint64_t sum = w.fnv.h;
        if (std::fwrite(&sum, 8, 1, f) != 1) throw std::runtime_error("checkpoint: write failed");
        if (std::fclose(f) != 0) throw std::runtime_error("checkpoint: close failed");
    } catch (...) {
        std::fclose(f);
        std::remove(tmp.c_str());
        throw;
    }
    if (std::rename(tmp.c_str(), path) != 0) throw std::runtime_error("checkpoint: rename failed");
}

// Loads a checkpoint written by a run with the same parameters (any
// mismatch is std::invalid_argument, like validate(RunConfig)).
void load_checkpoint(const char* path, const CkptHeader& want, CkptHeader& h, Rng& rng,
                     std::vector<Individual>& pop) {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::invalid_argument(std::string("checkpoint: cannot open ") + path);
    try {
        CkptReader r{f, {}};
        r.get(&h, sizeof h);
        if (std::memcmp(h.magic, kCkptMagic, 8) != 0) throw std::invalid_argument("checkpoint: bad magic");
        if (h.M != want.M || h.k != want.k || h.node_limit != want.node_limit || h.seed != want.seed ||
            h.memory_budget != want.memory_budget || h.grow_mode != want.grow_mode)
            throw std::invalid_argument("checkpoint: run parameters differ");
        if (h.rng_len > 1u << 20) throw std::invalid_argument("checkpoint: bad Rng state length");
        std::string rs(h.rng_len, '\0');
        r.get(rs.data(), rs.size());
        rng.set_state(rs);
        pop.assign(h.M, Individual{});
        for (auto& ind : pop) {
            ltgp_record rec;
            r.get(&rec, sizeof rec);
            ind.fitness = rec.fitness;
            ind.hits = rec.hits;
            ind.size = rec.size;
            ind.depth = rec.depth;
        }
        for (auto& ind : pop) {
            if (ind.size == 0 || ind.size > h.node_limit) throw std::invalid_argument("checkpoint: bad genome size");
            std::vector<uint8_t> ops(ind.size);
            r.get(ops.data(), ops.size());
            ind.genome = Genome(std::move(ops));
        }
        uint64_t sum = 0;
        if (std::fread(&sum, 8, 1, f) != 1 || sum != r.fnv.h)
            throw std::invalid_argument("checkpoint: checksum mismatch");
        std::fclose(f);
    } catch (...) {
        std::fclose(f);
        throw;
    }
}

}  // namespace

extern "C" {

// run.hpp:33-36 on the engine, optionally checkpointed
// every ckpt_every generations and/or resumed from a checkpoint.
int64_t ltgp_host_run_checkpointed(ltgp_engine* e, uint32_t M, uint32_t G, uint64_t node_limit, uint32_t k,
                                   uint64_t seed, int grow_mode, uint64_t memory_budget, const char* dump_path,
                                   const char* ckpt_path, uint32_t ckpt_every, const char* resume_path,
                                   int* reason, uint64_t* nodes, double* eval_seconds) {
    try {
        if (!reason || !nodes) throw std::invalid_argument("null reason / nodes_evaluated pointer");
        RunConfig cfg;
        cfg.population_size = M;
        cfg.max_generations = G;
        cfg.node_limit = node_limit;
        cfg.tournament_size = k;
        cfg.seed = seed;
        cfg.memory_budget_bytes = memory_budget;
        validate(cfg);
        if (ckpt_every && !ckpt_path) throw std::invalid_argument("ckpt_every without a checkpoint path");
        const TestSuite suite = make_suite(suite_seed(seed));
        Rng rng(seed);
        std::vector<Individual> pop(M), next;
        std::vector<WorkerState> pool(1);
        MemoryGauge gauge;
        ExecContext ctx{suite, cfg, pool, gauge, e};
        CkptHeader hdr{};
        std::memcpy(hdr.magic, kCkptMagic, 8);
        hdr.M = M;
        hdr.k = k;
        hdr.node_limit = node_limit;
        hdr.seed = seed;
        hdr.memory_budget = memory_budget;
        hdr.grow_mode = grow_mode;
        *reason = 0;
        *nodes = 0;
        double secs = 0.0;
        uint32_t gen0 = 0;
        uint64_t dump_bytes0 = 0;
        if (resume_path) {
            CkptHeader h;
            load_checkpoint(resume_path, hdr, h, rng, pop);
            gauge.restore(h.gauge_live, h.gauge_high);
            // the parents go back to the device; their records are restored,
            // not recomputed
            check(ltgp_set_suite(e, suite.inputs, suite.targets, suite.constants));
            std::vector<const std::uint8_t*> ptrs(M);
            std::vector<std::uint64_t> sizes(M);
            for (uint32_t i = 0; i < M; ++i) {
                ptrs[i] = pop[i].genome.data();
                sizes[i] = pop[i].genome.size();
            }
            check(ltgp_upload_population(e, M, ptrs.data(), sizes.data()));
            for (auto& ind : pop) ind.genome.release();
            gen0 = static_cast<uint32_t>(h.gen);
            dump_bytes0 = h.dump_bytes;
            *nodes = h.nodes;
            secs = h.secs;
        }
        FILE* dump = nullptr;
        if (dump_path && resume_path) {
            // generations dumped after the checkpoint (a run that died between
            // checkpoints) are cut off, so the resumed dump equals an
            // uninterrupted run's
            dump = std::fopen(dump_path, "r+");
            if (!dump) throw std::invalid_argument(std::string("resume: cannot open the dump ") + dump_path);
            std::fflush(dump);
            if (ftruncate(fileno(dump), static_cast<off_t>(dump_bytes0)) != 0)
                throw std::runtime_error("resume: cannot truncate the dump");
            std::fseek(dump, 0, SEEK_END);
        } else if (dump_path) {
            dump = std::fopen(dump_path, "w");
        }
        auto write_dump = [&](uint32_t gen) {  // stats.hpp:104-107
            if (!dump) return;
            for (uint32_t i = 0; i < M; ++i) {
                uint32_t bits;
                std::memcpy(&bits, &pop[i].fitness, 4);
                if (pop[i].fitness != pop[i].fitness) bits = 0x7fc00000u;
                std::fprintf(dump, "%u %u %u %u %d %08x\n", gen, i, pop[i].size, pop[i].depth, pop[i].hits, bits);
            }
        };
        auto checkpoint = [&](uint32_t gen) {
            if (!ckpt_path) return;
            hdr.gen = gen;
            hdr.nodes = *nodes;
            hdr.secs = secs;
            hdr.gauge_live = gauge.live();
            hdr.gauge_high = gauge.high_water();
            hdr.dump_bytes = 0;
            if (dump) {
                std::fflush(dump);
                hdr.dump_bytes = static_cast<uint64_t>(std::ftell(dump));
            }
            save_checkpoint(ckpt_path, e, hdr, rng, pop);
        };
        ltgp_stats st;
        if (!resume_path) {
            auto genomes = ramped_half_and_half(rng, M, node_limit, 2, 6, static_cast<GrowMode>(grow_mode));
            for (uint32_t i = 0; i < M; ++i) pop[i].genome = std::move(genomes[i]);
            gauge.add(M);
            evaluate_population(pop, ctx);
            check(ltgp_get_stats(e, &st));
            secs += st.eval_seconds;
            for (auto& ind : pop) *nodes += ind.size;
            write_dump(0);
            if (ckpt_every) checkpoint(0);
        }
        int64_t done = gen0;
        // LTGP_TRACE=1: host wall time of each generation's planning and
        // execution (the engine adds its own phase marks)
        static const bool trace = std::getenv("LTGP_TRACE") != nullptr;
        uint64_t draws = 0;  // the last generation's Rng draws
        for (uint32_t gen = gen0 + 1; gen <= G; ++gen) {
            const auto t0 = std::chrono::steady_clock::now();
            const uint64_t d0 = rng.draw_count();
            const auto plans = plan_generation(rng, pop, k);
            draws = rng.draw_count() - d0;
            const auto t1 = std::chrono::steady_clock::now();
            execute_generation_begin(plans, pop, ctx);
            // while the device runs the generation: the next one's Rng blocks
            // (its draws are a tie or two away from this one's)
            rng.prefill(draws + draws / 8 + 1024);
            const ExecOutcome o = execute_generation_end(plans, pop, next, ctx);
            if (trace) {
                const auto t2 = std::chrono::steady_clock::now();
                std::fprintf(stderr, "[ltgp] gen %u: plan_generation %.1f us, execute_generation %.1f us, %llu draws\n",
                             gen, std::chrono::duration<double, std::micro>(t1 - t0).count(),
                             std::chrono::duration<double, std::micro>(t2 - t1).count(), (unsigned long long)draws);
            }
            if (o.memory_budget_exceeded) { *reason = 2; break; }  // TerminationReason (evolve.hpp:34)
            if (o.size_limit_hit) { *reason = 1; break; }
            std::swap(pop, next);
            check(ltgp_get_stats(e, &st));
            secs += st.eval_seconds;
            for (auto& ind : pop) *nodes += ind.size;
            done = gen;
            write_dump(gen);
            if (ckpt_every && (gen % ckpt_every == 0 || gen == G)) checkpoint(gen);
        }
        if (dump) std::fclose(dump);
        if (eval_seconds) *eval_seconds = secs;
        return done;
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "ltgp_host_run: %s\n", ex.what());
        return -1;
    }
}

int ltgp_host_run_bench(const uint64_t* tree_sizes, uint32_t n_sizes, const uint32_t* worker_counts,
                        uint32_t n_workers, uint64_t seed, uint64_t min_corpus_nodes, int repeats,
                        ltgp_bench_cell* out) {
    try {
        if (!tree_sizes || !worker_counts || !out) throw std::invalid_argument("null argument");
        const std::vector<std::size_t> ts(tree_sizes, tree_sizes + n_sizes);
        const std::vector<std::uint32_t> wc(worker_counts, worker_counts + n_workers);
        const BenchReport r = run_bench(ts, wc, seed, min_corpus_nodes, repeats);
        for (std::size_t i = 0; i < r.cells.size(); ++i) {
            const BenchCell& c = r.cells[i];
            out[i] = ltgp_bench_cell{c.tree_size, c.workers, c.nodes, c.scalar_gpops, c.batch_gpops,
                                     c.parallel_gpops, c.vector_speedup, c.parallel_speedup,
                                     c.counters_consistent ? 1 : 0};
        }
        return 0;
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "ltgp_host_run_bench: %s\n", ex.what());
        return -1;
    }
}

int64_t ltgp_host_run(ltgp_engine* e, uint32_t M, uint32_t G, uint64_t node_limit, uint32_t k, uint64_t seed,
                      int grow_mode, uint64_t memory_budget, const char* dump_path, int* reason, uint64_t* nodes,
                      double* eval_seconds) {
    return ltgp_host_run_checkpointed(e, M, G, node_limit, k, seed, grow_mode, memory_budget, dump_path, nullptr,
                                      0, nullptr, reason, nodes, eval_seconds);
}

}  // extern "C"
