// ltgp.hpp — the reference's host-side population API (namespace ltgp, same
// names, argument meaning and error behaviour), re-implemented so that the
// evaluation and crossover hot path runs on the B200 engine behind
// include/ltgp_cuda.h. Each declaration cites the reference header it mirrors
// (/root/reference/proj/include/ltgp/).
//
// What differs from the reference, by design:
//  * Individual::genome may be empty after execute_generation: children live
//    in the engine's device arena; fitness/hits/size/depth are filled from
//    the engine's records, and plan_generation draws points from
//    Individual::size.
//  * ExecContext carries the engine handle (an extra trailing member; the
//    reference's four members keep their meaning).
#pragma once

#include <cstddef>
#include <cstdint>
#include <istream>
#include <ostream>
#include <limits>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/ltgp_cuda.h"

namespace ltgp {

inline constexpr std::size_t kLaneWidth = 48;           // common.hpp:10-11
inline constexpr std::uint8_t kOpAdd = 0, kOpSub = 1, kOpMul = 2, kOpDiv = 3, kOpX = 4;
inline constexpr std::uint8_t kOpFirstConstant = 5;     // opcodes.hpp:10-15
inline constexpr int kFunctionCount = 4, kConstantCount = 250;
constexpr bool is_function(std::uint8_t op) { return op < kFunctionCount; }  // opcodes.hpp:22

// rng.hpp:9-14
inline constexpr std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// The engine of rng.hpp:20-21 (std::mt19937_64) with bulk output: the
// same recurrence, seeding and tempering as the standard's
// mersenne_twister_engine<uint64_t, 64, 312, 156, 31, 0xb5026f5aa96619e9,
// 29, 0x5555555555555555, 17, 0x71d67fffeda60000, 37, 0xfff7eee000000000,
// 43, 6364136223846793005>, but each twist also tempers all 312 outputs in
// one vectorisable pass, so a draw is a load (the standard library tempers
// per call). Its text state is the standard's ("x0 ... x311 p"), so
// checkpoints read and write the same form; ltgp_host_rng_selftest checks
// outputs and text against std::mt19937_64. plan_generation is bound by
// this stream (64K draws per 4000-child generation).
//
// Blocks (one twist's state and its 312 tempered outputs) live in a ring:
// prefill(n) twists ahead so the next n draws are loads, which the run loop
// does while the device executes a generation (ltgp_execute_generation_launch
// .. _finish). The stream is the same with or without prefill.
class Mt64 {
public:
    static constexpr int kN = 312, kM = 156;
    explicit Mt64(std::uint64_t s) : ring_(4) {
        std::uint64_t* x = ring_[0].x;
        x[0] = s;
        for (int i = 1; i < kN; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + (std::uint64_t)i;
        temper(ring_[0]);
        p_ = kN;
    }
    std::uint64_t operator()() {
        if (p_ >= kN) advance();
        return ring_[cur_].out[p_++];
    }
    // twist ahead until the next n draws need no twist
    void prefill(std::uint64_t n) {
        const std::uint64_t have = (std::uint64_t)(kN - p_) + (std::uint64_t)ahead_ * kN;
        if (n <= have) return;
        const std::size_t blocks = (std::size_t)((n - have + kN - 1) / kN);
        if (ahead_ + blocks + 1 > ring_.size()) {  // grow, keeping current .. ahead in order
            std::vector<Block> r(std::max(2 * ring_.size(), ahead_ + blocks + 1));
            for (std::size_t i = 0; i <= ahead_; ++i) r[i] = ring_[(cur_ + i) % ring_.size()];
            ring_.swap(r);
            cur_ = 0;
        }
        for (std::size_t i = 0; i < blocks; ++i) {
            const std::size_t src = (cur_ + ahead_) % ring_.size();
            twist(ring_[src], ring_[(src + 1) % ring_.size()]);
            ++ahead_;
        }
    }
    friend std::ostream& operator<<(std::ostream& os, const Mt64& m) {
        const std::uint64_t* x = m.ring_[m.cur_].x;
        for (int i = 0; i < kN; ++i) os << x[i] << ' ';
        return os << m.p_;
    }
    friend std::istream& operator>>(std::istream& is, Mt64& m) {
        Block b;
        unsigned p = 0;
        for (int i = 0; i < kN; ++i) is >> b.x[i];
        is >> p;
        if (is && p > (unsigned)kN) is.setstate(std::ios::failbit);
        if (is) {
            temper(b);
            m.ring_.assign(4, Block{});
            m.ring_[0] = b;
            m.cur_ = 0;
            m.ahead_ = 0;
            m.p_ = p;
        }
        return is;
    }

private:
    friend class Rng;
    struct Block {
        std::uint64_t x[kN];    // the state after this block's twist
        std::uint64_t out[kN];  // its tempered outputs
    };
    // next block: prefilled, or twisted now
    void advance() {
        const std::size_t nx = (cur_ + 1) % ring_.size();
        if (ahead_ == 0) twist(ring_[cur_], ring_[nx]);
        else --ahead_;
        cur_ = nx;
        p_ = 0;
    }
    const std::uint64_t* out() const { return ring_[cur_].out; }
    // dst = the twist of src, tempered (ltgp_host.cpp: one clone per vector
    // ISA, AVX2 / AVX-512 where the host has it)
    static void twist(const Block& src, Block& dst);
    static void temper(Block& b) {
        for (int i = 0; i < kN; ++i) {
            std::uint64_t z = b.x[i];
            z ^= (z >> 29) & 0x5555555555555555ull;
            z ^= (z << 17) & 0x71d67fffeda60000ull;
            z ^= (z << 37) & 0xfff7eee000000000ull;
            z ^= z >> 43;
            b.out[i] = z;
        }
    }
    std::vector<Block> ring_;
    std::size_t cur_ = 0, ahead_ = 0;  // current block, blocks twisted beyond it
    unsigned p_;
};

// rng.hpp:20-51: sequential stream; value mappings by hand so every output
// is a pure function of the seed.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(splitmix64(seed)) {}
    std::uint64_t below(std::uint64_t n) {
        ++draws_;
        unsigned __int128 m = static_cast<unsigned __int128>(engine_()) * n;
        auto lo = static_cast<std::uint64_t>(m);
        if (lo < n) {
            const std::uint64_t threshold = (0 - n) % n;
            while (lo < threshold) {
                m = static_cast<unsigned __int128>(engine_()) * n;
                lo = static_cast<std::uint64_t>(m);
            }
        }
        return static_cast<std::uint64_t>(m >> 64);
    }
    float uniform_pm1() {
        ++draws_;
        const double u = static_cast<double>(engine_() >> 11) * 0x1.0p-53;
        return static_cast<float>(2.0 * u - 1.0);
    }
    std::uint64_t draw_count() const { return draws_; }
    // twist ahead so the next n draws are loads (same stream)
    void prefill(std::uint64_t n) { engine_.prefill(n); }

    // The same stream for a hot loop (plan_generation's 64K draws per
    // generation): the stream position and the draw count live in the
    // cursor's locals, i.e. registers. Through below() every draw is a
    // store-to-load chain on the Rng's members (~6 ns per draw there against
    // ~1.5 ns here). Written back when the cursor goes out of scope; the Rng
    // must not be used directly while a cursor on it is alive.
    class Cursor {
    public:
        explicit Cursor(Rng& r) : r_(r), out_(r.engine_.out()), p_(r.engine_.p_) {}
        ~Cursor() {
            r_.engine_.p_ = p_;
            r_.draws_ += draws_;
        }
        Cursor(const Cursor&) = delete;
        Cursor& operator=(const Cursor&) = delete;
        std::uint64_t raw() {
            if (p_ >= (unsigned)Mt64::kN) [[unlikely]] {
                r_.engine_.advance();
                out_ = r_.engine_.out();
                p_ = 0;
            }
            return out_[p_++];
        }
        // Rng::below, draw for draw
        std::uint64_t below(std::uint64_t n) {
            ++draws_;
            unsigned __int128 m = static_cast<unsigned __int128>(raw()) * n;
            auto lo = static_cast<std::uint64_t>(m);
            if (lo < n) [[unlikely]] {
                const std::uint64_t threshold = (0 - n) % n;
                while (lo < threshold) {
                    m = static_cast<unsigned __int128>(raw()) * n;
                    lo = static_cast<std::uint64_t>(m);
                }
            }
            return static_cast<std::uint64_t>(m >> 64);
        }
    private:
        Rng& r_;
        const std::uint64_t* out_;
        unsigned p_;
        std::uint64_t draws_ = 0;
    };
    // Checkpoint/resume: the engine state in the
    // standard's portable text form, then the draw counter.
    std::string state() const {
        std::ostringstream os;
        os << engine_ << ' ' << draws_;
        return os.str();
    }
    void set_state(const std::string& s) {
        std::istringstream is(s);
        is >> engine_ >> draws_;
        if (!is) throw std::invalid_argument("malformed Rng state");
    }

private:
    Mt64 engine_;  // std::mt19937_64's stream (rng.hpp:50)
    std::uint64_t draws_ = 0;
};

// genome.hpp:19-38
class Genome {
public:
    Genome() = default;
    explicit Genome(std::vector<std::uint8_t> ops) : ops_(std::move(ops)) {}
    std::size_t size() const noexcept { return ops_.size(); }
    bool empty() const noexcept { return ops_.empty(); }
    std::uint8_t operator[](std::size_t i) const noexcept { return ops_[i]; }
    const std::uint8_t* data() const noexcept { return ops_.data(); }
    std::span<const std::uint8_t> ops() const noexcept { return {ops_.data(), ops_.size()}; }
    void release() noexcept { std::vector<std::uint8_t>().swap(ops_); }
    friend bool operator==(const Genome&, const Genome&) = default;

private:
    std::vector<std::uint8_t> ops_;
};

// sextic.hpp:25-31
struct TestSuite {
    alignas(64) float inputs[kLaneWidth]{};
    alignas(64) float targets[kLaneWidth]{};
    float constants[kConstantCount]{};
};

float target(float x);                       // sextic.hpp:33-35
TestSuite make_suite(Rng& rng);              // sextic.hpp:50
TestSuite make_suite(std::uint64_t seed);    // sextic.hpp:51
std::uint64_t suite_seed(std::uint64_t run_seed);  // driver.hpp:17-19

// Grow-method primitive choice below the depth cap: the SPEC's rule
// (uniform over all 255 primitives) or the 50/50
// function-vs-terminal alternative the SPEC leaves open.
enum class GrowMode { kUniformPrimitive = 0, kHalfFunctions = 1 };

Genome gen_full(Rng& rng, int target_depth, std::size_t capacity);   // genome.hpp:61
Genome gen_grow(Rng& rng, int max_depth, std::size_t capacity,
                GrowMode mode = GrowMode::kUniformPrimitive);        // genome.hpp:64
std::vector<Genome> ramped_half_and_half(Rng& rng, std::size_t count, std::size_t capacity,
                                         int min_depth = 2, int max_depth = 6,
                                         GrowMode mode = GrowMode::kUniformPrimitive);  // genome.hpp:68
Genome random_tree_of_size(Rng& rng, std::size_t nodes);             // bench.hpp:15
void random_tree_of_size(Rng& rng, std::size_t nodes, std::uint8_t* out);

// evolve.hpp:17-23
struct Individual {
    Genome genome;
    float fitness = std::numeric_limits<float>::quiet_NaN();
    std::int32_t hits = 0;
    std::uint32_t size = 0;
    std::uint32_t depth = 0;
};

using CrossoverPlan = ltgp_plan;  // evolve.hpp:27-32 (same field order)

enum class TerminationReason { kMaxGenerations, kSizeLimitHit, kMemoryBudgetExceeded };  // evolve.hpp:34

struct RunConfig {  // evolve.hpp:37-47
    std::uint32_t population_size = 4000;
    std::uint32_t max_generations = 10000;
    std::uint64_t node_limit = 15'000'000;
    std::uint32_t tournament_size = 7;
    std::uint32_t worker_count = 1;
    std::uint64_t seed = 1;
    std::uint64_t memory_budget_bytes = 0;
    bool streaming_memory = false;
    double stack_safety = 2.0;
};
void validate(const RunConfig& config);  // evolve.hpp:49-50, throws std::invalid_argument

struct WorkerState {};   // evolve.hpp:73-77: per-worker stacks live on the GPU
struct MemoryGauge {     // evolve.hpp:52-71 (live genome accounting)
    void add(std::int64_t n = 1) { live_ += n; if (live_ > high_) high_ = live_; }
    void sub(std::int64_t n = 1) { live_ -= n; }
    std::int64_t live() const { return live_; }
    std::int64_t high_water() const { return high_; }
    void restore(std::int64_t live, std::int64_t high) { live_ = live; high_ = high; }
private:
    std::int64_t live_ = 0, high_ = 0;
};

struct ExecContext {     // evolve.hpp:95-100, plus the engine handle
    const TestSuite& suite;
    const RunConfig& config;
    std::vector<WorkerState>& pool;
    MemoryGauge& gauge;
    ltgp_engine* engine = nullptr;
};

struct ExecOutcome {  // evolve.hpp:102-104, plus the memory budget outcome
    bool size_limit_hit = false;
    bool memory_budget_exceeded = false;
};

inline bool fitness_better(float a, float b) {  // eval.hpp:90-94
    if (a != a) return false;
    if (b != b) return true;
    return a < b;
}
inline bool fitness_tied(float a, float b) { return (a != a && b != b) || a == b; }  // eval.hpp:96-98

std::size_t tournament(Rng& rng, std::span<const Individual> population, std::uint32_t k);  // evolve.hpp:82
std::vector<CrossoverPlan> plan_generation(Rng& rng, std::span<const Individual> population,
                                           std::uint32_t tournament_size);  // evolve.hpp:86-87

// evolve.hpp:106-117 — the drop-in boundary, on the engine.
void evaluate_population(std::vector<Individual>& population, ExecContext ctx);
ExecOutcome execute_generation(std::span<const CrossoverPlan> plans, std::vector<Individual>& parents,
                               std::vector<Individual>& children, ExecContext ctx);

// bench.hpp:17-35 on the engine. A cell's `workers` is a GPU count (devices
// 0..workers-1, the population sharded over them); batch_gpops is one GPU
// and parallel_gpops `workers` GPUs, both device-timed evaluations of the
// whole corpus (best of `repeats`). The engine has no CPU interpreter, so
// scalar_gpops and vector_speedup stay 0 (the reference's CPU columns are the
// oracle's, timed by bench.py's cpu_baseline). counters_consistent: the
// engine's node counter advanced by exactly the corpus size per evaluation.
struct BenchCell {
    std::size_t tree_size = 0;
    std::uint32_t workers = 0;
    std::uint64_t nodes = 0;
    double scalar_gpops = 0.0;
    double batch_gpops = 0.0;
    double parallel_gpops = 0.0;
    double vector_speedup = 0.0;
    double parallel_speedup = 0.0;
    bool counters_consistent = false;
};
struct BenchReport {
    std::vector<BenchCell> cells;
};
BenchReport run_bench(const std::vector<std::size_t>& tree_sizes, const std::vector<std::uint32_t>& worker_counts,
                      std::uint64_t seed, std::size_t min_corpus_nodes, int repeats);

// Throws std::runtime_error with ltgp_last_error() on an engine failure.
void check(int status);

}  // namespace ltgp
