// ltgp_engine.cu — libltgp_cuda.so: the C ABI declared in include/ltgp_cuda.h.
//
// Replaces the reference's population evaluation and crossover execution
// (/root/reference/proj/include/ltgp/evolve.hpp:106-117, genome.hpp:56-84,
// eval.hpp:70-87) with device-resident B200 kernels. Host code here only
// moves plans/records and orchestrates launches; every tree node is
// evaluated on the GPU (there is no CPU fallback in this library).

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sched.h>
#include <unistd.h>  // environ
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>  // types only: libnccl is opened at run time (see RecordGather)

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ltgp_cuda.h"
#include "ltgp_gen.cuh"
#include "ltgp_kernels.cuh"
#include "ltgp_pack.h"
#include "ltgp_splice.cuh"

using namespace ltgp_dev;

namespace {

constexpr int kWarps = 32;           // warps per k_eval CTA (one CTA per SM)
constexpr int kWindow = 20;          // shared stack window frames per warp
constexpr uint32_t kDefaultChunk = 16384;
constexpr uint32_t kMaxSteps = 1024;
constexpr uint32_t kMaxFrames = 256;
constexpr uint32_t kMaxChunk = 1048576;    // automatic chunk length ceiling
constexpr uint32_t kMaxWaveChunk = 1u << 22;  // ... of the one-wave rule for a few huge trees (launch_eval)
constexpr uint32_t kSpillFrames = 1024;  // per warp; items that need more are re-run
constexpr int kRerunCtas = 8;

thread_local std::string g_err;

// NVTX3 ranges (header-only; no-ops unless a tool such as nsys attaches):
// one range per engine phase (work list / plan / k_eval / combine / extents /
// splice / gather), so a timeline shows the host orchestration around the
// kernels.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// LTGP_TRACE=1: per-phase host wall times of execute_generation on stderr;
// every mark is also an NVTX marker, and the Trace's lifetime an NVTX range.
struct Trace {
    bool on = std::getenv("LTGP_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Trace(const char* name) { nvtxRangePushA(name); }
    ~Trace() { nvtxRangePop(); }
    void mark(const char* what) {
        nvtxMarkA(what);
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ltgp] %-12s %8.1f us\n", what,
                     std::chrono::duration<double, std::micro>(t - t0).count());
        t0 = t;
    }
};

void set_err(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            set_err("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
            return -1;                                                                    \
        }                                                                                 \
    } while (0)

// LTGP_DEBUG_SYNC=1: synchronize after every launch so a fault names its kernel.
static const bool g_debug_sync = std::getenv("LTGP_DEBUG_SYNC") != nullptr;
#define DEBUG_SYNC(st, what)                                                                  \
    do {                                                                                      \
        if (g_debug_sync) {                                                                   \
            cudaError_t _e = cudaStreamSynchronize(st);                                       \
            if (_e != cudaSuccess) {                                                          \
                set_err("%s failed: %s", what, cudaGetErrorString(_e));                       \
                return -1;                                                                    \
            }                                                                                 \
        }                                                                                     \
    } while (0)

#define TRY(x)                  \
    do {                        \
        if ((x) != 0) return -1; \
    } while (0)

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    int ensure(size_t need, int device) {
        if (need <= bytes && p) return 0;
        const size_t old = bytes;
        if (p) { cudaSetDevice(dev); cudaFree(p); p = nullptr; bytes = 0; }
        // geometric growth: bloating populations regrow O(log) times, and a
        // regrow costs a device synchronisation (cudaFree)
        size_t nb = std::max<size_t>({need + need / 8, 2 * old, size_t(256)});
        cudaSetDevice(device);
        cudaError_t e = cudaMalloc(&p, nb);
        if (e != cudaSuccess) {
            set_err("cudaMalloc(%zu) failed: %s", nb, cudaGetErrorString(e));
            p = nullptr;
            return -1;
        }
        bytes = nb;
        dev = device;
        return 0;
    }
    void release() {
        if (p) { cudaSetDevice(dev); cudaFree(p); }
        p = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct HostBuf {  // grow-only pinned host buffer
    void* p = nullptr;
    size_t bytes = 0;
    int ensure(size_t need) {
        if (need <= bytes && p) return 0;
        const size_t old = bytes;
        if (p) cudaFreeHost(p);
        p = nullptr;
        // geometric growth: per-generation work lists fluctuate in size, and
        // cudaFreeHost + cudaMallocHost costs ~100 us of host time that the
        // GPU would wait for
        size_t nb = std::max<size_t>({need + need / 4, 2 * old, size_t(256)});
        if (cudaMallocHost(&p, nb) != cudaSuccess) {
            set_err("cudaMallocHost(%zu) failed", nb);
            p = nullptr;
            bytes = 0;
            return -1;
        }
        bytes = nb;
        return 0;
    }
    void release() { if (p) cudaFreeHost(p); p = nullptr; bytes = 0; }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

inline uint64_t ceil16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// A set of trees resident on one device: tree i at arena + off[i].
struct TreeSet {
    DevBuf arena, off, size, decode, meta;
    std::vector<uint64_t> h_off;
    std::vector<uint32_t> h_size;
    uint32_t count = 0;
    uint64_t bytes = 0;   // used arena bytes
    uint64_t version = 0; // bumped whenever the layout (sizes) changes
    void release() { arena.release(); off.release(); size.release(); decode.release(); meta.release(); }
};

uint64_t g_version = 0;

// Streamed evaluation: slice g = trees [tree_begin, next slice's) whose bytes
// are host src[src, src+len) -> arena[dst, dst+len).
struct Slice {
    uint32_t tree_begin;
    uint64_t src, dst, len;
    uint64_t pk_off = 0;  // packed transfer (ltgp_pack.h): the slice's region in the staging buffers
};
constexpr uint32_t kMaxSlices = 64;
constexpr int kComputeStreams = 4;     // slice g runs on compute stream g % 4
constexpr uint32_t kCpopsSmem = 96 * 1024;  // k_cpops's shared segment stack (2 per chunk of a tree)
constexpr uint64_t kSlicePad = 2048;   // arena gap between slices (k_eval's record look-ahead < 1 KB)
// LTGP_TRACE=1: a streamed evaluation prints when each slice's copy, plan
// and evaluation ended (ms after the call's first event), to stderr
bool trace_slices() {
    static const bool v = std::getenv("LTGP_TRACE") != nullptr;
    return v;
}

// target bytes per slice and slice count cap of a streamed evaluation
// (LTGP_SLICE_KB / LTGP_SLICES override them; read per call)
uint64_t slice_bytes() {
    const char* v = std::getenv("LTGP_SLICE_KB");
    return v ? std::max<uint64_t>(1, std::strtoull(v, nullptr, 10)) << 10 : 16ull << 20;
}
uint32_t max_slices() {
    const char* v = std::getenv("LTGP_SLICES");
    // 48: the cross-slice launch takes each slice as it lands, so finer
    // slices start the device sooner (config 3: 16.2 ms at 48, 16.9 at 24)
    return v ? (uint32_t)std::min<long>(kMaxSlices, std::max<long>(1, std::strtol(v, nullptr, 10))) : 48u;
}
// packed PCIe transfer of streamed evaluations (LTGP_PACK=0 sends raw bytes)
// and its host threads (LTGP_PACK_THREADS, default: every hardware thread but one)
bool pack_enabled() {
    const char* v = std::getenv("LTGP_PACK");
    return !v || std::atoi(v) != 0;
}
int pack_threads() {
    const char* v = std::getenv("LTGP_PACK_THREADS");
    if (v) return std::max(1, std::min(std::atoi(v), 256));
    // the CPUs this process may run on, shared with the other ranks of a
    // one-process-per-GPU launch (torchrun sets LOCAL_WORLD_SIZE): spinning
    // packers must never outnumber the cores.
    cpu_set_t cs;
    int n = sched_getaffinity(0, sizeof cs, &cs) == 0 ? CPU_COUNT(&cs) : (int)std::thread::hardware_concurrency();
    if (const char* w = std::getenv("LOCAL_WORLD_SIZE")) n /= std::max(1, std::atoi(w));
    // two cores stay free: the calling thread (kernel launches, or a share
    // of the packing) and whatever else the host runs (config 3, 16 cores:
    // 14 threads 16.37 ms per call, 15 threads 16.71)
    return std::max(1, std::min(n - 2, 256));
}
constexpr uint32_t kQueueBase = 16;    // counters[16 + g]: work queue of slice g
constexpr uint32_t kPoolCounters = 8;  // counters[8..11]: chunk-summary pool claims (2 x u64)
constexpr uint32_t kXFlagBase = kQueueBase + kMaxSlices;  // counters[kXFlagBase ..): cross-slice flags (3 per slice)
constexpr size_t kCounterBytes = 2048;
static_assert(kCounterBytes >= 4 * (kXFlagBase + 4 * kMaxSlices), "every slice needs its queue counter and flags");
static_assert(kMaxSlices == kMaxXSlices, "one flag triple per slice");
// A packed streamed evaluation runs ONE persistent k_eval that also decodes
// and plans each slice as its bytes land (per-slice launches each left a
// drained-CTA tail and waited for SMs to plan): LTGP_XSLICE=0 selects the
// per-slice launches
bool xslice_enabled() {
    const char* v = std::getenv("LTGP_XSLICE");
    if (v) return std::atoi(v) != 0;
    // a tool that serialises kernel launches (ncu: NV_NSIGHT_INJECTION_* /
    // NV_COMPUTE_PROFILER_*; injection libraries: CUDA_INJECTION64_PATH;
    // compute-sanitizer; CUDA_LAUNCH_BLOCKING) would hold the host inside the
    // launch while the kernel waits for the host's copies
    const char* lb = std::getenv("CUDA_LAUNCH_BLOCKING");
    if (lb && std::atoi(lb) != 0) return false;
    for (char** e = environ; e && *e; ++e)
        if (!std::strncmp(*e, "NV_NSIGHT_INJECTION", 19) || !std::strncmp(*e, "NV_COMPUTE_PROFILER", 19) ||
            !std::strncmp(*e, "CUDA_INJECTION64_PATH=", 22) || !std::strncmp(*e, "NV_SANITIZER", 12) ||
            !std::strncmp(*e, "COMPUTE_SANITIZER", 17))
            return false;
    return true;
}
// cuStreamWriteValue32 (driver API, found at run time): the copy stream marks
// a slice copied without a kernel (every SM may be busy in k_eval)
typedef int (*StreamWriteValue32)(cudaStream_t, unsigned long long, uint32_t, unsigned int);
StreamWriteValue32 stream_write_value32() {
    static StreamWriteValue32 f = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<StreamWriteValue32>(fn);
    }();
    return f;
}

struct Shard {
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaStream_t xs[kComputeStreams] = {};      // compute streams of a streamed evaluation (xs[0] = st)
    cudaStream_t cst = nullptr;                 // its copy stream
    std::vector<cudaEvent_t> sev;               // 3 per slice: copied, planned, evaluated
    std::vector<Slice> slices;                  // non-empty during a streamed evaluation
    const uint8_t* src = nullptr;               // its pinned host source
    HostBuf pk_host;                            // packed slices (ltgp_pack.h), pinned, one region per slice
    DevBuf pk_dev;                              // and their device copies
    uint64_t h2d_bytes = 0;                     // bytes the last streamed evaluation sent
    HostBuf h_xsl, h_xblk;                      // cross-slice launch: the slice descriptors (XSlice), task blocks
    DevBuf xsl, xblk, xtime;                    // and its trace timestamps (LTGP_TRACE)
    std::vector<uint32_t> slice_items;          // slice g's items: [slice_items[g], slice_items[g+1])
    std::vector<uint32_t> slice_ct, slice_ch;   // slice g's chunked trees / chunks (same convention)
    std::vector<uint32_t> items_slices;         // work-list cache key (slice tree boundaries)
    DevBuf xspill[kComputeStreams];             // spill areas of xs[1..] (xs[0] uses spill)
    cudaEvent_t ev[8] = {};
    cudaEvent_t kev[2] = {};                    // around k_eval of a resident evaluation
    int sms = 0;
    int eval_grid = 0;
    uint32_t first = 0, count = 0;  // global slot range
    std::vector<Item> wl_items;                  // work-list scratch (host)
    std::vector<CombineTree> wl_ctrees;
    std::vector<uint8_t> wl_tier;                // tapered tail: tier of each tree (0 = full-length chunks)
    std::vector<uint64_t> wl_sorted;             // (size << 32 | tree) of the chunked trees, ascending
    bool kev_valid = false;         // kev bracket the last evaluation's k_eval
    TreeSet set[2];
    int cur = 0;
    TreeSet scratch;                // ltgp_eval_one
    // evaluation scratch
    DevBuf items, ctrees, hdr, steps, frames, dframes, segs, spill, counters, rec, outs;
    DevBuf runs, cch, cres, saddr, big_addr[2];  // spine combine: pop runs, per chunk / tree, step operand addresses
    DevBuf big_steps[2], big_frames[2], rerun_items[2], rerun_slot[2], ovf, big_spill;  // overflow re-runs (2 tiers)
    double rerun_ksecs = 0.0, rerun_csecs = 0.0;
    bool last_outs = false;
    uint32_t last_reruns = 0;
    HostBuf h_items, h_ctrees, h_counters;
    uint32_t last_items = 0, last_chunks = 0, last_ctrees = 0, max_tree_chunks = 0;
    uint32_t cur_chunk = kDefaultChunk, cur_max_frames = kMaxFrames, cur_max_steps = kMaxSteps;
    double pool_per_chunk_f = 0.0, pool_per_chunk_s = 0.0;  // summary pool claimed per chunk (last evaluation)
    uint64_t last_steps = 0;                                  // spine steps claimed (last evaluation)
    EvalArgs eargs;      // arguments of the last evaluation (for overflow reruns)
    CombineArgs cargs;
    const TreeSet* items_for = nullptr;  // work list cache: (set, version)
    uint64_t items_version = 0;
    // crossover scratch
    DevBuf plans, ext, csize, coff, dir;
    HostBuf h_csize, h_coff, h_dir;
    DevBuf gstats;      // generation statistics scratch (GenStatsDev + best bits)
    HostBuf h_gstats;
    // device-resident generation (execute_generation_device): its status,
    // per-child work-list scratch, pinned staging (plans in; status,
    // counters, records and the children's layout out) and one captured
    // CUDA graph per parity of s.cur, re-captured when an argument changes
    DevBuf gen_status, gen_tree;
    HostBuf h_gen;
    cudaGraphExec_t gen_exec[2] = {};
    std::vector<uint8_t> gen_sig[2];
    struct GenPending {  // a launched device generation, until its finish
        size_t o_st = 0, o_cnt = 0, o_rec = 0, o_off = 0, o_size = 0;  // staging offsets
        EvalArgs a{};
        CombineArgs ca{};
    } genp;
    void release() {
        set[0].release(); set[1].release(); scratch.release();
        for (DevBuf* b : {&items, &ctrees, &hdr, &steps, &frames, &dframes, &segs, &spill, &counters,
                          &rec, &outs, &plans, &ext, &csize, &coff, &dir, &big_steps[0], &big_frames[0],
                          &big_steps[1], &big_frames[1], &rerun_items[0], &rerun_slot[0], &rerun_items[1],
                          &rerun_slot[1], &ovf, &big_spill, &gstats, &runs, &cch, &cres, &saddr, &big_addr[0],
                          &big_addr[1]}) b->release();
        h_gstats.release();
        gen_status.release(); gen_tree.release(); h_gen.release();
        for (auto& g : gen_exec) if (g) cudaGraphExecDestroy(g);
        h_items.release(); h_ctrees.release(); h_counters.release();
        h_csize.release(); h_coff.release(); h_dir.release();
        for (auto& b : xspill) b.release();
        pk_host.release(); pk_dev.release(); h_xsl.release(); xsl.release(); xtime.release();
        h_xblk.release(); xblk.release();
        if (st) { cudaSetDevice(dev); cudaStreamDestroy(st); }
        for (int k = 1; k < kComputeStreams; ++k) if (xs[k]) cudaStreamDestroy(xs[k]);
        if (cst) cudaStreamDestroy(cst);
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        for (auto& e : kev) if (e) cudaEventDestroy(e);
        for (auto& e : sev) if (e) cudaEventDestroy(e);
    }
};

}  // namespace

struct ltgp_engine {
    ltgp_config cfg;
    uint32_t chunk = kDefaultChunk;
    bool chunk_fixed = false;  // chunk_nodes given in the config
    std::vector<Shard> shards;
    SuiteArgs suite;
    bool have_suite = false;
    uint32_t M = 0;
    uint64_t memory_budget = 0;  // planned generation bytes allowed (0: no check)
    // RunConfig::streaming_memory (evolve.hpp:45, :111-114): children are
    // spliced in waves of stream_wave into the parents' own arena, and a
    // parent's bytes are released for reuse after the wave holding its last
    // planned use (a first-fit heap over the arena)
    bool streaming = false;
    uint32_t stream_wave = 256;
    uint64_t live_high_water = 0;    // live genomes (parents not yet retired + children built)
    uint64_t used_high_water = 0;    // arena bytes holding live genomes
    ltgp_stats stats;
    HostBuf staging;
    ltgp_pack::Pool* pack = nullptr;  // host packing threads of streamed evaluations (ltgp_pack.h)
    // ltgp_execute_generation_launch .. _finish
    struct Pending {
        bool active = false, device = false;
        uint32_t M = 0;
        std::vector<ltgp_plan> plans;  // host path: the plans, run at finish
    } pend;
    // record all-gather of a multi-shard population: every
    // shard's records into one n_shards x cmax array on each device
    struct Gather {
        bool nccl = false;                       // NCCL across distinct devices
        void* lib = nullptr;                     // dlopen'ed libnccl.so.2
        ncclComm_t comms[LTGP_MAX_SHARDS] = {};
        ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
        ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
        ncclResult_t (*group_start)() = nullptr;
        ncclResult_t (*group_end)() = nullptr;
        ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
        const char* (*error_string)(ncclResult_t) = nullptr;
        ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
        DevBuf send[LTGP_MAX_SHARDS], recv[LTGP_MAX_SHARDS];  // NCCL: per shard; copies: recv[0] only
        HostBuf h;
        cudaEvent_t ev[2] = {};
        // one process per GPU (ltgp_nccl_attach): this engine is one rank of
        // a communicator across processes; every evaluation all-gathers the
        // ranks' records (rank r's block at r x count)
        bool mp = false;
        int mp_rank = 0, mp_nranks = 1;
        ncclComm_t mp_comm = nullptr;
        uint32_t mp_count = 0;  // records per rank of the last gather
    } gather;
};

namespace {

static_assert(EvalLayout<kWarps, kWindow>::kBytes <= 227u * 1024u, "k_eval needs more than 227 KB of shared memory");
size_t eval_smem_bytes() { return EvalLayout<kWarps, kWindow>::kBytes; }
uint32_t spill_frames_base() {  // LTGP_SPILL_FRAMES overrides (debugging)
    static const uint32_t v = std::getenv("LTGP_SPILL_FRAMES") ? (uint32_t)std::atoi(std::getenv("LTGP_SPILL_FRAMES"))
                                                                : kSpillFrames;
    return v;
}
// per-warp spill frames for chunk length C: a chunk's stack (a random walk
// for random trees) reaches a few sqrt(C) frames; deeper items are re-run
uint32_t spill_frames(uint32_t C) {
    if (std::getenv("LTGP_SPILL_FRAMES")) return spill_frames_base();
    uint32_t f = spill_frames_base();
    const uint32_t want = (uint32_t)(8.0 * std::sqrt((double)C));
    while (f < want) f *= 2;
    return f;
}
#define K_EVAL k_eval<kWarps, kWindow, false>
#define K_EVAL_XS k_eval<kWarps, kWindow, true>
static_assert(kWindow == kPlanWindow, "the plan tasks use the interpreter's window");

int init_shard(ltgp_engine* e, Shard& s) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    s.xs[0] = s.st;
    for (int k = 1; k < kComputeStreams; ++k) CK(cudaStreamCreateWithFlags(&s.xs[k], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s.cst, cudaStreamNonBlocking));
    for (auto& ev : s.ev) CK(cudaEventCreate(&ev));
    for (auto& ev : s.kev) CK(cudaEventCreate(&ev));
    s.sev.resize(3 * kMaxSlices);
    for (auto& ev : s.sev) CK(cudaEventCreateWithFlags(&ev, trace_slices() ? cudaEventDefault : cudaEventDisableTiming));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, s.dev));
    if (prop.major < 10) {
        set_err("device %d is sm_%d%d; this engine is built for sm_100a (B200)", s.dev, prop.major,
                prop.minor);
        return -1;
    }
    s.sms = prop.multiProcessorCount;
    const size_t smem = eval_smem_bytes();
    CK(cudaFuncSetAttribute(K_EVAL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(K_EVAL_XS, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_cpops, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCpopsSmem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K_EVAL, kWarps * 32, smem));
    if (per_sm < 1) { set_err("k_eval does not fit on an SM"); return -1; }
    s.eval_grid = per_sm * s.sms;
    TRY(s.spill.ensure((size_t)s.eval_grid * kWarps * spill_frames_base() * kFrameBytes, s.dev));
    TRY(s.counters.ensure(kCounterBytes, s.dev));
    TRY(s.h_counters.ensure(64));
    return 0;
}

int launch_combine(ltgp_engine* e, Shard& s, const CombineArgs& ca, cudaStream_t st, uint32_t& launches);

// The cross-slice launch's queue: slice v's decode and plan tasks ahead of
// slice v-1's eval tasks, so a slice's plans are done long before its first
// eval task is taken (a plan barrier right in front of the evals idled the
// warps between slices: an evolved population evaluated 40% slower).
// Returns the task count; blocks = {first task, slice | kind << 16}.
uint32_t xs_blocks(const XSlice* x, uint32_t G, std::vector<uint2>& blocks) {
    blocks.clear();
    uint32_t t = 0;
    auto add = [&](uint32_t v, uint32_t kind, uint32_t n) {
        if (n) blocks.push_back(make_uint2(t, v | kind << 16)), t += n;
    };
    for (uint32_t v = 0; v <= G; ++v) {
        if (v < G) {
            add(v, 0, x[v].nd);
            add(v, 1, x[v].np);
        }
        if (v > 0) add(v - 1, 2, x[v - 1].np);
    }
    return t;
}

// Tapered tail of a resident work list (LTGP_TAPER = "f1,f2,f3": the share of
// one grid wave given to chunks of C/2, C/4 and C/8 nodes; "0" = off).
// The persistent grid ends with every warp inside its last item: with
// full-length items that tail is one item's latency (config 3: 0.92 ms of a
// 12.8 ms k_eval). The smallest chunked trees are cut into shorter chunks and
// placed last, so the final items are short; small trees are chosen so no
// tree's spine combine becomes the longest chain.
struct Taper {
    double f[3];
    bool on;
};
static const Taper& taper_cfg() {
    static const Taper v = [] {
        Taper t{{0.5, 0.5, 0.5}, true};
        if (const char* e = std::getenv("LTGP_TAPER")) {
            t.f[0] = t.f[1] = t.f[2] = 0.0;
            std::sscanf(e, "%lf,%lf,%lf", &t.f[0], &t.f[1], &t.f[2]);
            t.on = t.f[0] > 0 || t.f[1] > 0 || t.f[2] > 0;
        }
        return t;
    }();
    return v;
}

// Evaluate every tree of `ts` on shard s: records (and optional per-case
// outputs) land in rec/outs. Asynchronous on s.st.
//
// Streamed evaluation (s.slices non-empty, ltgp_evaluate_packed): the trees
// arrive from pinned host memory in slices (consecutive trees, each slice
// 2 KB apart in the arena). Slice g's bytes go over a copy stream; its
// k_decode, k_plan and k_eval start as soon as they land, on compute stream
// g % 4: a slice's k_eval lasts at least one work item's latency, so slices
// must not queue behind each other, and each k_eval fills the SMs the earlier
// slices' tails free. The upload overlaps the evaluation. Without slices the
// arena is resident and the whole set is one slice on s.st.
int launch_eval(ltgp_engine* e, Shard& s, TreeSet& ts, bool want_outs) {
    Trace tr("ltgp.evaluate");
    CK(cudaSetDevice(s.dev));
    const bool streamed = !s.slices.empty();
    const uint32_t G = streamed ? (uint32_t)s.slices.size() : 1u;
    // --- work list (host), per slice: chunk items of large trees, then whole
    // trees by size. Cached while the tree set's layout and slicing are unchanged.
    std::vector<uint32_t> tb(G + 1);  // slice g = trees [tb[g], tb[g+1])
    for (uint32_t g = 0; g < G; ++g) tb[g] = streamed ? s.slices[g].tree_begin : 0u;
    tb[G] = ts.count;
    if (s.items_for != &ts || s.items_version != ts.version || s.items_slices != tb) {
        // chunk length: the configured one, or sized so the persistent grid
        // gets >= ~1 item per warp (small populations must not wait on one
        // warp per tree; more, shorter items cost per-item planning, exits
        // and combine work: a 15.6M-node evolved population is 13% faster at
        // 2048 than at 1024), 1024..16384 nodes;
        // and, for huge trees, long enough to balance one item's scan latency
        // (~C / 13e6 s) against the largest tree's sequential combine (~N/C
        // chunks x 1.6 sqrt(C) spine steps x ~60 ns): C >= (1.25 N)^(2/3),
        // up to kMaxChunk (1e7 nodes: 65536; 4e8 nodes: 1048576)
        uint32_t C = e->chunk;
        if (!e->chunk_fixed) {
            uint64_t total = 0, biggest = 0;
            for (uint32_t t = 0; t < ts.count; ++t) {
                total += ts.h_size[t];
                biggest = std::max<uint64_t>(biggest, ts.h_size[t]);
            }
            const uint64_t per = total / ((uint64_t)s.eval_grid * kWarps + 1);
            C = 1024;
            // C doubles while 2C <= 1.5 x the per-warp share: evolved
            // generations 200 / 300 / 600 of config 2 evaluate 12% / 8% / 10%
            // faster than with 2C <= share (fewer chunks and spine steps
            // outweigh the part-empty last wave); 2C <= 2 x share lost at 600
            while (C < kDefaultChunk && (uint64_t)C * 2 * 2 <= per * 3) C *= 2;
            const double want = std::pow(1.25 * (double)biggest, 2.0 / 3.0);
            while (C < kMaxChunk && (double)C < want) C *= 2;
            // Wave balance: when chunks fill only a few waves of the
            // persistent grid, the last wave runs part-full (48 x 1e7 nodes
            // at 65536: 7344 chunks on 4736 warps, 2 waves at 77%). Shorten
            // the chunks (down to C/2, multiples of 1024) to the shortest
            // length that keeps the same number of waves.
            const uint64_t W = (uint64_t)s.eval_grid * kWarps;
            auto chunks_of = [&](uint32_t c) {
                uint64_t k = 0;
                for (uint32_t t = 0; t < ts.count; ++t)
                    if (ts.h_size[t] > c) k += (ts.h_size[t] + c - 1) / c;
                return k;
            };
            // chunks at C (C is a power of two here: shifts) and the trees
            // that get chunked, in one pass
            uint64_t k0 = 0, big_trees = 0, big_nodes = 0;
            {
                const uint32_t sh = (uint32_t)__builtin_ctz(C);
                for (uint32_t t = 0; t < ts.count; ++t)
                    if (ts.h_size[t] > C) {
                        k0 += ((uint64_t)ts.h_size[t] + C - 1) >> sh;
                        big_nodes += ts.h_size[t];
                        ++big_trees;
                    }
            }
            const uint64_t waves = (k0 + W - 1) / W;
            // Only for a few huge trees (config 4's regime): with thousands of
            // chunked trees (an evolved generation 3000: 3000+) the shorter
            // chunks cost more than the fuller last wave gains (4.33 vs 4.62
            // ms per evaluation without the rule there).
            // (Also when the chunks fill less than half a wave but the chunked
            // trees hold most of the nodes, e.g. the 6 trees one of 8 GPUs gets
            // of config 4: the power of two above `want` is up to twice too
            // long there, and C / 2, the floor below, measured best: 6 x 4e8
            // nodes at 524288 instead of 1048576, 94 vs 118 ms.)
            if ((k0 > W / 2 || big_nodes * 2 >= total) && waves <= 8 && C >= 2048 && big_trees <= 512) {
                // k_eval's time does not depend on the chunk length while the
                // grid stays full, and the sequential combine shrinks like
                // 1/sqrt(C) (spine steps), so the best length is the one that
                // gives every warp exactly ONE chunk: 48 x 4e8 nodes at 4082688
                // instead of 1015808 (4 waves): k_eval 312 vs 310 ms, combine
                // 19.2 vs 37.4 ms; 48 x 1e7 at 102400 instead of 51200:
                // 12.7 vs 14.1 ms per evaluation. Half a wave (twice that
                // length) doubles k_eval. Above kMaxWaveChunk the fewest waves
                // that length allows, shortened as before.
                const uint64_t w = std::max<uint64_t>(1, (chunks_of(kMaxWaveChunk) + W - 1) / W);
                uint32_t lo = 1, hi = kMaxWaveChunk / 1024;  // in units of 1024
                while (lo < hi) {  // smallest c with chunks_of(c) <= w * W (non-increasing in c)
                    const uint32_t mid = (lo + hi) / 2;
                    if (chunks_of(mid * 1024) <= w * W) hi = mid; else lo = mid + 1;
                }
                C = std::max<uint32_t>(hi * 1024, std::max<uint32_t>(1024, C / 2));
            }
        }
        // chunk summaries are sized exactly by k_plan (PlanPool); these are
        // the per-chunk capacities of the first overflow re-run tier (x4).
        // A chunk's spine and frames grow like sqrt(C) (Remy-random trees:
        // mean ~1.6 sqrt(C), max ~3.6 sqrt(C) frames, ~6 sqrt(C) steps)
        tr.mark("   chunk len");
        const uint32_t rc = (uint32_t)std::lround(std::sqrt((double)C));
        s.cur_chunk = C;
        s.cur_max_frames = std::max<uint32_t>(kMaxFrames, (6 * rc + 63) & ~63u);
        s.cur_max_steps = std::min<uint32_t>(C, std::max<uint32_t>(kMaxSteps, 16 * rc));
        // host vectors reused across evaluations (capacity kept: fresh
        // allocations page-faulted ~100 us per generation on evolved runs)
        std::vector<Item>& all = s.wl_items;
        std::vector<CombineTree>& ctrees = s.wl_ctrees;
        all.clear();
        ctrees.clear();
        s.slice_items.assign(G + 1, 0);
        s.slice_ct.assign(G + 1, 0);
        s.slice_ch.assign(G + 1, 0);
        uint32_t nch = 0, max_chunks = 0;
        all.reserve(ts.count + 64);
        for (uint32_t g = 0; g < G; ++g) {
            s.slice_items[g] = (uint32_t)all.size();
            s.slice_ct[g] = (uint32_t)ctrees.size();
            s.slice_ch[g] = nch;
            // the last slice of a streamed evaluation is all that runs after
            // the final copy: shorter chunks shorten that tail (an item's
            // latency is ~C / 13e6 s)
            // (never longer than C: the re-run tiers size worst-case
            // capacities from C)
            const uint32_t Cg = (G > 1 && g == G - 1) ? std::min<uint32_t>(C, std::max<uint32_t>(1024, C / 4)) : C;
            // Item order. Whole trees come largest first for load balance (by
            // log2(size) buckets, descending; tree order within a bucket),
            // after the chunks in tree order. Resident evaluations of at most
            // 8 waves of the persistent grid take all items longest first
            // (chunks before whole trees within a bucket), so the last wave is
            // made of the shortest items: evolved populations -2 to -5% per
            // evaluation. With more waves (config 3: 11) chunks in tree order
            // measured 2% faster, so they keep it. Two linear passes place
            // every item directly (no push_back, no sort).
            auto bucket = [](uint32_t n) { return 32 - __builtin_clz(n); };
            // chunk counts by shift when the length is a power of two (a 64-bit
            // divide per tree and pass showed up in the per-generation host time)
            const bool cg_pow2 = (Cg & (Cg - 1)) == 0;
            // Tapered tail (taper_cfg): tier k > 0 trees are cut into Cg >> k
            // nodes per chunk and placed after the full-length chunks
            std::vector<uint8_t>& tier = s.wl_tier;
            tier.clear();
            const uint32_t tier_c[4] = {Cg, Cg / 2, Cg / 4, Cg / 8};
            auto clen = [&](uint32_t t) { return tier.empty() ? Cg : tier_c[tier[t]]; };
            auto nchunks = [&](uint32_t n, uint32_t c) {
                return cg_pow2 ? (n + c - 1) >> (uint32_t)__builtin_ctz(c) : (n + c - 1) / c;
            };
            uint32_t wcnt[33], ccnt[33], tcnt[4];
            uint32_t nct_g, nch_g, nitems_g;
            auto count_pass = [&] {
                std::fill(wcnt, wcnt + 33, 0u);
                std::fill(ccnt, ccnt + 33, 0u);
                std::fill(tcnt, tcnt + 4, 0u);
                nct_g = nch_g = 0;
                for (uint32_t t = tb[g]; t < tb[g + 1]; ++t) {
                    const uint32_t n = ts.h_size[t];
                    if (n <= Cg) { ++wcnt[bucket(n)]; continue; }
                    const uint32_t c = clen(t), k = nchunks(n, c);
                    ++nct_g;
                    nch_g += k;
                    max_chunks = std::max(max_chunks, k);
                    if (c != Cg) { tcnt[tier[t]] += k; continue; }
                    ccnt[bucket(c)] += k - 1;
                    ++ccnt[bucket(n - (k - 1) * c)];
                }
                nitems_g = nch_g;
                for (int b = 0; b <= 32; ++b) nitems_g += wcnt[b];
            };
            count_pass();
            const uint32_t a0 = (uint32_t)all.size();
            const uint64_t grid_warps = (uint64_t)std::max(s.eval_grid, 1) * kWarps;
            const bool lpt = G == 1 && (uint64_t)nitems_g <= 8 * grid_warps;
            const Taper& tp = taper_cfg();
            if (G == 1 && !lpt && tp.on && !e->chunk_fixed && cg_pow2 && Cg >= 8192) {
                // the smallest chunked trees take the shortest chunks: ascending by
                // size, tier 3 (Cg/8) first, each tier up to its share of a wave
                std::vector<uint64_t>& sorted = s.wl_sorted;
                sorted.clear();
                for (uint32_t t = tb[g]; t < tb[g + 1]; ++t)
                    if (ts.h_size[t] > Cg) sorted.push_back((uint64_t)ts.h_size[t] << 32 | t);
                std::sort(sorted.begin(), sorted.end());
                tier.assign(ts.count, 0);
                size_t i = 0;
                for (int k = 3; k >= 1 && i < sorted.size(); --k) {
                    const uint64_t budget = (uint64_t)(tp.f[k - 1] * (double)grid_warps * tier_c[k]);
                    uint64_t acc = 0;
                    while (i < sorted.size() && acc + (sorted[i] >> 32) <= budget) {
                        tier[(uint32_t)sorted[i]] = (uint8_t)k;
                        acc += sorted[i] >> 32;
                        ++i;
                    }
                }
                count_pass();
            }
            uint32_t cpos[33], wpos[33], tpos[4] = {};
            uint32_t pos = a0, ccur = a0;
            if (lpt) {
                for (int b = 32; b >= 0; --b) { cpos[b] = pos; pos += ccnt[b]; wpos[b] = pos; pos += wcnt[b]; }
            } else {
                // full-length chunks in tree order, then by descending size class:
                // whole trees, then the tier whose chunk length falls in the class
                pos += nch_g - tcnt[1] - tcnt[2] - tcnt[3];
                for (int b = 32; b >= 0; --b) {
                    wpos[b] = pos;
                    pos += wcnt[b];
                    for (int k = 1; k <= 3; ++k)
                        if (tcnt[k] && bucket(tier_c[k]) == b) { tpos[k] = pos; pos += tcnt[k]; }
                }
            }
            all.resize(a0 + nitems_g);
            const uint32_t c0 = (uint32_t)ctrees.size();
            ctrees.resize(c0 + nct_g);
            uint32_t ci = c0;
            for (uint32_t t = tb[g]; t < tb[g + 1]; ++t) {
                const uint32_t n = ts.h_size[t];
                if (n <= Cg) {
                    all[wpos[bucket(n)]++] = Item{t, kWholeTree, 0, n};
                    continue;
                }
                const uint32_t c = clen(t), k = nchunks(n, c);
                ctrees[ci++] = CombineTree{t, nch, k, n};
                for (uint32_t q = 0; q < k; ++q) {
                    const uint32_t lo = q * c, hi = std::min(n, lo + c);
                    uint32_t& at = c != Cg ? tpos[tier[t]] : lpt ? cpos[bucket(hi - lo)] : ccur;
                    all[at++] = Item{t, nch + q, lo, hi};
                }
                nch += k;
            }
        }
        tr.mark("   items");
        s.slice_items[G] = (uint32_t)all.size();
        s.slice_ct[G] = (uint32_t)ctrees.size();
        s.slice_ch[G] = nch;
        const uint32_t nitems = (uint32_t)all.size();
        // the pinned staging buffers are reused: wait for their last copies
        // (not for the whole stream: a splice may still be running)
        CK(cudaEventSynchronize(s.ev[7]));
        tr.mark("   ev7 wait");
        TRY(s.h_items.ensure(sizeof(Item) * std::max<uint32_t>(nitems, 1)));
        std::copy(all.begin(), all.end(), s.h_items.as<Item>());
        TRY(s.items.ensure(sizeof(Item) * std::max<uint32_t>(nitems, 1), s.dev));
        if (nitems) CK(cudaMemcpyAsync(s.items.p, s.h_items.p, sizeof(Item) * nitems, cudaMemcpyHostToDevice, s.st));
        const uint32_t nct = (uint32_t)ctrees.size();
        if (nct) {
            TRY(s.h_ctrees.ensure(sizeof(CombineTree) * nct));
            std::copy(ctrees.begin(), ctrees.end(), s.h_ctrees.as<CombineTree>());
            TRY(s.ctrees.ensure(sizeof(CombineTree) * nct, s.dev));
            CK(cudaMemcpyAsync(s.ctrees.p, s.h_ctrees.p, sizeof(CombineTree) * nct,
                               cudaMemcpyHostToDevice, s.st));
            TRY(s.hdr.ensure(sizeof(ChunkHdr) * nch, s.dev));
            TRY(s.dframes.ensure((size_t)kFrameBytes * nch, s.dev));
            TRY(s.segs.ensure(sizeof(Seg) * 2 * nch, s.dev));
            TRY(s.runs.ensure(sizeof(PopRun) * 3 * nch, s.dev));
            TRY(s.cch.ensure(sizeof(CombChunk) * nch, s.dev));
            TRY(s.cres.ensure(sizeof(CombResult) * nct, s.dev));
        }
        tr.mark("  work list");
        s.last_items = nitems;
        s.last_chunks = nch;
        s.last_ctrees = nct;
        s.max_tree_chunks = max_chunks;
        s.items_for = &ts;
        s.items_version = ts.version;
        s.items_slices = tb;
        CK(cudaEventRecord(s.ev[7], s.st));  // h_items / h_ctrees copies issued
    }
    const uint32_t nitems = s.last_items, nct = s.last_ctrees, nch = s.last_chunks;
    // chunk-summary pool (k_plan claims every chunk's exact summary): an
    // estimate per chunk (Remy-random chunks: mean 1.6 sqrt(C) frames and
    // steps), raised to what earlier evaluations actually claimed per chunk
    PlanPool pool{};
    if (nch) {
        const double rc = std::sqrt((double)s.cur_chunk);
        const double pf = std::max(std::min(2.0 * rc, (double)s.cur_chunk + 2), s.pool_per_chunk_f * 1.25);
        const double ps = std::max(std::min(2.0 * rc, (double)s.cur_chunk), s.pool_per_chunk_s * 1.25);
        pool.cap_frames = (unsigned long long)(pf * nch) + 64;
        pool.cap_steps = (unsigned long long)(ps * nch) + 1024;
        TRY(s.frames.ensure((size_t)pool.cap_frames * kFrameBytes, s.dev));
        TRY(s.steps.ensure((size_t)pool.cap_steps, s.dev));
        pool.hdr = s.hdr.as<ChunkHdr>();
        pool.frames = s.frames.as<float2>();
        pool.steps = s.steps.as<uint8_t>();
        pool.used = reinterpret_cast<unsigned long long*>(s.counters.as<uint32_t>() + kPoolCounters);
        TRY(s.saddr.ensure((size_t)pool.cap_steps * 8, s.dev));
    }
    pool.spill_frames = spill_frames(s.cur_chunk);
    pool.adjusts = s.counters.as<uint32_t>() + 5;  // inline window adjusts join the statistics
    pool.flags = s.counters.as<uint32_t>() + 1;    // opcode 255 inside a tree: malformed
    TRY(s.rec.ensure(sizeof(ltgp_record) * std::max<uint32_t>(ts.count, 1), s.dev));
    if (want_outs) TRY(s.outs.ensure(sizeof(float) * kLanes * std::max<uint32_t>(ts.count, 1), s.dev));
    CK(cudaMemsetAsync(s.counters.p, 0, kCounterBytes, s.st));
    EvalArgs& a = s.eargs;
    a.arena = ts.arena.as<uint8_t>();
    a.off = ts.off.as<uint64_t>();
    a.size = ts.size.as<uint32_t>();
    a.items = s.items.as<Item>();
    a.n_items = nitems;
    a.n_items_dev = nullptr;
    a.counters = s.counters.as<uint32_t>();
    a.queue = s.counters.as<uint32_t>();
    a.item_base = 0;
    a.xsl = nullptr;
    a.n_xs = 0;
    a.xblk = nullptr;
    a.n_xblk = 0;
    a.n_tasks = 0;
    a.xflags = nullptr;
    a.meta = nullptr;
    a.xs_skip = 0;
    a.xtime = nullptr;
    a.hdr = s.hdr.as<ChunkHdr>();
    a.steps = s.steps.as<uint8_t>();
    a.frames = s.frames.as<float2>();
    a.max_steps = 0xffffffffu;   // first pass: k_plan's exact buffers (checked at item end)
    a.max_frames = 0xffffffffu;
    a.spill_frames = spill_frames(s.cur_chunk);
    TRY(s.spill.ensure((size_t)s.eval_grid * kWarps * a.spill_frames * kFrameBytes, s.dev));
    a.spill = s.spill.as<float2>();
    TRY(s.ovf.ensure(sizeof(uint32_t) * std::max<uint32_t>(nitems, 1), s.dev));
    a.ovf = s.ovf.as<uint32_t>();
    a.rec = s.rec.as<float>();
    a.outs = want_outs ? s.outs.as<float>() : nullptr;
    a.slot = nullptr;
    CombineArgs& ca = s.cargs;
    ca.trees = s.ctrees.as<CombineTree>();
    ca.n_trees = nct;
    ca.hdr = s.hdr.as<ChunkHdr>();
    ca.n_chunks = nch;
    ca.chunk0 = 0;
    ca.dframes = s.dframes.as<float2>();
    ca.segs = s.segs.as<Seg>();
    ca.runs = s.runs.as<PopRun>();
    ca.cch = s.cch.as<CombChunk>();
    ca.cres = s.cres.as<CombResult>();
    ca.space[0] = StepSpace{s.steps.as<uint8_t>(), nch ? pool.cap_steps : 0, s.saddr.as<uint64_t>()};
    ca.space[1] = ca.space[2] = StepSpace{nullptr, 0, nullptr};
    ca.rec = s.rec.as<float>();
    ca.outs = a.outs;
    ca.counters = s.counters.as<uint32_t>();
    ca.counts_dev = nullptr;
    s.last_outs = want_outs;
    s.last_reruns = 0;
    s.rerun_ksecs = s.rerun_csecs = 0.0;
    const uint64_t packets = (ts.bytes + 15) / 16;
    // +1 KB: the fast path stages record groups up to 512 B past an item
    TRY(ts.decode.ensure(std::max<uint64_t>(packets, 1) * 32 + 1024, s.dev));
    TRY(ts.meta.ensure(std::max<uint64_t>(packets, 1) * 4, s.dev));
    uint4* dec = ts.decode.as<uint4>();
    a.decode = dec;
    a.packets = packets;
    if (streamed)
        for (int k = 1; k < kComputeStreams && k < (int)G; ++k) TRY(s.xspill[k].ensure(s.spill.bytes, s.dev));
    tr.mark("  pool/setup");
    CK(cudaEventRecord(s.ev[0], s.st));
    s.kev_valid = false;
    uint32_t launches = 0;
    const bool xslice = streamed && G > 1 && nitems && e->pack && xslice_enabled() && stream_write_value32();
    if (xslice) {
        // one k_eval for every slice on s.st: its warps decode, plan and
        // evaluate each slice once the copy stream has marked it copied
        TRY(s.h_xsl.ensure(sizeof(XSlice) * G));
        TRY(s.xsl.ensure(sizeof(XSlice) * G, s.dev));
        XSlice* hx = s.h_xsl.as<XSlice>();
        uint32_t task = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const Slice& sl = s.slices[g];
            const ltgp_pack::Layout L(sl.len);
            XSlice& x = hx[g];
            x.pk = s.pk_dev.as<uint8_t>() + sl.pk_off;
            x.plane_bytes = L.plane_bytes;
            x.base_off = L.base_off;
            x.lit_off = L.lit_off;
            x.npk = L.npk;
            x.p_lo = sl.dst / 16;
            x.task0 = task;
            x.nd = (uint32_t)L.nblk;
            x.np = s.slice_items[g + 1] - s.slice_items[g];
            x.item0 = s.slice_items[g];
            task += x.nd + 2 * x.np;
        }
        std::vector<uint2> blk;
        task = xs_blocks(hx, G, blk);
        TRY(s.h_xblk.ensure(sizeof(uint2) * blk.size()));
        TRY(s.xblk.ensure(sizeof(uint2) * blk.size(), s.dev));
        std::memcpy(s.h_xblk.p, blk.data(), sizeof(uint2) * blk.size());
        CK(cudaMemcpyAsync(s.xblk.p, s.h_xblk.p, sizeof(uint2) * blk.size(), cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(s.xsl.p, hx, sizeof(XSlice) * G, cudaMemcpyHostToDevice, s.st));
        EvalArgs ag = a;
        ag.xsl = s.xsl.as<XSlice>();
        ag.n_xs = G;
        ag.xblk = s.xblk.as<uint2>();
        ag.n_xblk = (uint32_t)blk.size();
        ag.n_tasks = task;
        ag.xflags = s.counters.as<uint32_t>() + kXFlagBase;
        ag.meta = ts.meta.as<uint32_t>();
        ag.pool = pool;
        ag.queue = s.counters.as<uint32_t>() + kQueueBase;
        ag.xs_skip = std::getenv("LTGP_XS_SKIP") ? (uint32_t)std::atoi(std::getenv("LTGP_XS_SKIP")) : 0u;
        if (trace_slices()) {  // device timestamps of each slice's phases
            TRY(s.xtime.ensure(8 * (1 + 3 * kMaxSlices), s.dev));
            CK(cudaMemsetAsync(s.xtime.p, 0, 8 * (1 + 3 * kMaxSlices), s.st));
            ag.xtime = s.xtime.as<unsigned long long>();
        }
        K_EVAL_XS<<<s.eval_grid, kWarps * 32, eval_smem_bytes(), s.st>>>(ag, e->suite);
        CK(cudaGetLastError());
        ++launches;
    }
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t xk = g % kComputeStreams;
        cudaStream_t X = s.xs[xk];
        uint64_t p_lo = 0, p_hi = packets;
        if (streamed) {
            const Slice& sl = s.slices[g];
            if (g == 0) CK(cudaStreamWaitEvent(s.cst, s.ev[0], 0));  // counters cleared, arena free
            if (e->pack) {
                // packed transfer: the host threads pack this slice (~0.63 B per
                // node instead of 1) while the previous slices are in flight;
                // the next slice's packing starts before this one's kernels
                // are launched
                NvtxRange nr_pack("ltgp.pack");
                // (the cross-slice launch leaves the calling thread idle: it packs too)
                if (g == 0)
                    ltgp_pack::pack_start(e->pack, s.src + sl.src, sl.len, s.pk_host.as<uint8_t>() + sl.pk_off, xslice);
                const uint64_t nb = ltgp_pack::pack_wait(e->pack);
                CK(cudaMemcpyAsync(s.pk_dev.as<uint8_t>() + sl.pk_off, s.pk_host.as<uint8_t>() + sl.pk_off, nb,
                                   cudaMemcpyHostToDevice, s.cst));
                if (g + 1 < G) {
                    const Slice& nx = s.slices[g + 1];
                    ltgp_pack::pack_start(e->pack, s.src + nx.src, nx.len, s.pk_host.as<uint8_t>() + nx.pk_off, xslice);
                }
                s.h2d_bytes += nb;
            } else {
                CK(cudaMemcpyAsync(ts.arena.as<uint8_t>() + sl.dst, s.src + sl.src, sl.len, cudaMemcpyHostToDevice,
                                   s.cst));
                s.h2d_bytes += sl.len;
            }
            CK(cudaEventRecord(s.sev[3 * g], s.cst));
            if (xslice) {  // the slice's decode tasks may start
                const unsigned long long flag =
                    reinterpret_cast<unsigned long long>(s.counters.as<uint32_t>() + kXFlagBase + g);
                if (stream_write_value32()(s.cst, flag, 1u, 0u) != 0) {
                    set_err("cuStreamWriteValue32 failed");
                    return -1;
                }
                continue;
            }
            CK(cudaStreamWaitEvent(X, s.sev[3 * g], 0));
            // the previous slice's records are final before this slice's
            // kernels (its k_eval's look-ahead may read them)
            if (g > 0) CK(cudaStreamWaitEvent(X, s.sev[3 * (g - 1) + 1], 0));
            p_lo = sl.dst / 16;
            p_hi = (sl.dst + sl.len + 15) / 16;
        }
        const uint32_t i0 = s.slice_items[g], ni = s.slice_items[g + 1] - i0;
        // k_plan_warp (a warp per item, lane-parallel replay between window
        // adjustments) beats k_plan (a thread per item) on every measured
        // population (config 3: 14.13 vs 14.20 ms per evaluation; an evolved
        // 15.6M-node population: 0.66 vs 0.72 ms); LTGP_PLAN=0 selects k_plan.
        // On a resident evaluation k_plan_warp also decodes the packets it
        // plans (no k_decode pass: config 3 0.86 -> 0.64 ms). A streamed
        // slice keeps the separate, fully parallel k_decode: the fused pass
        // holds SMs longer while earlier slices' k_eval CTAs still occupy the
        // rest (e2e 2.37 -> 2.14 T GPops/s when fused).
        static const int plan_mode = std::getenv("LTGP_PLAN") ? std::atoi(std::getenv("LTGP_PLAN")) : 1;
        const bool plan_warp = plan_mode != 0;
        const bool fuse_decode = plan_warp && !streamed;
        NvtxRange nr_plan("ltgp.decode+plan");
        if (p_hi > p_lo && streamed && e->pack) {  // rebuild the slice's bytes into the arena, decoding them
            const Slice& sl = s.slices[g];
            const ltgp_pack::Layout L(sl.len);
            const uint64_t blocks = std::min<uint64_t>(L.nblk, (uint64_t)s.sms * 8);
            k_decode_packed<<<(unsigned)blocks, kPackBlock, 0, X>>>(
                s.pk_dev.as<uint8_t>() + sl.pk_off, L.plane_bytes, L.base_off, L.lit_off, L.npk, ts.arena.as<uint4>(),
                dec, ts.meta.as<uint32_t>(), packets, p_lo);
            CK(cudaGetLastError());
            DEBUG_SYNC(X, "k_decode_packed");
            ++launches;
        } else if (p_hi > p_lo && !fuse_decode) {
            const uint64_t blocks = std::min<uint64_t>((p_hi - p_lo + 255) / 256, (uint64_t)s.sms * 16);
            k_decode<<<(unsigned)blocks, 256, 0, X>>>(ts.arena.as<uint4>(), dec, ts.meta.as<uint32_t>(), packets,
                                                     p_lo, p_hi);
            CK(cudaGetLastError());
            DEBUG_SYNC(X, "k_decode");
            ++launches;
        }
        if (ni && fuse_decode) {  // a warp per item, decoding as it plans
            k_plan_warp<true><<<(ni + 3) / 4, 128, 0, X>>>(s.items.as<Item>() + i0, ni, nullptr, ts.off.as<uint64_t>(),
                                                          reinterpret_cast<uint8_t*>(dec), ts.meta.as<uint32_t>(),
                                                          ts.arena.as<uint4>(), packets, kWindow, pool);
            CK(cudaGetLastError());
            DEBUG_SYNC(X, "k_plan_warp");
            ++launches;
        } else if (ni && plan_warp) {  // a warp per item, after k_decode
            k_plan_warp<false><<<(ni + 3) / 4, 128, 0, X>>>(s.items.as<Item>() + i0, ni, nullptr, ts.off.as<uint64_t>(),
                                                           reinterpret_cast<uint8_t*>(dec), ts.meta.as<uint32_t>(),
                                                           ts.arena.as<uint4>(), packets, kWindow, pool);
            CK(cudaGetLastError());
            DEBUG_SYNC(X, "k_plan_warp");
            ++launches;
        } else if (ni) {
            k_plan<<<(ni + 127) / 128, 128, 0, X>>>(s.items.as<Item>() + i0, ni, ts.off.as<uint64_t>(),
                                                   reinterpret_cast<uint8_t*>(dec), ts.meta.as<uint32_t>(), packets,
                                                   kWindow, pool);
            CK(cudaGetLastError());
            DEBUG_SYNC(X, "k_plan");
            ++launches;
        }
        if (streamed) CK(cudaEventRecord(s.sev[3 * g + 1], X));
        if (ni) {
            EvalArgs ag = a;
            ag.items = a.items + i0;
            ag.n_items = ni;
            ag.item_base = i0;
            ag.queue = s.counters.as<uint32_t>() + kQueueBase + g;
            if (xk) ag.spill = s.xspill[xk].as<float2>();
            const int grid = std::min<int>(s.eval_grid, (int)ni);
            if (!streamed) CK(cudaEventRecord(s.kev[0], X));
            K_EVAL<<<std::max(grid, 1), kWarps * 32, eval_smem_bytes(), X>>>(ag, e->suite);
            CK(cudaGetLastError());
            if (!streamed) CK(cudaEventRecord(s.kev[1], X));
            s.kev_valid = !streamed;
            DEBUG_SYNC(X, "k_eval");
            ++launches;
        }
        if (streamed && s.slice_ct[g + 1] > s.slice_ct[g]) {
            // this slice's chunked trees, combined on its stream right away
            // (only the last slice's combine is left after the final copy)
            CombineArgs cg = ca;
            cg.trees = ca.trees + s.slice_ct[g];
            cg.cres = ca.cres + s.slice_ct[g];
            cg.n_trees = s.slice_ct[g + 1] - s.slice_ct[g];
            cg.chunk0 = s.slice_ch[g];
            cg.n_chunks = s.slice_ch[g + 1] - s.slice_ch[g];
            TRY(launch_combine(e, s, cg, X, launches));
        }
        if (streamed) CK(cudaEventRecord(s.sev[3 * g + 2], X));
    }
    if (xslice) {  // k_eval has waited for every copy; the trace's plan / eval marks are its end
        for (uint32_t g = 0; g < G; ++g) {
            CK(cudaEventRecord(s.sev[3 * g + 1], s.st));
            CK(cudaEventRecord(s.sev[3 * g + 2], s.st));
        }
    } else if (streamed) {  // join the other compute streams: the last slice each ran
        for (uint32_t g = G > (uint32_t)kComputeStreams ? G - kComputeStreams : 0; g < G; ++g)
            if (g % kComputeStreams) CK(cudaStreamWaitEvent(s.st, s.sev[3 * g + 2], 0));
    }
    CK(cudaEventRecord(s.ev[4], s.st));
    if (nct && (!streamed || xslice)) TRY(launch_combine(e, s, ca, s.st, launches));
    CK(cudaEventRecord(s.ev[1], s.st));
    CK(cudaMemcpyAsync(s.h_counters.p, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
    e->stats.kernel_launches = launches;
    tr.mark("  launches");
    return 0;
}

// Items whose stack outgrew the per-warp spill area, or chunks whose summary
// outgrew the per-chunk capacity, are re-scanned in two tiers: first with 4x
// the summary capacities on the full grid (a long-spined random tree
// occasionally needs that), then whatever still overflows with worst-case
// capacities (a chunk of C nodes holds at most C stack values, C spine steps)
// on a small grid with its own spill area; then every chunked tree is
// recombined once. Synchronous; only taken when the counters report an
// overflow. Device time is added to the evaluation's.
// The spine combine (k_cpops -> k_caddr -> k_combine) of the chunked trees
// and chunks `ca` names, on stream st.
int launch_combine(ltgp_engine* e, Shard& s, const CombineArgs& ca, cudaStream_t st, uint32_t& launches) {
    if (ca.n_trees == 0) return 0;
    NvtxRange nr("ltgp.spine_combine");
    // k_cpops's segment stack in shared memory: 2 per chunk of the tree
    const uint32_t segs = std::min<uint32_t>(2 * s.max_tree_chunks, kCpopsSmem / (uint32_t)sizeof(Seg));
    k_cpops<<<ca.n_trees, 32, segs * sizeof(Seg), st>>>(ca, segs);
    CK(cudaGetLastError());
    DEBUG_SYNC(st, "k_cpops");
    const uint32_t ablocks = std::min<uint32_t>((ca.n_chunks + 3) / 4, (uint32_t)s.sms * 16);
    k_caddr<<<std::max<uint32_t>(ablocks, 1), 128, 0, st>>>(ca);
    CK(cudaGetLastError());
    DEBUG_SYNC(st, "k_caddr");
    const int blocks = (int)std::min<uint32_t>((ca.n_trees + kCombineWarps - 1) / kCombineWarps, (uint32_t)s.sms * 16);
    k_combine<<<blocks, kCombineWarps * 32, 0, st>>>(ca, e->suite);
    CK(cudaGetLastError());
    DEBUG_SYNC(st, "k_combine");
    launches += 3;
    return 0;
}

int rerun_overflowed(ltgp_engine* e, Shard& s) {
    NvtxRange nr("ltgp.overflow_rerun");
    CK(cudaSetDevice(s.dev));
    const uint32_t C = s.cur_chunk;
    std::vector<Item> prev(s.h_items.as<Item>(), s.h_items.as<Item>() + s.last_items);
    uint32_t total = 0;
    float ms = 0.0f;
    // k_eval's error flags other than "overflow" and the pass statistics
    // survive the tiers (the first combine's verdict, [6], is superseded)
    uint32_t* hc = s.h_counters.as<uint32_t>();
    uint32_t keep = hc[1] & ~1u;
    const uint32_t exits = hc[4], adjusts = hc[5];
    for (int tier = 1; tier <= 2; ++tier) {
        const uint32_t n = hc[2];
        if (n == 0) break;
        std::vector<uint32_t> idx(n);
        CK(cudaMemcpyAsync(idx.data(), s.ovf.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        std::sort(idx.begin(), idx.end());
        std::vector<Item> items(n);
        std::vector<uint32_t> slots(n);
        for (uint32_t k = 0; k < n; ++k) {
            items[k] = prev[idx[k]];
            slots[k] = k;
        }
        if (tier == 1) total = n;
        const bool worst = tier == 2;
        const uint32_t fcap = worst ? C + 2 : std::min(C + 2, 4 * s.cur_max_frames);
        const uint32_t scap = worst ? C : std::min(C, 4 * s.cur_max_steps);
        DevBuf& bsteps = s.big_steps[tier - 1];
        DevBuf& bframes = s.big_frames[tier - 1];
        TRY(bsteps.ensure((size_t)n * scap, s.dev));
        TRY(bframes.ensure((size_t)n * fcap * kFrameBytes, s.dev));
        TRY(s.big_addr[tier - 1].ensure((size_t)n * scap * 8, s.dev));
        s.cargs.space[tier] = StepSpace{bsteps.as<uint8_t>(), (uint64_t)n * scap, s.big_addr[tier - 1].as<uint64_t>()};
        int grid;
        EvalArgs a = s.eargs;
        if (worst) {
            // worst-case spill is (C + 8) frames per warp: keep it within ~8 GB
            const int mem_ctas = (int)std::max<uint64_t>(
                1, (8ull << 30) / ((uint64_t)kWarps * (C + 8) * kFrameBytes));
            grid = std::max(1, std::min<int>({kRerunCtas, mem_ctas, (int)((n + kWarps - 1) / kWarps)}));
            TRY(s.big_spill.ensure((size_t)grid * kWarps * (C + 8) * kFrameBytes, s.dev));
            a.spill = s.big_spill.as<float2>();
            a.spill_frames = C + 8;
        } else {
            grid = std::max(1, std::min<int>(s.eval_grid, (int)((n + kWarps - 1) / kWarps)));
        }
        TRY(s.rerun_items[tier - 1].ensure(sizeof(Item) * n, s.dev));
        TRY(s.rerun_slot[tier - 1].ensure(sizeof(uint32_t) * n, s.dev));
        CK(cudaMemcpyAsync(s.rerun_items[tier - 1].p, items.data(), sizeof(Item) * n, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(s.rerun_slot[tier - 1].p, slots.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice,
                           s.st));
        CK(cudaMemsetAsync(s.counters.p, 0, 64, s.st));
        a.items = s.rerun_items[tier - 1].as<Item>();
        a.n_items = n;
        a.slot = s.rerun_slot[tier - 1].as<uint32_t>();
        a.steps = bsteps.as<uint8_t>();
        a.frames = bframes.as<float2>();
        a.max_steps = scap;
        a.max_frames = fcap;
        CK(cudaEventRecord(s.ev[5], s.st));
        K_EVAL<<<grid, kWarps * 32, eval_smem_bytes(), s.st>>>(a, e->suite);
        CK(cudaGetLastError());
        DEBUG_SYNC(s.st, "k_eval (re-run)");
        CK(cudaEventRecord(s.ev[6], s.st));
        CK(cudaMemcpyAsync(s.h_counters.p, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        CK(cudaEventElapsedTime(&ms, s.ev[5], s.ev[6]));
        s.rerun_ksecs += ms * 1e-3;
        e->stats.kernel_launches += 1;
        if (tier == 1) keep |= hc[1] & ~1u;
        prev.swap(items);
    }
    if (s.last_ctrees) {
        CK(cudaEventRecord(s.ev[5], s.st));
        uint32_t nl = 0;
        TRY(launch_combine(e, s, s.cargs, s.st, nl));
        CK(cudaEventRecord(s.ev[6], s.st));
        CK(cudaMemcpyAsync(s.h_counters.p, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        CK(cudaEventElapsedTime(&ms, s.ev[5], s.ev[6]));
        s.rerun_csecs += ms * 1e-3;
        e->stats.kernel_launches += nl;
    }
    hc[1] |= keep;
    hc[4] = exits;
    hc[5] = adjusts;
    s.last_reruns = total;
    return 0;
}

int check_eval(Shard& s) {
    const uint32_t* c = s.h_counters.as<uint32_t>();
    const uint32_t flags = c[1] | c[6];  // k_eval's and k_combine's
    if (c[2] != 0 || (flags & 1u)) {
        set_err("stack / chunk summary overflow in %u items after the worst-case re-run", c[2]);
        return -1;
    }
    if (flags & 8u) { set_err("k_eval shared-memory layout does not fit"); return -1; }
    if (flags & 64u) {
        set_err("cross-slice k_eval: a slice's copy never landed (kernel launches serialised by a tool? "
                "set LTGP_XSLICE=0)");
        return -1;
    }
    // malformed first: an invalid genome also derails the plan/scan cross-check
    if (flags & 2u) { set_err("malformed genome (stack underflow, leftover values or opcode 255 inside a tree)"); return -1; }
    if (flags & 16u) { set_err("chunk summary differs from k_plan's sizing (internal error)"); return -1; }
    return 0;
}

// After the stream is synchronized: re-run overflowed chunks if any.
int finish_eval(ltgp_engine* e, Shard& s) {
    const uint32_t* c = s.h_counters.as<uint32_t>();
    s.last_steps = 0;
    if (s.last_chunks) {  // what this evaluation's chunks claimed from the summary pool
        uint64_t uf, us;
        std::memcpy(&uf, c + kPoolCounters, 8);
        std::memcpy(&us, c + kPoolCounters + 2, 8);
        s.pool_per_chunk_f = (double)uf / s.last_chunks;
        s.pool_per_chunk_s = (double)us / s.last_chunks;
        s.last_steps = us;
    }
    if (c[2] != 0) TRY(rerun_overflowed(e, s));
    return check_eval(s);
}

// Assign contiguous slot ranges to shards, balanced by bytes.
void partition(ltgp_engine* e, uint32_t M, const uint64_t* sizes) {
    const int G = (int)e->shards.size();
    uint64_t total = 0;
    for (uint32_t i = 0; i < M; ++i) total += sizes ? sizes[i] : 1;
    uint32_t i = 0;
    uint64_t acc = 0;
    for (int g = 0; g < G; ++g) {
        Shard& s = e->shards[g];
        s.first = i;
        const uint64_t goal = (total * (uint64_t)(g + 1)) / (uint64_t)G;
        while (i < M && (g == G - 1 || acc + (sizes ? sizes[i] : 1) / 2 < goal)) {
            acc += sizes ? sizes[i] : 1;
            ++i;
        }
        s.count = i - s.first;
    }
}

int set_layout(Shard& s, TreeSet& ts, uint32_t count, const uint64_t* sizes, uint64_t* offs_out) {
    bool same = ts.count == count && ts.h_size.size() == count && ts.version != 0;
    for (uint32_t i = 0; same && i < count; ++i) same = ts.h_size[i] == sizes[i];
    if (!same) ts.version = ++g_version;
    ts.count = count;
    ts.h_off.resize(count);
    ts.h_size.resize(count);
    uint64_t o = 0;
    for (uint32_t i = 0; i < count; ++i) {
        if (sizes[i] == 0 || sizes[i] > 0xffffffffull) {
            set_err("genome size %llu out of range", (unsigned long long)sizes[i]);
            return -1;
        }
        ts.h_off[i] = o;
        ts.h_size[i] = (uint32_t)sizes[i];
        if (offs_out) offs_out[i] = o;
        o += ceil16(sizes[i]);
    }
    ts.bytes = o;
    TRY(ts.arena.ensure(std::max<uint64_t>(o, 16) + 64, s.dev));
    TRY(ts.off.ensure(sizeof(uint64_t) * std::max<uint32_t>(count, 1), s.dev));
    TRY(ts.size.ensure(sizeof(uint32_t) * std::max<uint32_t>(count, 1), s.dev));
    return 0;
}

int upload_tables(Shard& s, TreeSet& ts) {
    CK(cudaSetDevice(s.dev));
    if (ts.count == 0) return 0;
    CK(cudaMemcpyAsync(ts.off.p, ts.h_off.data(), sizeof(uint64_t) * ts.count, cudaMemcpyHostToDevice, s.st));
    CK(cudaMemcpyAsync(ts.size.p, ts.h_size.data(), sizeof(uint32_t) * ts.count, cudaMemcpyHostToDevice, s.st));
    CK(cudaStreamSynchronize(s.st));  // host vectors may change after return
    return 0;
}

// libnccl.so.2, opened at run time with RTLD_LOCAL (torch may have loaded
// its own copy into the process; its soname resolves to that copy)
int open_nccl(ltgp_engine::Gather& g) {
    if (g.lib) return 0;
    g.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!g.lib) { set_err("cannot open libnccl.so.2: %s", dlerror()); return -1; }
    g.comm_init_all = reinterpret_cast<decltype(g.comm_init_all)>(dlsym(g.lib, "ncclCommInitAll"));
    g.comm_init_rank = reinterpret_cast<decltype(g.comm_init_rank)>(dlsym(g.lib, "ncclCommInitRank"));
    g.all_gather = reinterpret_cast<decltype(g.all_gather)>(dlsym(g.lib, "ncclAllGather"));
    g.group_start = reinterpret_cast<decltype(g.group_start)>(dlsym(g.lib, "ncclGroupStart"));
    g.group_end = reinterpret_cast<decltype(g.group_end)>(dlsym(g.lib, "ncclGroupEnd"));
    g.comm_destroy = reinterpret_cast<decltype(g.comm_destroy)>(dlsym(g.lib, "ncclCommDestroy"));
    g.error_string = reinterpret_cast<decltype(g.error_string)>(dlsym(g.lib, "ncclGetErrorString"));
    if (!g.comm_init_all || !g.comm_init_rank || !g.all_gather || !g.group_start || !g.group_end ||
        !g.comm_destroy || !g.error_string) {
        set_err("libnccl.so.2 lacks a required symbol");
        return -1;
    }
    return 0;
}

// Opens NCCL for a population sharded over distinct devices (cfg.use_nccl):
// one communicator per shard, created in-process by ncclCommInitAll. The
// library is opened at run time with RTLD_LOCAL (torch may have loaded its
// own libnccl.so.2 into the process; its soname resolves to that copy).
int init_gather(ltgp_engine* e) {
    auto& g = e->gather;
    const int n = (int)e->shards.size();
    CK(cudaSetDevice(e->shards[0].dev));
    CK(cudaEventCreate(&g.ev[0]));
    CK(cudaEventCreate(&g.ev[1]));
    bool distinct = n > 1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j)
            if (e->shards[i].dev == e->shards[j].dev) distinct = false;
    if (!e->cfg.use_nccl || !distinct) return 0;
    TRY(open_nccl(g));
    int devs[LTGP_MAX_SHARDS];
    for (int i = 0; i < n; ++i) devs[i] = e->shards[i].dev;
    const ncclResult_t r = g.comm_init_all(g.comms, n, devs);
    if (r != ncclSuccess) { set_err("ncclCommInitAll: %s", g.error_string(r)); return -1; }
    g.nccl = true;
    // one line per engine so a multi-GPU run shows its communicator size
    std::string dl;
    for (int i = 0; i < n; ++i) dl += (i ? "," : "") + std::to_string(devs[i]);
    std::fprintf(stderr, "[ltgp] NCCL record all-gather: ncclCommInitAll nranks=%d devices=%s\n", n, dl.c_str());
    return 0;
}

void release_gather(ltgp_engine* e) {
    auto& g = e->gather;
    if (g.nccl)
        for (size_t i = 0; i < e->shards.size(); ++i) g.comm_destroy(g.comms[i]);
    if (g.mp && g.mp_comm) g.comm_destroy(g.mp_comm);
    for (auto& b : g.send) b.release();
    for (auto& b : g.recv) b.release();
    g.h.release();
    for (auto& ev : g.ev) if (ev) cudaEventDestroy(ev);
    if (g.lib) dlclose(g.lib);
    g = ltgp_engine::Gather{};
}

// All-gather of the shards' 16-byte records after an evaluation (every
// shard's stream already synchronised): shard s's block lands at
// [s * cmax, s * cmax + count_s) of an n x cmax array — on every device with
// NCCL (one grouped ncclAllGather, NVLink), on shard 0's device otherwise
// (peer copies; shards that repeat a device). Shard 0's array then goes to
// the host in one copy and is unpacked into slot order.
int gather_records(ltgp_engine* e, ltgp_record* out) {
    NvtxRange nr("ltgp.record_all_gather");
    auto& g = e->gather;
    const int n = (int)e->shards.size();
    uint32_t cmax = 1;
    for (const Shard& s : e->shards) cmax = std::max(cmax, s.count);
    const size_t blk = sizeof(ltgp_record) * cmax;
    Shard& s0 = e->shards[0];
    CK(cudaSetDevice(s0.dev));
    CK(cudaEventRecord(g.ev[0], s0.st));
    if (g.nccl) {
        for (int i = 0; i < n; ++i) {
            Shard& s = e->shards[i];
            TRY(g.send[i].ensure(blk, s.dev));
            TRY(g.recv[i].ensure(blk * n, s.dev));
            CK(cudaSetDevice(s.dev));
            if (s.count)
                CK(cudaMemcpyAsync(g.send[i].p, s.rec.p, sizeof(ltgp_record) * s.count, cudaMemcpyDeviceToDevice,
                                   s.st));
        }
        g.group_start();
        for (int i = 0; i < n; ++i) {
            const ncclResult_t r = g.all_gather(g.send[i].p, g.recv[i].p, blk, ncclUint8, g.comms[i], e->shards[i].st);
            if (r != ncclSuccess) { g.group_end(); set_err("ncclAllGather: %s", g.error_string(r)); return -1; }
        }
        const ncclResult_t r = g.group_end();
        if (r != ncclSuccess) { set_err("ncclGroupEnd: %s", g.error_string(r)); return -1; }
    } else {
        TRY(g.recv[0].ensure(blk * n, s0.dev));
        CK(cudaSetDevice(s0.dev));
        for (int i = 0; i < n; ++i) {
            const Shard& s = e->shards[i];
            if (s.count)
                CK(cudaMemcpyPeerAsync(g.recv[0].as<uint8_t>() + blk * i, s0.dev, s.rec.p, s.dev,
                                       sizeof(ltgp_record) * s.count, s0.st));
        }
    }
    CK(cudaSetDevice(s0.dev));
    CK(cudaEventRecord(g.ev[1], s0.st));
    TRY(g.h.ensure(blk * n));
    CK(cudaMemcpyAsync(g.h.p, g.recv[0].p, blk * n, cudaMemcpyDeviceToHost, s0.st));
    for (int i = 1; i < n && g.nccl; ++i) {  // every device holds the array; wait for all
        CK(cudaSetDevice(e->shards[i].dev));
        CK(cudaStreamSynchronize(e->shards[i].st));
    }
    CK(cudaSetDevice(s0.dev));
    CK(cudaStreamSynchronize(s0.st));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, g.ev[0], g.ev[1]));
    e->stats.gather_seconds = ms * 1e-3;
    if (out)
        for (int i = 0; i < n; ++i) {
            const Shard& s = e->shards[i];
            std::memcpy(out + s.first, g.h.as<uint8_t>() + blk * i, sizeof(ltgp_record) * s.count);
        }
    return 0;
}

// One process per GPU (ltgp_nccl_attach): the ranks' records to every rank,
// one ncclAllGather over the engine's own communicator. Ranks must hold equal
// population sizes (a one-process-per-GPU batch: N config-3 batches).
int gather_records_mp(ltgp_engine* e) {
    NvtxRange nr("ltgp.record_all_gather");
    auto& g = e->gather;
    Shard& s = e->shards[0];
    const size_t blk = sizeof(ltgp_record) * std::max<uint32_t>(s.count, 1);
    CK(cudaSetDevice(s.dev));
    TRY(g.recv[0].ensure(blk * g.mp_nranks, s.dev));
    CK(cudaEventRecord(g.ev[0], s.st));
    const ncclResult_t r = g.all_gather(s.rec.p, g.recv[0].p, blk, ncclUint8, g.mp_comm, s.st);
    if (r != ncclSuccess) { set_err("ncclAllGather: %s", g.error_string(r)); return -1; }
    CK(cudaEventRecord(g.ev[1], s.st));
    TRY(g.h.ensure(blk * g.mp_nranks));
    CK(cudaMemcpyAsync(g.h.p, g.recv[0].p, blk * g.mp_nranks, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, g.ev[0], g.ev[1]));
    e->stats.gather_seconds = ms * 1e-3;
    g.mp_count = s.count;
    return 0;
}

int collect(ltgp_engine* e, ltgp_record* out, float* outs48) {
    double secs = 0.0, ksecs = 0.0, csecs = 0.0, kev = 0.0;
    uint64_t nodes = 0, chunks = 0, reruns = 0, exits = 0, adjusts = 0, steps = 0;
    for (Shard& s : e->shards) {
        if (!s.count) continue;
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.st));
        TRY(finish_eval(e, s));
        if (out && e->shards.size() == 1)
            CK(cudaMemcpyAsync(out + s.first, s.rec.p, sizeof(ltgp_record) * s.count,
                               cudaMemcpyDeviceToHost, s.st));
        if (outs48) CK(cudaMemcpyAsync(outs48 + (size_t)s.first * kLanes, s.outs.p,
                                       sizeof(float) * kLanes * s.count, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        float ms = 0.0f;
        // device time of the pass plus any overflow re-run (its k_eval tiers
        // count as evaluation, its recombine replaces the first combine)
        CK(cudaEventElapsedTime(&ms, s.ev[0], s.ev[4]));
        const double k = ms * 1e-3 + s.rerun_ksecs;
        CK(cudaEventElapsedTime(&ms, s.ev[4], s.ev[1]));
        const double cmb = ms * 1e-3 + s.rerun_csecs;
        if (s.kev_valid) {
            CK(cudaEventElapsedTime(&ms, s.kev[0], s.kev[1]));
            kev = std::max(kev, (double)ms * 1e-3);
        }
        secs = std::max(secs, k + cmb);
        ksecs = std::max(ksecs, k);
        csecs = std::max(csecs, cmb);
        const TreeSet& ts = s.set[s.cur];
        for (uint32_t i = 0; i < ts.count; ++i) nodes += ts.h_size[i];
        chunks += s.last_chunks;
        reruns += s.last_reruns;
        exits += s.h_counters.as<uint32_t>()[4];
        adjusts += s.h_counters.as<uint32_t>()[5];
        steps += s.last_steps;
    }
    if (e->shards.size() > 1) TRY(gather_records(e, out));
    else if (e->gather.mp) TRY(gather_records_mp(e));
    e->stats.last_spine_steps = steps;
    e->stats.last_exits = exits;
    e->stats.last_window_adjusts = adjusts;
    e->stats.last_fallback_items = reruns;
    e->stats.eval_seconds = secs;
    e->stats.eval_kernel_seconds = ksecs;
    e->stats.combine_seconds = csecs;
    e->stats.keval_seconds = kev;
    e->stats.nodes_evaluated += nodes;
    e->stats.last_chunks = chunks;
    return 0;
}

}  // namespace

extern "C" {

const char* ltgp_last_error(void) { return g_err.c_str(); }
const char* ltgp_version(void) { return "ltgp_cuda 0.2 (sm_100a)"; }

int ltgp_device_count(int* n) {
    if (!n) { set_err("null argument"); return -1; }
    *n = 0;
    CK(cudaGetDeviceCount(n));
    return 0;
}

int ltgp_engine_create(const ltgp_config* cfg, ltgp_engine** out) {
    if (!cfg || !out) { set_err("null argument"); return -1; }
    if (cfg->n_shards < 1 || cfg->n_shards > LTGP_MAX_SHARDS) { set_err("n_shards out of range"); return -1; }
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int i = 0; i < cfg->n_shards; ++i)
        if (cfg->devices[i] < 0 || cfg->devices[i] >= ndev) {
            set_err("device %d not present (%d visible)", cfg->devices[i], ndev);
            return -1;
        }
    auto e = std::make_unique<ltgp_engine>();
    e->cfg = *cfg;
    if (cfg->chunk_nodes) {
        // <= 2^24: an item's float depth lanes stay exact (ltgp_kernels.cuh)
        if (cfg->chunk_nodes % 16 || cfg->chunk_nodes < 64 || cfg->chunk_nodes > (1u << 24)) {
            set_err("chunk_nodes must be a multiple of 16 in [64, 2^24]");
            return -1;
        }
        e->chunk = cfg->chunk_nodes;
        e->chunk_fixed = true;
    }
    std::memset(&e->stats, 0, sizeof e->stats);
    e->shards.resize(cfg->n_shards);
    for (int i = 0; i < cfg->n_shards; ++i) {
        e->shards[i].dev = cfg->devices[i];
        if (init_shard(e.get(), e->shards[i]) != 0) {
            for (auto& s : e->shards) s.release();
            return -1;
        }
    }
    // peer access between distinct devices (parents are read over NVLink)
    for (int i = 0; i < cfg->n_shards; ++i)
        for (int j = 0; j < cfg->n_shards; ++j) {
            const int a = cfg->devices[i], b = cfg->devices[j];
            if (a == b) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, a, b);
            if (!can) { set_err("no peer access %d -> %d", a, b); return -1; }
            cudaSetDevice(a);
            cudaError_t pe = cudaDeviceEnablePeerAccess(b, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
                set_err("cudaDeviceEnablePeerAccess(%d->%d): %s", a, b, cudaGetErrorString(pe));
                return -1;
            }
            cudaGetLastError();
        }
    if (init_gather(e.get()) != 0) {
        release_gather(e.get());
        for (auto& s : e->shards) s.release();
        return -1;
    }
    *out = e.release();
    return 0;
}

int ltgp_engine_destroy(ltgp_engine* e) {
    if (!e) return 0;
    for (auto& s : e->shards) {
        cudaSetDevice(s.dev);
        if (s.st) cudaStreamSynchronize(s.st);
        s.release();
    }
    release_gather(e);
    e->staging.release();
    if (e->pack) ltgp_pack::pool_destroy(e->pack);
    e->pack = nullptr;
    delete e;
    return 0;
}

int ltgp_generation_stats(ltgp_engine* e, ltgp_gen_stats* out) {
    if (!e || !out) { set_err("null argument"); return -1; }
    if (!e->M) { set_err("no population"); return -1; }
    const size_t kS = sizeof(GenStatsDev);
    // pass 1 per shard: best slot, max size, sums
    for (Shard& s : e->shards) {
        if (!s.count) continue;
        CK(cudaSetDevice(s.dev));
        TRY(s.gstats.ensure(kS + 16, s.dev));
        TRY(s.h_gstats.ensure(kS + 16));
        k_gen_stats<<<1, 1024, 0, s.st>>>(s.rec.as<float>(), s.count, s.gstats.as<GenStatsDev>(), nullptr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(s.h_gstats.p, s.gstats.p, kS, cudaMemcpyDeviceToHost, s.st));
    }
    ltgp_gen_stats r{};
    float bf = 0.0f;
    uint32_t bi = 0xffffffffu, bbits = 0;
    const Shard* bs = nullptr;
    auto better = [](float fa, uint32_t ia, float fb, uint32_t ib) {  // fitness_better + lower slot
        if (fa != fa) return (fb != fb) && ia < ib;
        if (fb != fb) return true;
        return fa < fb || (fa == fb && ia < ib);
    };
    for (Shard& s : e->shards) {  // shards hold consecutive slot ranges: slot order
        if (!s.count) continue;
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.st));
        const GenStatsDev g = *s.h_gstats.as<GenStatsDev>();
        float f;
        std::memcpy(&f, &g.best_bits, 4);
        const uint32_t slot = s.first + g.best_slot;
        if (bi == 0xffffffffu || better(f, slot, bf, bi)) { bf = f; bi = slot; bbits = g.best_bits; bs = &s; }
        r.max_size = std::max(r.max_size, g.max_size);
        r.sum_size += g.sum_size;
        r.sum_depth += g.sum_depth;
        r.sum_fitness += g.sum_fitness;
    }
    // the best record, then pass 2: convergence against the global best's bits
    {
        ltgp_record br;
        CK(cudaSetDevice(bs->dev));
        CK(cudaMemcpy(&br, bs->rec.as<ltgp_record>() + (bi - bs->first), sizeof br, cudaMemcpyDeviceToHost));
        r.best_index = bi;
        r.best_fitness = br.fitness;
        r.best_hits = br.hits;
        r.best_size = br.size;
        r.best_depth = br.depth;
    }
    for (Shard& s : e->shards) {
        if (!s.count) continue;
        CK(cudaSetDevice(s.dev));
        uint32_t* hb = reinterpret_cast<uint32_t*>(s.h_gstats.as<uint8_t>() + kS);
        *hb = bbits;
        uint32_t* db = reinterpret_cast<uint32_t*>(s.gstats.as<uint8_t>() + kS);
        CK(cudaMemcpyAsync(db, hb, 4, cudaMemcpyHostToDevice, s.st));
        k_gen_stats<<<1, 1024, 0, s.st>>>(s.rec.as<float>(), s.count, s.gstats.as<GenStatsDev>(), db);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(s.h_gstats.p, s.gstats.p, kS, cudaMemcpyDeviceToHost, s.st));
    }
    for (Shard& s : e->shards) {
        if (!s.count) continue;
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.st));
        r.convergence += s.h_gstats.as<GenStatsDev>()->convergence;
    }
    *out = r;
    return 0;
}

int ltgp_set_streaming(ltgp_engine* e, int on, uint32_t wave) {
    if (!e) { set_err("null engine"); return -1; }
    if (on && e->shards.size() != 1) { set_err("streaming memory mode needs a single-shard engine"); return -1; }
    e->streaming = on != 0;
    if (wave) e->stream_wave = wave;
    return 0;
}

int ltgp_set_memory_budget(ltgp_engine* e, uint64_t bytes) {
    if (!e) { set_err("null engine"); return -1; }
    e->memory_budget = bytes;
    return 0;
}

int ltgp_set_suite(ltgp_engine* e, const float* in, const float* tg, const float* cs) {
    if (!e || !in || !tg || !cs) { set_err("null argument"); return -1; }
    for (int l = 0; l < 24; ++l) {
        e->suite.x[l] = make_float2(in[2 * l], in[2 * l + 1]);
        e->suite.t[l] = make_float2(tg[2 * l], tg[2 * l + 1]);
    }
    for (int i = 0; i < 256; ++i) e->suite.c[i] = (i >= 5 && i < 255) ? cs[i - 5] : 0.0f;
    e->have_suite = true;
    return 0;
}

}  // extern "C"

namespace {
int check_packed(const ltgp_engine* e, uint32_t M, const uint8_t* buf, uint64_t buf_bytes, const uint64_t* offsets,
                 const uint64_t* sizes) {
    if (!e || (M && (!buf || !offsets || !sizes))) { set_err("null argument"); return -1; }
    for (uint32_t i = 0; i < M; ++i) {
        if (offsets[i] % 16) { set_err("offset of genome %u not 16-aligned", i); return -1; }
        if (i && offsets[i] < offsets[i - 1] + sizes[i - 1]) { set_err("offsets not increasing/overlapping at %u", i); return -1; }
        if (offsets[i] + sizes[i] > buf_bytes) {
            set_err("genome %u exceeds buffer", i);
            return -1;
        }
    }
    return 0;
}
}  // namespace

extern "C" {

int ltgp_upload_packed(ltgp_engine* e, uint32_t M, const uint8_t* buf, uint64_t buf_bytes,
                       const uint64_t* offsets, const uint64_t* sizes) {
    TRY(check_packed(e, M, buf, buf_bytes, offsets, sizes));
    partition(e, M, sizes);
    for (Shard& s : e->shards) {
        s.cur = 0;
        TreeSet& ts = s.set[0];
        if (s.count == 0) { ts.count = 0; continue; }
        const uint64_t base = offsets[s.first];
        std::vector<uint64_t> rel(s.count);
        TRY(set_layout(s, ts, s.count, sizes + s.first, nullptr));
        for (uint32_t i = 0; i < s.count; ++i) ts.h_off[i] = offsets[s.first + i] - base;
        const uint64_t last = s.first + s.count - 1;
        const uint64_t span = std::min<uint64_t>(ceil16(offsets[last] + sizes[last]), buf_bytes) - base;
        TRY(ts.arena.ensure(span + 64, s.dev));
        ts.bytes = span;
        CK(cudaSetDevice(s.dev));
        CK(cudaMemcpyAsync(ts.arena.p, buf + base, span, cudaMemcpyHostToDevice, s.st));
        TRY(upload_tables(s, ts));
    }
    e->M = M;
    return 0;
}

int ltgp_upload_population(ltgp_engine* e, uint32_t M, const uint8_t* const* ops,
                           const uint64_t* sizes) {
    if (!e || (M && (!ops || !sizes))) { set_err("null argument"); return -1; }
    partition(e, M, sizes);
    for (Shard& s : e->shards) {
        s.cur = 0;
        TreeSet& ts = s.set[0];
        if (s.count == 0) { ts.count = 0; continue; }
        TRY(set_layout(s, ts, s.count, sizes + s.first, nullptr));
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.st));
        TRY(e->staging.ensure(ts.bytes + 16));
        uint8_t* h = e->staging.as<uint8_t>();
        for (uint32_t i = 0; i < s.count; ++i) {
            std::memcpy(h + ts.h_off[i], ops[s.first + i], sizes[s.first + i]);
            const uint64_t pad = ceil16(sizes[s.first + i]) - sizes[s.first + i];
            if (pad) std::memset(h + ts.h_off[i] + sizes[s.first + i], 0xff, pad);
        }
        CK(cudaMemcpyAsync(ts.arena.p, h, ts.bytes, cudaMemcpyHostToDevice, s.st));
        TRY(upload_tables(s, ts));  // synchronizes: staging reusable
    }
    e->M = M;
    return 0;
}

int ltgp_evaluate_launch(ltgp_engine* e) {
    if (!e) { set_err("null engine"); return -1; }
    if (!e->have_suite) { set_err("ltgp_set_suite not called"); return -1; }
    for (Shard& s : e->shards)
        if (s.count) TRY(launch_eval(e, s, s.set[s.cur], false));
    return 0;
}

int ltgp_evaluate_collect(ltgp_engine* e, ltgp_record* out, uint64_t* nodes) {
    if (!e) { set_err("null engine"); return -1; }
    const uint64_t before = e->stats.nodes_evaluated;
    TRY(collect(e, out, nullptr));
    if (nodes) *nodes = e->stats.nodes_evaluated - before;
    return 0;
}

int ltgp_evaluate_population(ltgp_engine* e, ltgp_record* out, uint64_t* nodes) {
    TRY(ltgp_evaluate_launch(e));
    return ltgp_evaluate_collect(e, out, nodes);
}

int ltgp_evaluate_packed(ltgp_engine* e, uint32_t M, const uint8_t* buf, uint64_t buf_bytes,
                         const uint64_t* offsets, const uint64_t* sizes, ltgp_record* out, float* outs48) {
    TRY(check_packed(e, M, buf, buf_bytes, offsets, sizes));
    if (!e->have_suite) { set_err("ltgp_set_suite not called"); return -1; }
    partition(e, M, sizes);
    for (Shard& s : e->shards) {
        s.cur = 0;
        TreeSet& ts = s.set[0];
        if (s.count == 0) { ts.count = 0; continue; }
        TRY(set_layout(s, ts, s.count, sizes + s.first, nullptr));
        // slices of ~kSliceBytes at tree boundaries, laid out kSlicePad apart
        const uint64_t base = offsets[s.first];
        const uint64_t last = s.first + s.count - 1;
        const uint64_t end = std::min<uint64_t>(ceil16(offsets[last] + sizes[last]), buf_bytes);
        const uint64_t span = end - base;
        const uint32_t G = (uint32_t)std::min<uint64_t>(max_slices(), std::max<uint64_t>(1, span / slice_bytes()));
        s.slices.clear();
        // the last three slices taper (1/2, 1/4, 1/8 of the others): what is
        // left to evaluate after the final copy is short
        // and so do the first two (1/4, 1/2): the evaluation starts after
        // the first slice is packed and copied
        auto weight = [&](uint32_t g) -> uint64_t {
            if (G >= 8 && g < 2) return 2u << g;
            return G >= 4 && g + 3 >= G ? 8u >> (g + 4 - G) : 8u;
        };
        uint64_t wsum = 0;
        for (uint32_t g = 0; g < G; ++g) wsum += weight(g);
        uint64_t wcum = 0;
        uint32_t t = 0;
        uint64_t dst = 0;
        for (uint32_t g = 0; g < G && t < s.count; ++g) {
            wcum += weight(g);
            const uint64_t goal = base + span * wcum / wsum;
            const uint32_t t0 = t;
            do { ++t; } while (t < s.count && (g == G - 1 || offsets[s.first + t] < goal));
            const uint64_t src = offsets[s.first + t0];
            const uint64_t stop = t < s.count ? offsets[s.first + t] : end;
            s.slices.push_back({t0, src, dst, stop - src});
            for (uint32_t i = t0; i < t; ++i) ts.h_off[i] = dst + (offsets[s.first + i] - src);
            dst = ceil16(dst + (stop - src)) + kSlicePad;
        }
        const Slice& ls = s.slices.back();
        ts.bytes = ls.dst + ls.len;
        TRY(ts.arena.ensure(ts.bytes + 64, s.dev));
        s.h2d_bytes = 0;
        if (pack_enabled()) {  // packed transfer: worst-case regions per slice
            if (!e->pack) e->pack = ltgp_pack::pool_create(pack_threads());
            uint64_t o = 0;
            for (Slice& sl : s.slices) {
                sl.pk_off = o;  // 64-B aligned: the packer's non-temporal stores
                o += ltgp_pack::ceil64(ltgp_pack::Layout(sl.len).max_bytes());
            }
            TRY(s.pk_host.ensure(o));
            TRY(s.pk_dev.ensure(o, s.dev));
        }
        TRY(upload_tables(s, ts));
        s.src = buf;
        const int rc = launch_eval(e, s, ts, outs48 != nullptr);
        if (rc == 0 && trace_slices()) {
            CK(cudaStreamSynchronize(s.st));
            float t[3], tot = 0.0f;
            CK(cudaEventElapsedTime(&tot, s.ev[0], s.ev[1]));
            std::fprintf(stderr, "ltgp trace: %zu slices, %.3f ms to the last record\n", s.slices.size(), tot);
            for (size_t g = 0; g < s.slices.size(); ++g) {
                for (int k = 0; k < 3; ++k) CK(cudaEventElapsedTime(&t[k], s.ev[0], s.sev[3 * g + k]));
                std::fprintf(stderr, "  slice %2zu: %7.2f MB, %3u trees, copied %7.3f planned %7.3f evaluated %7.3f\n", g,
                             s.slices[g].len / 1e6,
                             (g + 1 < s.slices.size() ? s.slices[g + 1].tree_begin : s.count) - s.slices[g].tree_begin,
                             t[0], t[1], t[2]);
            }
            if (s.xtime.p) {  // cross-slice launch: device time of each slice's phases after the launch began
                std::vector<unsigned long long> xt(1 + 3 * kMaxSlices);
                CK(cudaMemcpy(xt.data(), s.xtime.p, 8 * xt.size(), cudaMemcpyDeviceToHost));
                for (size_t g = 0; g < s.slices.size(); ++g)
                    std::fprintf(stderr, "  xs slice %2zu: decoded %7.3f planned %7.3f evaluated %7.3f (ms after launch)\n", g,
                                 (xt[1 + 3 * g] - xt[0]) * 1e-6, (xt[2 + 3 * g] - xt[0]) * 1e-6, (xt[3 + 3 * g] - xt[0]) * 1e-6);
            }
        }
        s.slices.clear();
        s.src = nullptr;
        TRY(rc);
    }
    e->M = M;
    e->stats.last_h2d_bytes = 0;
    for (const Shard& s : e->shards) e->stats.last_h2d_bytes += s.h2d_bytes;
    return collect(e, out, outs48);
}

int ltgp_nccl_unique_id(uint8_t* out128) {
    if (!out128) { set_err("null argument"); return -1; }
    static ltgp_engine::Gather g;  // the library only
    TRY(open_nccl(g));
    auto get_id = reinterpret_cast<ncclResult_t (*)(ncclUniqueId*)>(dlsym(g.lib, "ncclGetUniqueId"));
    if (!get_id) { set_err("libnccl.so.2 lacks ncclGetUniqueId"); return -1; }
    ncclUniqueId id;
    const ncclResult_t r = get_id(&id);
    if (r != ncclSuccess) { set_err("ncclGetUniqueId: %s", g.error_string(r)); return -1; }
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL_UNIQUE_ID_BYTES");
    std::memcpy(out128, &id, 128);
    return 0;
}

int ltgp_nccl_attach(ltgp_engine* e, const uint8_t* id128, int nranks, int rank) {
    if (!e || !id128) { set_err("null argument"); return -1; }
    if (e->shards.size() != 1) { set_err("ltgp_nccl_attach: one shard (one GPU) per process"); return -1; }
    if (nranks < 1 || rank < 0 || rank >= nranks) { set_err("ltgp_nccl_attach: rank %d of %d", rank, nranks); return -1; }
    auto& g = e->gather;
    if (g.mp) { set_err("ltgp_nccl_attach: already attached"); return -1; }
    TRY(open_nccl(g));
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    CK(cudaSetDevice(e->shards[0].dev));
    const ncclResult_t r = g.comm_init_rank(&g.mp_comm, nranks, id, rank);
    if (r != ncclSuccess) { set_err("ncclCommInitRank: %s", g.error_string(r)); return -1; }
    g.mp = true;
    g.mp_rank = rank;
    g.mp_nranks = nranks;
    std::fprintf(stderr, "[ltgp] NCCL record all-gather across processes: ncclCommInitRank nranks=%d rank=%d device=%d\n",
                 nranks, rank, e->shards[0].dev);
    return 0;
}

int ltgp_gathered_records(ltgp_engine* e, ltgp_record* out, uint32_t cap, uint32_t* n) {
    if (!e || !n) { set_err("null argument"); return -1; }
    const auto& g = e->gather;
    if (!g.mp) { set_err("ltgp_gathered_records: not attached (ltgp_nccl_attach)"); return -1; }
    const uint32_t total = g.mp_count * (uint32_t)g.mp_nranks;
    *n = total;
    if (out) {
        if (cap < total) { set_err("ltgp_gathered_records: %u records, room for %u", total, cap); return -1; }
        const size_t blk = sizeof(ltgp_record) * std::max<uint32_t>(g.mp_count, 1);
        for (int r = 0; r < g.mp_nranks; ++r)
            std::memcpy(out + (size_t)r * g.mp_count, g.h.as<uint8_t>() + blk * r, sizeof(ltgp_record) * g.mp_count);
    }
    return 0;
}

uint64_t ltgp_pack_bound(uint64_t len) { return ltgp_pack::Layout(len).max_bytes(); }

uint64_t ltgp_pack_host(const uint8_t* src, uint64_t len, uint8_t* dst, int threads) {
    if ((!src && len) || !dst) { set_err("null argument"); return 0; }
    ltgp_pack::Pool* P = ltgp_pack::pool_create(std::max(1, threads));
    const uint64_t n = ltgp_pack::pack(P, src, len, dst);
    ltgp_pack::pool_destroy(P);
    return n;
}

int ltgp_evaluate_outputs(ltgp_engine* e, ltgp_record* out, float* outs48) {
    if (!e) { set_err("null engine"); return -1; }
    if (!e->have_suite) { set_err("ltgp_set_suite not called"); return -1; }
    for (Shard& s : e->shards)
        if (s.count) TRY(launch_eval(e, s, s.set[s.cur], true));
    return collect(e, out, outs48);
}

int ltgp_eval_one(ltgp_engine* e, const uint8_t* ops, uint64_t n, float* out48) {
    return ltgp_eval_one_record(e, ops, n, out48, nullptr);
}

int ltgp_eval_one_record(ltgp_engine* e, const uint8_t* ops, uint64_t n, float* out48, ltgp_record* rec) {
    if (!e || !ops || !out48) { set_err("null argument"); return -1; }
    if (n == 0) { set_err("empty genome"); return -1; }
    if (!e->have_suite) { set_err("ltgp_set_suite not called"); return -1; }
    Shard& s = e->shards[0];
    TreeSet& ts = s.scratch;
    uint64_t sz = n;
    TRY(set_layout(s, ts, 1, &sz, nullptr));
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.st));
    TRY(e->staging.ensure(ceil16(n) + 16));
    uint8_t* h = e->staging.as<uint8_t>();
    std::memcpy(h, ops, n);
    std::memset(h + n, 0xff, ceil16(n) - n);
    CK(cudaMemcpyAsync(ts.arena.p, h, ceil16(n), cudaMemcpyHostToDevice, s.st));
    TRY(upload_tables(s, ts));
    TRY(launch_eval(e, s, ts, true));
    CK(cudaStreamSynchronize(s.st));
    TRY(finish_eval(e, s));
    CK(cudaMemcpyAsync(out48, s.outs.p, sizeof(float) * kLanes, cudaMemcpyDeviceToHost, s.st));
    if (rec) CK(cudaMemcpyAsync(rec, s.rec.p, sizeof(ltgp_record), cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    float ms = 0.0f;  // device time of this evaluation (launch_eval brackets it with ev[0] / ev[1])
    CK(cudaEventElapsedTime(&ms, s.ev[0], s.ev[1]));
    e->stats.eval_seconds = ms * 1e-3 + s.rerun_ksecs + s.rerun_csecs;
    e->stats.nodes_evaluated += n;
    return 0;
}

int ltgp_get_stats(ltgp_engine* e, ltgp_stats* out) {
    if (!e || !out) { set_err("null argument"); return -1; }
    uint64_t hw = 0;
    for (Shard& s : e->shards)
        for (auto& ts : s.set) hw = std::max<uint64_t>(hw, ts.arena.bytes);
    e->stats.arena_high_water = hw;
    e->stats.gather_nccl = e->gather.mp ? 2u : e->gather.nccl ? 1u : 0u;
    e->stats.live_genomes_high_water = e->live_high_water;
    e->stats.arena_used_high_water = e->used_high_water;
    *out = e->stats;
    return 0;
}

uint32_t ltgp_population_size(ltgp_engine* e) { return e ? e->M : 0; }

int ltgp_shard_records(ltgp_engine* e, int s, void** dev_records, uint32_t* first, uint32_t* count,
                       void** stream) {
    if (!e || s < 0 || s >= (int)e->shards.size()) { set_err("bad shard"); return -1; }
    Shard& sh = e->shards[s];
    if (dev_records) *dev_records = sh.rec.p;
    if (first) *first = sh.first;
    if (count) *count = sh.count;
    if (stream) *stream = (void*)sh.st;
    return 0;
}

int ltgp_download_genome(ltgp_engine* e, uint32_t idx, uint8_t* buf, uint64_t cap, uint64_t* size) {
    if (!e || !size) { set_err("null argument"); return -1; }
    for (Shard& s : e->shards) {
        if (idx < s.first || idx >= s.first + s.count) continue;
        const TreeSet& ts = s.set[s.cur];
        const uint32_t i = idx - s.first;
        *size = ts.h_size[i];
        if (!buf || cap < ts.h_size[i]) return 0;
        CK(cudaSetDevice(s.dev));
        CK(cudaMemcpyAsync(buf, ts.arena.as<uint8_t>() + ts.h_off[i], ts.h_size[i],
                           cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        return 0;
    }
    set_err("slot %u out of range (M=%u)", idx, e->M);
    return -1;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Crossover on device: execute_generation (evolve.hpp:111-117).
// ---------------------------------------------------------------------------


namespace {

// Directory of the current population: per global slot, its device address
// and size (parents may be read from any shard's GPU).
int build_directory(ltgp_engine* e, std::vector<DirEntry>& dir) {
    dir.assign(e->M, DirEntry{nullptr, 0});
    for (Shard& s : e->shards) {
        const TreeSet& ts = s.set[s.cur];
        for (uint32_t i = 0; i < s.count; ++i)
            dir[s.first + i] = DirEntry{ts.arena.as<uint8_t>() + ts.h_off[i], ts.h_size[i]};
    }
    return 0;
}

int upload_directory(ltgp_engine* e, Shard& s, const std::vector<DirEntry>& dir) {
    CK(cudaSetDevice(s.dev));
    TRY(s.dir.ensure(sizeof(DirEntry) * std::max<size_t>(dir.size(), 1), s.dev));
    TRY(s.h_dir.ensure(sizeof(DirEntry) * std::max<size_t>(dir.size(), 1)));
    CK(cudaStreamSynchronize(s.st));
    std::memcpy(s.h_dir.p, dir.data(), sizeof(DirEntry) * dir.size());
    CK(cudaMemcpyAsync(s.dir.p, s.h_dir.p, sizeof(DirEntry) * dir.size(), cudaMemcpyHostToDevice, s.st));
    (void)e;
    return 0;
}

}  // namespace

extern "C" {

// Streaming memory mode (RunConfig::streaming_memory, evolve.hpp:45,
// :111-114): the paper's "specialised
// heap for the population". Children are placed, in plan order and in waves
// of stream_wave, into the parents' own arena by first fit over its free
// intervals; after the wave that holds a parent's last planned use, the
// parent's bytes join the free list (released in the sequential coordinator,
// as SPEC.md:392 asks: here the host computes the whole placement before
// any kernel runs, since every child size is known from the crossover
// algebra). Waves splice in stream order, so a wave never overwrites a
// parent an earlier or the same wave still reads. Live genomes (parents not
// yet retired + children built) and arena bytes in use are tracked at every
// wave: live_high_water / used_high_water.
static int splice_streaming(ltgp_engine* e, const ltgp_plan* plans, uint32_t M, const std::vector<uint64_t>& csize) {
    Shard& s = e->shards[0];
    TreeSet& ts = s.set[s.cur];
    const uint32_t P = ts.count;  // parents
    const uint32_t W = std::max<uint32_t>(1, e->stream_wave);
    std::vector<int64_t> last(P, -1);
    for (uint32_t c = 0; c < M; ++c) {
        last[plans[c].mum_index] = c;
        last[plans[c].dad_index] = c;
    }
    // free intervals [start, end), address ordered; the tail is unbounded
    std::map<uint64_t, uint64_t> fr;
    {
        std::vector<std::pair<uint64_t, uint64_t>> occ(P);
        for (uint32_t i = 0; i < P; ++i) occ[i] = {ts.h_off[i], ts.h_off[i] + ceil16(ts.h_size[i])};
        std::sort(occ.begin(), occ.end());
        uint64_t at = 0;
        for (const auto& o : occ) {
            if (o.first > at) fr[at] = o.first;
            at = std::max(at, o.second);
        }
        fr[at] = ~0ull;
    }
    auto release = [&](uint64_t a, uint64_t b) {
        auto it = fr.lower_bound(a);
        if (it != fr.end() && it->first == b) {  // merge with the next interval
            b = it->second;
            it = fr.erase(it);
        }
        if (it != fr.begin()) {
            auto pv = std::prev(it);
            if (pv->second == a) {  // merge with the previous interval
                pv->second = b;
                return;
            }
        }
        fr[a] = b;
    };
    std::vector<std::vector<uint32_t>> retire((M + W - 1) / W + 1);
    for (uint32_t p = 0; p < P; ++p) retire[last[p] < 0 ? 0 : (uint32_t)(last[p] / W) + 1].push_back(p);
    uint64_t live_bytes = 0;
    for (uint32_t i = 0; i < P; ++i) live_bytes += ceil16(ts.h_size[i]);
    int64_t live = P;
    uint64_t used_hw = live_bytes, end = 0;
    int64_t live_hw = live;
    for (uint32_t p : retire[0]) {  // parents no plan uses
        release(ts.h_off[p], ts.h_off[p] + ceil16(ts.h_size[p]));
        live_bytes -= ceil16(ts.h_size[p]);
        --live;
    }
    for (uint32_t i = 0; i < P; ++i) end = std::max<uint64_t>(end, ts.h_off[i] + ceil16(ts.h_size[i]));
    std::vector<uint64_t> coff(M);
    for (uint32_t w0 = 0, wi = 1; w0 < M; w0 += W, ++wi) {
        const uint32_t w1 = std::min(M, w0 + W);
        for (uint32_t c = w0; c < w1; ++c) {
            const uint64_t need = ceil16(csize[c]);
            auto it = fr.begin();
            while (it->second - it->first < need) ++it;  // the tail interval always fits
            coff[c] = it->first;
            const uint64_t a = it->first + need, b = it->second;
            fr.erase(it);
            if (a < b) fr[a] = b;
            end = std::max(end, coff[c] + need);
            live_bytes += need;
            ++live;
        }
        live_hw = std::max(live_hw, live);
        used_hw = std::max(used_hw, live_bytes);
        for (uint32_t p : retire[wi]) {  // last planned use was in this wave
            release(ts.h_off[p], ts.h_off[p] + ceil16(ts.h_size[p]));
            live_bytes -= ceil16(ts.h_size[p]);
            --live;
        }
    }
    e->live_high_water = std::max<uint64_t>(e->live_high_water, (uint64_t)live_hw);
    e->used_high_water = std::max<uint64_t>(e->used_high_water, used_hw);
    CK(cudaSetDevice(s.dev));
    // the arena must hold the placement; growing keeps the parents' bytes
    const uint64_t need_bytes = end + 64;
    if (need_bytes > ts.arena.bytes) {
        DevBuf grown;
        TRY(grown.ensure(need_bytes, s.dev));
        CK(cudaMemcpyAsync(grown.p, ts.arena.p, ts.arena.bytes, cudaMemcpyDeviceToDevice, s.st));
        CK(cudaStreamSynchronize(s.st));
        ts.arena.release();
        ts.arena = grown;
        grown.p = nullptr;  // owned by ts.arena now
        std::vector<DirEntry> dir;  // the parents moved: rebuild the directory
        build_directory(e, dir);
        TRY(upload_directory(e, s, dir));
    }
    TRY(s.coff.ensure(sizeof(uint64_t) * M, s.dev));
    TRY(s.h_coff.ensure(sizeof(uint64_t) * M * 2));
    uint8_t* hb = s.h_coff.as<uint8_t>();
    std::memcpy(hb, coff.data(), sizeof(uint64_t) * M);
    std::memcpy(hb + 8 * (size_t)M, csize.data(), sizeof(uint64_t) * M);
    CK(cudaMemcpyAsync(s.coff.p, hb, 8 * (size_t)M, cudaMemcpyHostToDevice, s.st));
    CK(cudaMemcpyAsync(s.csize.p, hb + 8 * (size_t)M, 8 * (size_t)M, cudaMemcpyHostToDevice, s.st));
    CK(cudaEventRecord(s.ev[2], s.st));
    {
        NvtxRange nr("ltgp.splice_streaming");
        for (uint32_t w0 = 0; w0 < M; w0 += W) {  // waves in stream order
            const uint32_t n = std::min(M, w0 + W) - w0;
            k_splice<<<std::min<uint32_t>(n, (uint32_t)s.sms * 8), 256, 0, s.st>>>(
                s.plans.as<PlanDev>() + w0, n, s.dir.as<DirEntry>(), s.ext.as<Extent>() + w0,
                s.coff.as<uint64_t>() + w0, s.csize.as<uint64_t>() + w0, ts.arena.as<uint8_t>(), nullptr);
            CK(cudaGetLastError());
        }
    }
    CK(cudaEventRecord(s.ev[3], s.st));
    // the children become the population, in the same arena
    ts.version = ++g_version;
    ts.count = M;
    ts.h_off.assign(coff.begin(), coff.end());
    ts.h_size.resize(M);
    for (uint32_t c = 0; c < M; ++c) ts.h_size[c] = (uint32_t)csize[c];
    ts.bytes = end;
    TRY(ts.off.ensure(sizeof(uint64_t) * std::max<uint32_t>(M, 1), s.dev));
    TRY(ts.size.ensure(sizeof(uint32_t) * std::max<uint32_t>(M, 1), s.dev));
    CK(cudaMemcpyAsync(ts.off.p, ts.h_off.data(), sizeof(uint64_t) * M, cudaMemcpyHostToDevice, s.st));
    CK(cudaMemcpyAsync(ts.size.p, ts.h_size.data(), sizeof(uint32_t) * M, cudaMemcpyHostToDevice, s.st));
    s.first = 0;
    s.count = M;
    CK(cudaStreamSynchronize(s.st));  // the host vectors above back async copies
    return 0;
}

// Device-resident generation:
// single shard, double-buffered. One launch sequence on s.st, captured as a
// CUDA graph (one per parity of s.cur; LTGP_GEN_GRAPH=0: plain launches):
//   plans H2D -> k_gen_dir -> k_extent -> k_gen_control (child sizes,
//   layout, budget / size-limit / capacity checks, chunk length, work-list
//   bases) -> k_gen_items -> k_splice -> k_plan_warp -> k_eval -> k_cpops ->
//   k_caddr -> k_combine -> status, counters, records and the children's
//   layout D2H
// and one synchronisation. Every kernel after k_gen_control reads its counts
// (or its skip word) from the device status, so a generation that hits a
// limit splices and evaluates nothing. Capacities are grow-only buffers
// sized from the previous generation; a generation that outgrows the
// children's arena returns 1 (the host path runs it, growing the arena); one
// whose work list outgrows its buffers is evaluated by the host path's
// launch_eval after the device splice.
static bool gen_graph_enabled() {
    static const bool v = !(std::getenv("LTGP_GEN_GRAPH") && std::atoi(std::getenv("LTGP_GEN_GRAPH")) == 0);
    return v;
}
static bool device_generation_enabled() {
    static const bool v = !(std::getenv("LTGP_DEVICE_GEN") && std::atoi(std::getenv("LTGP_DEVICE_GEN")) == 0);
    return v;
}

static int gen_device_launch(ltgp_engine* e, const ltgp_plan* plans, uint32_t M) {
    Trace tr("ltgp.execute_generation_device");
    Shard& s = e->shards[0];
    TreeSet& par = s.set[s.cur];
    TreeSet& ch = s.set[1 - s.cur];
    CK(cudaSetDevice(s.dev));
    // --- capacities (grow-only; estimates from the parents and the last evaluation)
    TRY(ch.arena.ensure(std::max<uint64_t>(par.bytes + par.bytes / 4, 4096) + 64, s.dev));
    TRY(ch.off.ensure(sizeof(uint64_t) * M, s.dev));
    TRY(ch.size.ensure(sizeof(uint32_t) * M, s.dev));
    const uint64_t packets = ch.arena.bytes / 16;
    TRY(ch.decode.ensure(packets * 32 + 1024, s.dev));
    TRY(ch.meta.ensure(64, s.dev));  // k_plan_warp<true> decodes itself: no metadata pass
    TRY(s.plans.ensure(sizeof(PlanDev) * M, s.dev));
    TRY(s.ext.ensure(sizeof(Extent) * M, s.dev));
    TRY(s.csize.ensure(sizeof(uint64_t) * M, s.dev));
    TRY(s.dir.ensure(sizeof(DirEntry) * M, s.dev));
    TRY(s.gen_status.ensure(sizeof(GenStatus), s.dev));
    TRY(s.gen_tree.ensure(sizeof(uint32_t) * 2 * M, s.dev));
    TRY(s.items.ensure(sizeof(Item) * ((uint64_t)s.last_items + s.last_items / 2 + M + 1024), s.dev));
    const uint32_t items_cap = (uint32_t)std::min<uint64_t>(s.items.bytes / sizeof(Item), 0xffffffffu);
    TRY(s.ovf.ensure(sizeof(uint32_t) * items_cap, s.dev));
    const uint64_t chunks_want = (uint64_t)s.last_chunks + s.last_chunks / 2 + 1024;
    TRY(s.hdr.ensure(sizeof(ChunkHdr) * chunks_want, s.dev));
    TRY(s.dframes.ensure((size_t)kFrameBytes * chunks_want, s.dev));
    TRY(s.segs.ensure(sizeof(Seg) * 2 * chunks_want, s.dev));
    TRY(s.runs.ensure(sizeof(PopRun) * 3 * chunks_want, s.dev));
    TRY(s.cch.ensure(sizeof(CombChunk) * chunks_want, s.dev));
    const uint32_t chunks_cap = (uint32_t)std::min<uint64_t>(
        {s.hdr.bytes / sizeof(ChunkHdr), s.dframes.bytes / kFrameBytes, s.segs.bytes / (2 * sizeof(Seg)),
         s.runs.bytes / (3 * sizeof(PopRun)), s.cch.bytes / sizeof(CombChunk), 0xffffffffull});
    TRY(s.ctrees.ensure(sizeof(CombineTree) * M, s.dev));
    TRY(s.cres.ensure(sizeof(CombResult) * M, s.dev));
    {   // chunk-summary pool: launch_eval's estimate at the last chunk length
        const double rc = std::sqrt((double)s.cur_chunk);
        const double pf = std::max(std::min(2.0 * rc, (double)s.cur_chunk + 2), s.pool_per_chunk_f * 1.25);
        const double ps = std::max(std::min(2.0 * rc, (double)s.cur_chunk), s.pool_per_chunk_s * 1.25);
        TRY(s.frames.ensure((size_t)((pf * chunks_want + 64) * kFrameBytes), s.dev));
        TRY(s.steps.ensure((size_t)(ps * chunks_want + 1024), s.dev));
        TRY(s.saddr.ensure(s.steps.bytes * 8, s.dev));
    }
    TRY(s.rec.ensure(sizeof(ltgp_record) * M, s.dev));
    const uint32_t sf = spill_frames(s.cur_chunk);
    TRY(s.spill.ensure((size_t)s.eval_grid * kWarps * sf * kFrameBytes, s.dev));
    // pinned staging: plans | status | counters | records | child offsets | child sizes
    const size_t o_st = (sizeof(PlanDev) * M + 255) & ~size_t(255);
    const size_t o_cnt = o_st + ((sizeof(GenStatus) + 255) & ~size_t(255));
    const size_t o_rec = o_cnt + 256;
    const size_t o_off = o_rec + sizeof(ltgp_record) * M;
    const size_t o_size = o_off + sizeof(uint64_t) * M;
    TRY(s.h_gen.ensure(o_size + sizeof(uint32_t) * M));
    uint8_t* hg = s.h_gen.as<uint8_t>();
    tr.mark("capacities");
    // --- arguments
    GenStatus* st = s.gen_status.as<GenStatus>();
    GenArgs ga{};
    ga.plans = s.plans.as<PlanDev>();
    ga.dir = s.dir.as<DirEntry>();
    ga.ext = s.ext.as<Extent>();
    ga.ext_err = s.counters.as<uint32_t>() + 3;
    ga.M = M;
    ga.node_limit = e->cfg.node_limit;
    ga.budget = e->memory_budget;
    ga.arena_cap = ch.arena.bytes;
    ga.csize = s.csize.as<uint64_t>();
    ga.child_off = ch.off.as<uint64_t>();
    ga.child_size = ch.size.as<uint32_t>();
    ga.tree_chunk0 = s.gen_tree.as<uint32_t>();
    ga.tree_ct = s.gen_tree.as<uint32_t>() + M;
    ga.items = s.items.as<Item>();
    ga.items_cap = items_cap;
    ga.ctrees = s.ctrees.as<CombineTree>();
    ga.chunks_cap = chunks_cap;
    ga.fixed_chunk = e->chunk_fixed ? e->chunk : 0u;
    ga.default_chunk = kDefaultChunk;
    ga.max_chunk = kMaxChunk;
    ga.max_wave_chunk = kMaxWaveChunk;
    ga.grid_warps = (uint32_t)s.eval_grid * kWarps;
    ga.st = st;
    PlanPool pool{};
    pool.hdr = s.hdr.as<ChunkHdr>();
    pool.frames = s.frames.as<float2>();
    pool.steps = s.steps.as<uint8_t>();
    pool.used = reinterpret_cast<unsigned long long*>(s.counters.as<uint32_t>() + kPoolCounters);
    pool.cap_frames = s.frames.bytes / kFrameBytes;
    pool.cap_steps = s.steps.bytes;
    pool.spill_frames = sf;
    pool.adjusts = s.counters.as<uint32_t>() + 5;
    pool.flags = s.counters.as<uint32_t>() + 1;
    EvalArgs a{};
    a.arena = ch.arena.as<uint8_t>();
    a.decode = ch.decode.as<uint4>();
    a.off = ch.off.as<uint64_t>();
    a.size = ch.size.as<uint32_t>();
    a.items = s.items.as<Item>();
    a.n_items = 0;
    a.n_items_dev = &st->n_items;
    a.counters = s.counters.as<uint32_t>();
    a.hdr = s.hdr.as<ChunkHdr>();
    a.steps = s.steps.as<uint8_t>();
    a.frames = s.frames.as<float2>();
    a.max_steps = 0xffffffffu;
    a.max_frames = 0xffffffffu;
    a.spill = s.spill.as<float2>();
    a.spill_frames = sf;
    a.rec = s.rec.as<float>();
    a.outs = nullptr;
    a.slot = nullptr;
    a.packets = packets;
    a.ovf = s.ovf.as<uint32_t>();
    a.queue = s.counters.as<uint32_t>();
    a.item_base = 0;
    CombineArgs ca{};
    ca.trees = s.ctrees.as<CombineTree>();
    ca.counts_dev = &st->n_trees;
    ca.hdr = s.hdr.as<ChunkHdr>();
    ca.chunk0 = 0;
    ca.dframes = s.dframes.as<float2>();
    ca.segs = s.segs.as<Seg>();
    ca.runs = s.runs.as<PopRun>();
    ca.cch = s.cch.as<CombChunk>();
    ca.cres = s.cres.as<CombResult>();
    ca.space[0] = StepSpace{s.steps.as<uint8_t>(), pool.cap_steps, s.saddr.as<uint64_t>()};
    ca.space[1] = ca.space[2] = StepSpace{nullptr, 0, nullptr};
    ca.rec = s.rec.as<float>();
    ca.outs = nullptr;
    ca.counters = s.counters.as<uint32_t>();
    const uint32_t seg_cap = kCpopsSmem / (uint32_t)sizeof(Seg);
    const unsigned plan_blocks = (items_cap + 3) / 4;
    const unsigned cblocks = std::min<unsigned>((M + kCombineWarps - 1) / kCombineWarps, (unsigned)s.sms * 16);
    const unsigned ablocks = (unsigned)s.sms * 16;
    // --- the launch sequence (recorded into a graph, or issued directly)
    const bool graph = gen_graph_enabled();
    auto record = [&](cudaEvent_t ev) {
        return graph ? cudaEventRecordWithFlags(ev, s.st, cudaEventRecordExternal) : cudaEventRecord(ev, s.st);
    };
    auto issue = [&]() -> int {
        CK(cudaMemcpyAsync(s.plans.p, hg, sizeof(PlanDev) * M, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemsetAsync(s.counters.p, 0, kCounterBytes, s.st));
        k_gen_dir<<<(M + 255) / 256, 256, 0, s.st>>>(par.arena.as<uint8_t>(), par.off.as<uint64_t>(),
                                                     par.size.as<uint32_t>(), M, s.dir.as<DirEntry>());
        CK(cudaGetLastError());
        k_extent<<<(2 * M + 3) / 4, 128, 0, s.st>>>(s.plans.as<PlanDev>(), M, s.dir.as<DirEntry>(), s.ext.as<Extent>(),
                                                  nullptr, s.counters.as<uint32_t>() + 3);
        CK(cudaGetLastError());
        k_gen_control<<<1, 1024, 0, s.st>>>(ga);
        CK(cudaGetLastError());
        k_gen_items<<<(M + 7) / 8, 256, 0, s.st>>>(ga);
        CK(cudaGetLastError());
        CK(record(s.ev[2]));
        k_splice<<<std::min<uint32_t>(M, (uint32_t)s.sms * 8), 256, 0, s.st>>>(
            s.plans.as<PlanDev>(), M, s.dir.as<DirEntry>(), s.ext.as<Extent>(), ch.off.as<uint64_t>(),
            s.csize.as<uint64_t>(), ch.arena.as<uint8_t>(), &st->fatal);
        CK(cudaGetLastError());
        CK(record(s.ev[3]));
        CK(record(s.ev[0]));
        k_plan_warp<true><<<plan_blocks, 128, 0, s.st>>>(s.items.as<Item>(), 0u, &st->n_items, ch.off.as<uint64_t>(),
                                                         reinterpret_cast<uint8_t*>(ch.decode.p), ch.meta.as<uint32_t>(),
                                                         ch.arena.as<uint4>(), packets, kWindow, pool);
        CK(cudaGetLastError());
        CK(record(s.kev[0]));
        K_EVAL<<<s.eval_grid, kWarps * 32, eval_smem_bytes(), s.st>>>(a, e->suite);
        CK(cudaGetLastError());
        CK(record(s.kev[1]));
        CK(record(s.ev[4]));
        k_cpops<<<M, 32, seg_cap * sizeof(Seg), s.st>>>(ca, seg_cap);
        CK(cudaGetLastError());
        k_caddr<<<ablocks, 128, 0, s.st>>>(ca);
        CK(cudaGetLastError());
        k_combine<<<cblocks, kCombineWarps * 32, 0, s.st>>>(ca, e->suite);
        CK(cudaGetLastError());
        CK(record(s.ev[1]));
        CK(cudaMemcpyAsync(hg + o_st, st, sizeof(GenStatus), cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(hg + o_cnt, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(hg + o_rec, s.rec.p, sizeof(ltgp_record) * M, cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(hg + o_off, ch.off.p, sizeof(uint64_t) * M, cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(hg + o_size, ch.size.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToHost, s.st));
        return 0;
    };
    std::memcpy(hg, plans, sizeof(PlanDev) * M);
    tr.mark("arguments");
    if (graph) {
        // the graph bakes in every argument: re-capture when one changes
        std::vector<uint8_t> sig;
        auto add = [&](const void* p, size_t n) {
            const uint8_t* b = static_cast<const uint8_t*>(p);
            sig.insert(sig.end(), b, b + n);
        };
        const void* ptrs[] = {par.arena.p, par.off.p, par.size.p, hg, s.spill.p};
        add(&ga, sizeof ga); add(&pool, sizeof pool); add(&a, sizeof a); add(&ca, sizeof ca);
        add(&e->suite, sizeof e->suite); add(ptrs, sizeof ptrs); add(&s.eval_grid, sizeof s.eval_grid);
        cudaGraphExec_t& ex = s.gen_exec[s.cur];
        if (!ex || s.gen_sig[s.cur] != sig) {
            if (ex) { cudaGraphExecDestroy(ex); ex = nullptr; }
            cudaGraph_t g = nullptr;
            CK(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeThreadLocal));
            const int r = issue();
            const cudaError_t ce = cudaStreamEndCapture(s.st, &g);
            if (r != 0) { if (g) cudaGraphDestroy(g); return -1; }
            CK(ce);
            const cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
            cudaGraphDestroy(g);
            CK(ie);
            s.gen_sig[s.cur] = std::move(sig);
            tr.mark("capture");
        }
        CK(cudaGraphLaunch(ex, s.st));
    } else {
        TRY(issue());
    }
    auto& gp = s.genp;
    gp.o_st = o_st; gp.o_cnt = o_cnt; gp.o_rec = o_rec; gp.o_off = o_off; gp.o_size = o_size;
    gp.a = a;
    gp.ca = ca;
    tr.mark("launch");
    return 0;
}

// The launched generation's outcome (after one synchronisation). Returns 1
// when the host path must run the generation instead (arena grown).
static int gen_device_finish(ltgp_engine* e, uint32_t M, ltgp_record* out, int* size_limit_hit) {
    Trace tr("ltgp.execute_generation_device");
    Shard& s = e->shards[0];
    TreeSet& ch = s.set[1 - s.cur];
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.st));
    tr.mark("sync");
    const auto& gp = s.genp;
    const size_t o_st = gp.o_st, o_cnt = gp.o_cnt, o_rec = gp.o_rec, o_off = gp.o_off, o_size = gp.o_size;
    const EvalArgs& a = gp.a;
    const CombineArgs& ca = gp.ca;
    const uint8_t* hg = s.h_gen.as<uint8_t>();
    // --- outcome
    const GenStatus g = *reinterpret_cast<const GenStatus*>(hg + o_st);
    std::memcpy(s.h_counters.p, hg + o_cnt, 64);
    if (g.fatal & 32u) { set_err("malformed parent genome in extent scan"); return -1; }
    if (g.fatal & 2u) { *size_limit_hit = 2; return 0; }  // MemoryBudgetExceeded: nothing was built
    if (g.fatal & 1u) { *size_limit_hit = 1; return 0; }  // SizeLimitHit
    if (g.fatal & 4u) {
        set_err("child of %llu nodes: beyond the engine's 2^32-1-node tree capacity (node_limit %llu)",
                (unsigned long long)g.max_child, (unsigned long long)e->cfg.node_limit);
        return -1;
    }
    if (g.fatal & 8u) {  // the children need a larger arena: grow it, the host path runs this generation
        TRY(ch.arena.ensure(g.child_bytes + 64, s.dev));
        return 1;
    }
    // the children (spliced) become the population
    ch.version = ++g_version;
    ch.count = M;
    ch.h_off.assign(reinterpret_cast<const uint64_t*>(hg + o_off), reinterpret_cast<const uint64_t*>(hg + o_off) + M);
    ch.h_size.assign(reinterpret_cast<const uint32_t*>(hg + o_size),
                     reinterpret_cast<const uint32_t*>(hg + o_size) + M);
    ch.bytes = g.child_bytes;
    s.cur = 1 - s.cur;
    s.first = 0;
    s.count = M;
    s.items_for = nullptr;  // the host work-list cache does not describe these items
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, s.ev[2], s.ev[3]));
    const double splice_s = ms * 1e-3;
    if (g.flags & 16u) {  // work list beyond its buffers: the host path evaluates (and grows them)
        TRY(ltgp_evaluate_launch(e));
        TRY(ltgp_evaluate_collect(e, out, nullptr));
        e->stats.splice_seconds = splice_s;
        return 0;
    }
    const uint32_t C = g.chunk;
    const uint32_t rc = (uint32_t)std::lround(std::sqrt((double)C));
    s.cur_chunk = C;
    s.cur_max_frames = std::max<uint32_t>(kMaxFrames, (6 * rc + 63) & ~63u);
    s.cur_max_steps = std::min<uint32_t>(C, std::max<uint32_t>(kMaxSteps, 16 * rc));
    s.last_items = g.n_items;
    s.last_chunks = g.n_chunks;
    s.last_ctrees = g.n_trees;
    s.max_tree_chunks = g.max_chunks;
    s.eargs = a;  // for the overflow re-runs: the counts on the host
    s.eargs.n_items = g.n_items;
    s.eargs.n_items_dev = nullptr;
    s.cargs = ca;
    s.cargs.n_trees = g.n_trees;
    s.cargs.n_chunks = g.n_chunks;
    s.cargs.counts_dev = nullptr;
    s.last_outs = false;
    s.last_reruns = 0;
    s.rerun_ksecs = s.rerun_csecs = 0.0;
    const uint32_t* hc = s.h_counters.as<uint32_t>();
    const bool reruns = hc[2] != 0;
    if (reruns) {  // rerun_overflowed reads the work list from s.h_items
        TRY(s.h_items.ensure(sizeof(Item) * std::max<uint32_t>(g.n_items, 1)));
        CK(cudaMemcpyAsync(s.h_items.p, s.items.p, sizeof(Item) * g.n_items, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
    }
    TRY(finish_eval(e, s));
    if (out) {
        if (reruns) {
            CK(cudaMemcpyAsync(out, s.rec.p, sizeof(ltgp_record) * M, cudaMemcpyDeviceToHost, s.st));
            CK(cudaStreamSynchronize(s.st));
        } else {
            std::memcpy(out, hg + o_rec, sizeof(ltgp_record) * M);
        }
    }
    CK(cudaEventElapsedTime(&ms, s.ev[0], s.ev[4]));
    const double k = ms * 1e-3 + s.rerun_ksecs;
    CK(cudaEventElapsedTime(&ms, s.ev[4], s.ev[1]));
    const double cmb = ms * 1e-3 + s.rerun_csecs;
    CK(cudaEventElapsedTime(&ms, s.kev[0], s.kev[1]));
    e->stats.keval_seconds = ms * 1e-3;
    e->stats.eval_seconds = k + cmb;
    e->stats.eval_kernel_seconds = k;
    e->stats.combine_seconds = cmb;
    e->stats.splice_seconds = splice_s;
    e->stats.nodes_evaluated += g.nodes;
    e->stats.last_chunks = g.n_chunks;
    e->stats.last_spine_steps = s.last_steps;
    e->stats.last_exits = hc[4];
    e->stats.last_window_adjusts = hc[5];
    e->stats.last_fallback_items = s.last_reruns;
    e->stats.kernel_launches = 10;
    s.kev_valid = true;
    tr.mark("finish");
    return 0;
}

// The host-orchestrated generation (multi-shard and streaming engines, and
// the device path's fallback): directory, extents, limit checks and layout
// on the host, kernels per phase.
static int execute_generation_host(ltgp_engine* e, const ltgp_plan* plans, uint32_t M, ltgp_record* out,
                                   int* size_limit_hit) {
    Trace tr("ltgp.execute_generation");
    std::vector<DirEntry> dir;
    build_directory(e, dir);
    for (uint32_t c = 0; c < M; ++c)
        if (plans[c].mum_pt >= dir[plans[c].mum_index].size || plans[c].dad_pt >= dir[plans[c].dad_index].size) {
            set_err("plan %u: crossover point out of range", c);  // std::out_of_range
            return -1;
        }
    // 1. extents for children in equal-count ranges
    const int G = (int)e->shards.size();
    std::vector<uint32_t> qfirst(G), qcount(G);
    for (int g = 0; g < G; ++g) {
        qfirst[g] = (uint32_t)((uint64_t)M * g / G);
        qcount[g] = (uint32_t)((uint64_t)M * (g + 1) / G) - qfirst[g];
    }
    std::vector<Extent> ext(M);
    std::vector<uint64_t> csize(M);
    for (int g = 0; g < G; ++g) {
        Shard& s = e->shards[g];
        TRY(upload_directory(e, s, dir));
        if (!qcount[g]) continue;
        TRY(s.plans.ensure(sizeof(PlanDev) * M, s.dev));
        TRY(s.ext.ensure(sizeof(Extent) * M, s.dev));
        TRY(s.csize.ensure(sizeof(uint64_t) * M, s.dev));
        CK(cudaMemcpyAsync(s.plans.p, plans + qfirst[g], sizeof(PlanDev) * qcount[g], cudaMemcpyHostToDevice, s.st));
        CK(cudaMemsetAsync(s.counters.p, 0, 64, s.st));
        CK(cudaEventRecord(s.ev[2], s.st));
        const uint32_t warps = 2 * qcount[g];
        NvtxRange nr_ext("ltgp.extents");
        k_extent<<<(warps + 3) / 4, 128, 0, s.st>>>(s.plans.as<PlanDev>(), qcount[g], s.dir.as<DirEntry>(),
                                                  s.ext.as<Extent>(), nullptr, s.counters.as<uint32_t>() + 3);
        CK(cudaGetLastError());
        k_child_size<<<(qcount[g] + 127) / 128, 128, 0, s.st>>>(s.plans.as<PlanDev>(), qcount[g],
                                                              s.dir.as<DirEntry>(), s.ext.as<Extent>(),
                                                              s.csize.as<uint64_t>());
        CK(cudaGetLastError());
        // one shard splices exactly the children whose extents it computed:
        // the extents and plans stay on the device (no round trip)
        if (G > 1)
            CK(cudaMemcpyAsync(ext.data() + qfirst[g], s.ext.p, sizeof(Extent) * qcount[g], cudaMemcpyDeviceToHost,
                               s.st));
        CK(cudaMemcpyAsync(csize.data() + qfirst[g], s.csize.p, sizeof(uint64_t) * qcount[g], cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(s.h_counters.p, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
    }
    for (int g = 0; g < G; ++g) {
        Shard& s = e->shards[g];
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.st));
        if (qcount[g] && s.h_counters.as<uint32_t>()[3]) { set_err("malformed parent genome in extent scan"); return -1; }
    }
    tr.mark("extents");
    // 2. MemoryBudgetExceeded (evolve.hpp:89-93): the
    // generation's planned genome bytes (parents plus every child, sizes from
    // the crossover algebra) over the budget, checked before materializing
    if (e->memory_budget) {
        uint64_t bytes = 0;
        for (uint32_t c = 0; c < M; ++c) bytes += dir[c].size + csize[c];
        if (bytes > e->memory_budget) { *size_limit_hit = 2; return 0; }
    }
    // 3. SizeLimitHit (genome.hpp:71-84): child >= node_limit
    for (uint32_t c = 0; c < M; ++c)
        if (csize[c] >= e->cfg.node_limit) { *size_limit_hit = 1; return 0; }
    // a child below node_limit (node_limit > 2^32) but beyond the engine's
    // u32 sizes is an engine capacity error, not the run's SizeLimitHit
    for (uint32_t c = 0; c < M; ++c)
        if (csize[c] > 0xffffffffull) {
            set_err("child %u has %llu nodes: beyond the engine's 2^32-1-node tree capacity (node_limit %llu)", c,
                    (unsigned long long)csize[c], (unsigned long long)e->cfg.node_limit);
            return -1;
        }
    if (e->streaming) {
        TRY(splice_streaming(e, plans, M, csize));
        tr.mark("splice (streaming)");
        TRY(ltgp_evaluate_launch(e));
        TRY(ltgp_evaluate_collect(e, out, nullptr));
        Shard& s = e->shards[0];
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, s.ev[2], s.ev[3]));
        e->stats.splice_seconds = ms * 1e-3;
        return 0;
    }
    // 4. children partitioned by bytes; splice into the other buffer
    // (parents stay readable until every shard has spliced).
    std::vector<uint32_t> old_cur(G);
    for (int g = 0; g < G; ++g) old_cur[g] = e->shards[g].cur;
    partition(e, M, csize.data());
    float splice_ms = 0.0f;
    for (int g = 0; g < G; ++g) {
        Shard& s = e->shards[g];
        TreeSet& ts = s.set[1 - s.cur];
        if (s.count == 0) { ts.count = 0; continue; }
        std::vector<uint64_t> coff(s.count);
        TRY(set_layout(s, ts, s.count, csize.data() + s.first, coff.data()));
        CK(cudaSetDevice(s.dev));
        TRY(s.coff.ensure(sizeof(uint64_t) * s.count, s.dev));
        TRY(s.h_coff.ensure(sizeof(uint64_t) * s.count * 2 + sizeof(Extent) * s.count + sizeof(PlanDev) * s.count));
        uint8_t* hb = s.h_coff.as<uint8_t>();
        std::memcpy(hb, coff.data(), sizeof(uint64_t) * s.count);
        std::memcpy(hb + 8 * s.count, csize.data() + s.first, sizeof(uint64_t) * s.count);
        if (G > 1) {
            std::memcpy(hb + 16 * s.count, ext.data() + s.first, sizeof(Extent) * s.count);
            std::memcpy(hb + 32 * s.count, plans + s.first, sizeof(PlanDev) * s.count);
        }
        CK(cudaMemcpyAsync(s.coff.p, hb, 8 * s.count, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(s.csize.p, hb + 8 * s.count, 8 * s.count, cudaMemcpyHostToDevice, s.st));
        if (G > 1) {
            CK(cudaMemcpyAsync(s.ext.p, hb + 16 * s.count, sizeof(Extent) * s.count, cudaMemcpyHostToDevice, s.st));
            CK(cudaMemcpyAsync(s.plans.p, hb + 32 * s.count, sizeof(PlanDev) * s.count, cudaMemcpyHostToDevice,
                               s.st));
        }
        CK(cudaEventRecord(s.ev[2], s.st));
        NvtxRange nr_splice("ltgp.splice");
        k_splice<<<std::min<uint32_t>(s.count, (uint32_t)s.sms * 8), 256, 0, s.st>>>(
            s.plans.as<PlanDev>(), s.count, s.dir.as<DirEntry>(), s.ext.as<Extent>(), s.coff.as<uint64_t>(),
            s.csize.as<uint64_t>(), ts.arena.as<uint8_t>(), nullptr);
        CK(cudaGetLastError());
        CK(cudaEventRecord(s.ev[3], s.st));
        CK(cudaMemcpyAsync(ts.off.p, ts.h_off.data(), sizeof(uint64_t) * ts.count, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(ts.size.p, ts.h_size.data(), sizeof(uint32_t) * ts.count, cudaMemcpyHostToDevice, s.st));
    }
    // no sync here: each shard evaluates its children on the stream that
    // spliced them, and a parent arena is overwritten only by the next
    // generation's splice, after this generation's collect has synchronised
    // every shard (the splice reads parents on other shards through P2P)
    for (int g = 0; g < G; ++g) e->shards[g].cur = 1 - old_cur[g];
    tr.mark("splice");
    // 5. evaluate the children
    TRY(ltgp_evaluate_launch(e));
    tr.mark("eval launch");
    TRY(ltgp_evaluate_collect(e, out, nullptr));
    for (Shard& s : e->shards)
        if (s.count) {
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, s.ev[2], s.ev[3]));
            splice_ms = std::max(splice_ms, ms);
        }
    e->stats.splice_seconds = splice_ms * 1e-3;
    tr.mark("eval collect");
    return 0;
}

int ltgp_execute_generation_launch(ltgp_engine* e, const ltgp_plan* plans, uint32_t M) {
    if (!e || !plans) { set_err("null argument"); return -1; }
    if (e->pend.active) { set_err("the launched generation is not finished (ltgp_execute_generation_finish)"); return -1; }
    if (M != e->M) { set_err("plan count %u != population size %u", M, e->M); return -1; }
    if (!e->have_suite) { set_err("ltgp_set_suite not called"); return -1; }
    for (uint32_t c = 0; c < M; ++c)
        if (plans[c].mum_index >= M || plans[c].dad_index >= M) {
            set_err("plan %u references slot outside the population", c);
            return -1;
        }
    auto& p = e->pend;
    p.M = M;
    p.device = e->shards.size() == 1 && !e->streaming && device_generation_enabled();
    if (p.device) {
        const TreeSet& par = e->shards[0].set[e->shards[0].cur];
        for (uint32_t c = 0; c < M; ++c)
            if (plans[c].mum_pt >= par.h_size[plans[c].mum_index] || plans[c].dad_pt >= par.h_size[plans[c].dad_index]) {
                set_err("plan %u: crossover point out of range", c);  // std::out_of_range
                return -1;
            }
        TRY(gen_device_launch(e, plans, M));
    } else {
        p.plans.assign(plans, plans + M);
    }
    p.active = true;
    return 0;
}

int ltgp_execute_generation_finish(ltgp_engine* e, ltgp_record* out, int* size_limit_hit) {
    if (!e || !size_limit_hit) { set_err("null argument"); return -1; }
    auto& p = e->pend;
    if (!p.active) { set_err("no launched generation (ltgp_execute_generation_launch)"); return -1; }
    p.active = false;
    *size_limit_hit = 0;
    if (p.device) {
        const int r = gen_device_finish(e, p.M, out, size_limit_hit);
        if (r <= 0) return r;
        // the children's arena was grown: the host path runs this generation
        p.plans.resize(p.M);
        std::memcpy(p.plans.data(), e->shards[0].h_gen.p, sizeof(ltgp_plan) * p.M);
    }
    return execute_generation_host(e, p.plans.data(), p.M, out, size_limit_hit);
}

int ltgp_execute_generation(ltgp_engine* e, const ltgp_plan* plans, uint32_t M, ltgp_record* out,
                            int* size_limit_hit) {
    if (!e || !plans || !size_limit_hit) { set_err("null argument"); return -1; }
    TRY(ltgp_execute_generation_launch(e, plans, M));
    return ltgp_execute_generation_finish(e, out, size_limit_hit);
}

int ltgp_subtree_extents(ltgp_engine* e, uint32_t count, const uint32_t* slots, const uint32_t* points,
                         uint64_t* out) {
    if (!e || (count && (!slots || !points || !out))) { set_err("null argument"); return -1; }
    std::vector<DirEntry> dir;
    build_directory(e, dir);
    std::vector<PlanDev> q(count);
    for (uint32_t i = 0; i < count; ++i) {
        if (slots[i] >= e->M) { set_err("slot out of range"); return -1; }
        if (points[i] >= dir[slots[i]].size) { set_err("point out of range"); return -1; }
        q[i] = PlanDev{slots[i], slots[i], points[i], points[i]};
    }
    Shard& s = e->shards[0];
    TRY(upload_directory(e, s, dir));
    TRY(s.plans.ensure(sizeof(PlanDev) * std::max<uint32_t>(count, 1), s.dev));
    TRY(s.ext.ensure(sizeof(Extent) * std::max<uint32_t>(count, 1), s.dev));
    CK(cudaMemcpyAsync(s.plans.p, q.data(), sizeof(PlanDev) * count, cudaMemcpyHostToDevice, s.st));
    CK(cudaMemsetAsync(s.counters.p, 0, 64, s.st));
    if (count) {
        k_extent<<<(2 * count + 3) / 4, 128, 0, s.st>>>(s.plans.as<PlanDev>(), count, s.dir.as<DirEntry>(),
                                                        s.ext.as<Extent>(), nullptr, s.counters.as<uint32_t>() + 3);
        CK(cudaGetLastError());
    }
    std::vector<Extent> ext(count);
    CK(cudaMemcpyAsync(ext.data(), s.ext.p, sizeof(Extent) * count, cudaMemcpyDeviceToHost, s.st));
    CK(cudaMemcpyAsync(s.h_counters.p, s.counters.p, 64, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    if (s.h_counters.as<uint32_t>()[3]) { set_err("malformed genome in extent scan"); return -1; }
    for (uint32_t i = 0; i < count; ++i) { out[2 * i] = ext[i].ms; out[2 * i + 1] = ext[i].me; }
    return 0;
}

}  // extern "C"
