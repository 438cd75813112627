// ltgp_pack.cpp — multi-threaded host packing of opcode slices (format in
// ltgp_pack.h). Host code only (g++), linked into libltgp_cuda.so.
//
// Workers claim chunks of 16 blocks of 256 packets: the three code planes go
// to the destination with non-temporal stores (a block's plane words are
// 512 B each), literals to the chunk's scratch region (still in the thread's
// cache when it copies them). At a barrier the last worker turns the block
// literal counts into bases; then the chunks' literals are streamed to their
// final place. The destination is
// pinned memory the copy engine reads next, so nothing is gained by leaving
// it in the CPU caches; non-temporal stores also skip the read-for-ownership
// traffic. The AVX-512 path (VBMI2 byte compress) encodes 64 bytes per step;
// other hosts use the scalar loop of ltgp_pack.h. Either way the bytes are
// identical.
#include "ltgp_pack.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

namespace ltgp_pack {

namespace {

__attribute__((target("avx512f,avx512bw,avx512vbmi2,popcnt"))) uint64_t
encode_avx512(const uint8_t* src, uint64_t len, const Layout& L, uint8_t* dst, uint64_t b0, uint64_t b1,
              uint8_t* lit, uint32_t* blk_count) {
    const __m512i c1 = _mm512_set1_epi8(1), c2 = _mm512_set1_epi8(2), c4 = _mm512_set1_epi8(4),
                  c5 = _mm512_set1_epi8(5), cff = _mm512_set1_epi8((char)0xff);
    alignas(64) uint64_t w[3][64];
    uint64_t n = 0;
    for (uint64_t b = b0; b < b1; ++b) {
        uint64_t nb = 0;
        const uint64_t i0 = b * kBlockPackets * 16;
        for (int j = 0; j < 64; ++j) {  // 4 packets (64 bytes) a step
            const uint64_t i = i0 + 64 * (uint64_t)j;
            __m512i v;
            if (i + 64 <= len) {
                v = _mm512_loadu_si512(src + i);
            } else {
                const __mmask64 m = i >= len ? 0 : (~0ull >> (64 - (len - i)));
                v = _mm512_mask_loadu_epi8(cff, m, src + i);
            }
            const __mmask64 func = _mm512_cmplt_epu8_mask(v, c4);
            const __mmask64 ff = _mm512_cmpeq_epi8_mask(v, cff);
            const __mmask64 lit_m = ~(_mm512_cmplt_epu8_mask(v, c5) | ff);
            // bits 16k..16k+15: the plane word of packet 4j+k (little endian)
            w[0][j] = (_mm512_test_epi8_mask(v, c1) & func) | lit_m;
            w[1][j] = (_mm512_test_epi8_mask(v, c2) & func) | ff;
            w[2][j] = ~func;
            _mm512_storeu_si512(lit + n + nb, _mm512_maskz_compress_epi8(lit_m, v));  // 64 B of slack
            nb += (uint64_t)_mm_popcnt_u64(lit_m);
        }
        for (int q = 0; q < 3; ++q) {
            uint8_t* o = dst + q * L.plane_bytes + b * kBlockPackets * 2;  // 512 B (64-B aligned in the engine)
            const bool aligned = ((uintptr_t)o & 63) == 0;
            for (int k = 0; k < 8; ++k) {
                const __m512i x = _mm512_load_si512(reinterpret_cast<const __m512i*>(&w[q][8 * k]));
                if (aligned) _mm512_stream_si512(reinterpret_cast<__m512i*>(o + 64 * k), x);
                else _mm512_storeu_si512(o + 64 * k, x);
            }
        }
        blk_count[b - b0] = (uint32_t)nb;
        n += nb;
    }
    return n;
}

__attribute__((target("avx512f"))) void copy_nt(uint8_t* d, const uint8_t* s, size_t n) {
    size_t h = (64 - ((uintptr_t)d & 63)) & 63;
    if (h > n) h = n;
    memcpy(d, s, h);
    d += h, s += h, n -= h;
    for (; n >= 64; n -= 64, d += 64, s += 64)
        _mm512_stream_si512(reinterpret_cast<__m512i*>(d), _mm512_loadu_si512(s));
    memcpy(d, s, n);
}

// spin-wait step: pause, then yield (an oversubscribed host must not starve
// the thread being waited for)
inline void relax(int i) {
    if (i < 4096) _mm_pause();
    else std::this_thread::yield();
}

bool cpu_avx512() {
    if (std::getenv("LTGP_PACK_SCALAR")) return false;  // tests: the scalar encoder
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
           __builtin_cpu_supports("avx512vbmi2");
}

}  // namespace

bool have_avx512() {
    static const bool v = cpu_avx512();
    return v;
}

// n worker threads packing one slice at a time (the caller starts, then
// waits, or helps). Work is claimed dynamically in chunks of kChunkBlocks
// blocks, so a thread the OS preempts (the host is shared with the caller,
// a driver thread, a clock sampler) delays one chunk, not a fixed share of
// the slice. A streamed evaluation packs a slice every ~0.3 ms, so idle
// workers spin for a while (no futex wake-up on the critical path) before
// sleeping.
constexpr uint64_t kChunkBlocks = 16;  // 64 KB of input
struct Pool {
    int n;
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> gen{0};
    std::atomic<int> pending{0}, arrived{0};
    std::atomic<uint64_t> phase2{0};
    std::atomic<uint64_t> next1{0}, next2{0};
    std::atomic<int> sleepers{0};
    std::atomic<bool> stop{false};
    std::vector<uint8_t> scratch;   // literals of chunk c at c * kChunkBlocks * 4096
    // the job
    const uint8_t* src = nullptr;
    uint64_t len = 0;
    uint8_t* dst = nullptr;
    Layout L{0};
    uint64_t nchunks = 0;
    int parts = 0;      // threads taking part: the workers, plus the caller when it helps
    std::vector<uint32_t> cnt;     // literals per block
    std::vector<uint64_t> cl, co;  // literals per chunk, and their offsets
    uint64_t total = 0;

    explicit Pool(int nthreads) : n(std::max(1, nthreads)) {
        for (int t = 0; t < n; ++t) th.emplace_back([this, t] { worker(t); });
    }
    ~Pool() {
        stop = true;
        {
            std::lock_guard<std::mutex> g(mu);
        }
        cv.notify_all();
        for (auto& x : th) x.join();
    }
    void work(uint64_t my_gen) {
        const bool simd = have_avx512();
        for (uint64_t c; (c = next1.fetch_add(1)) < nchunks;) {
            const uint64_t b0 = c * kChunkBlocks, b1 = std::min(L.nblk, b0 + kChunkBlocks);
            uint8_t* lit = scratch.data() + c * kChunkBlocks * kBlockPackets * 16;
            cl[c] = simd ? encode_avx512(src, len, L, dst, b0, b1, lit, cnt.data() + b0)
                         : encode_scalar(src, len, L, dst, b0, b1, lit, cnt.data() + b0);
        }
        if (arrived.fetch_add(1) == parts - 1) {  // the last one: block literal bases
            uint32_t* base = reinterpret_cast<uint32_t*>(dst + L.base_off);
            uint64_t acc = 0;
            for (uint64_t c = 0; c < nchunks; ++c) {
                co[c] = acc;
                const uint64_t b1 = std::min(L.nblk, (c + 1) * kChunkBlocks);
                for (uint64_t b = c * kChunkBlocks; b < b1; ++b) {
                    base[b] = (uint32_t)acc;
                    acc += cnt[b];
                }
            }
            total = L.bytes(acc);
            phase2.store(my_gen);
        } else {
            for (int i = 0; phase2.load() != my_gen; ++i) relax(i);
        }
        for (uint64_t c; (c = next2.fetch_add(1)) < nchunks;)
            if (cl[c]) copy_nt(dst + L.lit_off + co[c], scratch.data() + c * kChunkBlocks * kBlockPackets * 16, cl[c]);
        _mm_sfence();
    }
    void worker(int) {
        uint64_t seen = 0;
        for (;;) {
            for (int i = 0; i < 100000 && gen.load() == seen && !stop; ++i) _mm_pause();
            if (gen.load() == seen && !stop) {
                std::unique_lock<std::mutex> g(mu);
                ++sleepers;
                cv.wait(g, [&] { return stop.load() || gen.load() != seen; });
                --sleepers;
            }
            if (stop) return;
            seen = gen.load();
            work(seen);
            --pending;
        }
    }
    void start(const uint8_t* s, uint64_t l, uint8_t* d, bool help) {
        src = s, len = l, dst = d;
        L = Layout(l);
        nchunks = (L.nblk + kChunkBlocks - 1) / kChunkBlocks;
        parts = n + (help ? 1 : 0);
        const uint64_t sb = nchunks * kChunkBlocks * kBlockPackets * 16 + 64;
        if (scratch.size() < sb) scratch.resize(sb);
        cnt.assign(L.nblk, 0);
        cl.assign(nchunks, 0);
        co.assign(nchunks, 0);
        next1 = 0;
        next2 = 0;
        arrived = 0;
        pending = n;
        ++gen;
        if (sleepers.load()) {
            std::lock_guard<std::mutex> g(mu);
            cv.notify_all();
        }
    }
    uint64_t wait() {
        if (parts > n) work(gen.load());  // the caller takes chunks too
        for (int i = 0; pending.load(); ++i) relax(i);
        return total;
    }
};

Pool* pool_create(int nthreads) { return new Pool(nthreads); }
void pool_destroy(Pool* p) { delete p; }
int pool_threads(const Pool* p) { return p->n; }
void pack_start(Pool* P, const uint8_t* src, uint64_t len, uint8_t* dst, bool caller_helps) {
    P->start(src, len, dst, caller_helps);
}
uint64_t pack_wait(Pool* P) { return P->wait(); }
uint64_t pack(Pool* P, const uint8_t* src, uint64_t len, uint8_t* dst) {
    P->start(src, len, dst, true);
    return P->wait();
}

}  // namespace ltgp_pack
