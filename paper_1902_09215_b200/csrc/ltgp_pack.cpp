// ltgp_pack.cpp — multi-threaded host packing of opcode slices (format in
// ltgp_pack.h). Host code only (g++), linked into libltgp_cuda.so.
//
// Worker t packs a run of whole 256-packet blocks: the three code planes go
// to the destination with non-temporal stores (a block's plane words are
// 512 B each), literals to a per-thread scratch that stays in its cache. At a
// barrier the last worker turns the block literal counts into bases; then
// every worker streams its literals to their final place. The destination is
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

// n worker threads packing one slice at a time (the caller only starts and
// waits). A streamed evaluation packs a slice every ~0.5 ms, so idle workers
// spin for a while (no futex wake-up on the critical path) before sleeping.
struct Pool {
    int n;
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> gen{0};
    std::atomic<int> pending{0}, arrived{0};
    std::atomic<uint64_t> phase2{0};
    std::atomic<int> sleepers{0};
    std::atomic<bool> stop{false};
    std::vector<std::vector<uint8_t>> scratch;
    // the job
    const uint8_t* src = nullptr;
    uint64_t len = 0;
    uint8_t* dst = nullptr;
    Layout L{0};
    int T = 0;
    int parts = 0;      // workers + the caller when it helps (pack_wait(help))
    std::vector<uint64_t> b0, nlit, tl;
    std::vector<uint32_t> cnt;
    uint64_t total = 0;

    explicit Pool(int nthreads) : n(std::max(1, nthreads)), scratch(n + 1) {
        b0.resize(n + 2);
        nlit.resize(n + 1);
        tl.resize(n + 1);
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
    void work(int t, uint64_t my_gen) {
        if (t < T) {
            std::vector<uint8_t>& s = scratch[t];
            const uint64_t bytes = (b0[t + 1] - b0[t]) * kBlockPackets * 16 + 64;
            if (s.size() < bytes) s.resize(bytes);
            nlit[t] = have_avx512() ? encode_avx512(src, len, L, dst, b0[t], b0[t + 1], s.data(), cnt.data() + b0[t])
                                    : encode_scalar(src, len, L, dst, b0[t], b0[t + 1], s.data(), cnt.data() + b0[t]);
        }
        if (arrived.fetch_add(1) == parts - 1) {  // the last one: block literal bases
            uint32_t* base = reinterpret_cast<uint32_t*>(dst + L.base_off);
            uint64_t acc = 0;
            for (int u = 0; u < T; ++u) {
                tl[u] = acc;
                for (uint64_t b = b0[u]; b < b0[u + 1]; ++b) {
                    base[b] = (uint32_t)acc;
                    acc += cnt[b];
                }
            }
            total = L.bytes(acc);
            phase2.store(my_gen);
        } else {
            for (int i = 0; phase2.load() != my_gen; ++i) relax(i);
        }
        if (t < T && nlit[t]) copy_nt(dst + L.lit_off + tl[t], scratch[t].data(), nlit[t]);
        _mm_sfence();
    }
    void worker(int t) {
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
            work(t, seen);
            --pending;
        }
    }
    void start(const uint8_t* s, uint64_t l, uint8_t* d, bool help) {
        src = s, len = l, dst = d;
        L = Layout(l);
        parts = n + (help ? 1 : 0);
        T = (int)std::min<uint64_t>((uint64_t)parts, std::max<uint64_t>(1, L.nblk));
        for (int t = 0; t <= T; ++t) b0[t] = L.nblk * t / T;
        for (int t = 0; t < parts; ++t) nlit[t] = 0;
        cnt.assign(L.nblk, 0);
        arrived = 0;
        pending = n;
        ++gen;
        if (sleepers.load()) {
            std::lock_guard<std::mutex> g(mu);
            cv.notify_all();
        }
    }
    uint64_t wait() {
        if (parts > n) work(n, gen.load());  // the caller's part
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
