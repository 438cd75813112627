// Host-side probe for the packed PCIe transfer (csrc/ltgp_pack.*): packs a
// config-3-like byte stream with 1..T threads and compares with plain memcpy
// bandwidth on the same host. Build + run: bash tools/pack_probe.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "../paper_1902_09215_b200/csrc/ltgp_pack.h"

using clk = std::chrono::steady_clock;
static double secs(clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); }

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 855759280ull;
    const uint64_t slice = 36ull << 20;
    std::vector<uint8_t> src(n), out(n);
    std::mt19937_64 r(1);
    for (uint64_t i = 0; i < n; i += 8) {
        uint64_t w = r();
        for (int k = 0; k < 8 && i + k < n; ++k) {
            const uint32_t u = (w >> (8 * k)) & 0xff;  // ~50% functions, 25% X, 25% constants
            src[i + k] = u < 128 ? (uint8_t)(u & 3) : u < 192 ? 4 : (uint8_t)(5 + (u * 7) % 250);
        }
    }
    std::printf("host threads %u, avx512 %d, %.0f MB\n", std::thread::hardware_concurrency(), (int)ltgp_pack::have_avx512(), n / 1e6);
    uint8_t* dst_raw = static_cast<uint8_t*>(std::aligned_alloc(4096, (ltgp_pack::Layout(slice).max_bytes() + 64) * ((n + slice - 1) / slice) + 4096));
    struct { uint8_t* p; uint8_t* data() { return p; } } dst{dst_raw};
    for (int T : {1, 4, 8, 12, 15, 16}) {
        // memcpy bandwidth with T threads
        auto t0 = clk::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] { std::memcpy(out.data() + n * t / T, src.data() + n * t / T, n * (t + 1) / T - n * t / T); });
        for (auto& x : th) x.join();
        const double mc = secs(t0);
        ltgp_pack::Pool* P = ltgp_pack::pool_create(T);
        double best = 1e9;
        uint64_t tot = 0;
        for (int rep = 0; rep < 3; ++rep) {
            t0 = clk::now();
            tot = 0;
            uint64_t o = 0;
            for (uint64_t s = 0; s < n; s += slice) {
                const uint64_t len = std::min(slice, n - s);
                const uint64_t b = ltgp_pack::pack(P, src.data() + s, len, dst.data() + o);
                o += (b + 63) & ~63ull;
                tot += b;
            }
            best = std::min(best, secs(t0));
        }
        ltgp_pack::pool_destroy(P);
        std::printf("T=%2d memcpy %6.1f GB/s | pack %6.1f GB/s in (%.2f ms), %.3f B/node out\n", T, n / mc / 1e9, n / best / 1e9,
                    best * 1e3, (double)tot / n);
    }
    // round trip of the last packing
    uint64_t o = 0;
    for (uint64_t s = 0; s < n; s += slice) {
        const uint64_t len = std::min(slice, n - s);
        ltgp_pack::unpack_scalar(dst.data() + o, len, out.data() + s);
        const ltgp_pack::Layout L(len);
        const uint32_t* base = reinterpret_cast<const uint32_t*>(dst.data() + o + L.base_off);
        (void)base;
        // size of this slice's packing: recompute from the literal count
        uint64_t nl = 0;
        for (uint64_t i = 0; i < len; ++i) nl += ltgp_pack::code_of(src[s + i]) == 5;
        o += (L.bytes(nl) + 63) & ~63ull;
    }
    std::printf("round trip %s\n", std::memcmp(src.data(), out.data(), n) == 0 ? "identical" : "MISMATCH");
    return 0;
}
