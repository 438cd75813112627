// ref_kat.cpp — known-answer generator built AGAINST THE REFERENCE'S OWN
// inline code (test infrastructure only). The reference is a header-only
// skeleton: only rng.hpp:9-51, eval.hpp:54-63 (protected_div,
// apply_op), eval.hpp:89-98 (fitness_better/tied) and the struct layouts are
// executable. This program links nothing but those headers, which it reads
// where they lie under /root/reference (see oracle/Makefile target `ref`),
// and prints JSON known answers that tests/golden/make_golden.py freezes into
// tests/golden/ref_inline_kats.json.
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "ltgp/eval.hpp"
#include "ltgp/evolve.hpp"
#include "ltgp/rng.hpp"

static uint32_t bits(float f) { uint32_t b; std::memcpy(&b, &f, 4); return b; }
static float fbits(uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; }

int main() {
    std::printf("{\n");
    // splitmix64
    std::printf("\"splitmix64\": [");
    const uint64_t sm[] = {0, 1, 2, 3, 7, 42, 12345, 0x53554954ull, 0x8000000000000000ull, ~0ull};
    for (size_t i = 0; i < sizeof sm / sizeof sm[0]; ++i)
        std::printf("%s[\"%llu\", \"%llu\"]", i ? ", " : "", (unsigned long long)sm[i],
                    (unsigned long long)ltgp::splitmix64(sm[i]));
    std::printf("],\n");
    // below(n) sequences
    const uint64_t seeds[] = {1, 2, 3, 42, 12345};
    const uint64_t ns[] = {1, 2, 3, 4, 7, 250, 251, 255, 2001, 4000, 1000000, 4294967297ull,
                           9223372036854775809ull};
    std::printf("\"below\": [");
    bool first = true;
    for (uint64_t s : seeds)
        for (uint64_t n : ns) {
            ltgp::Rng r(s);
            std::printf("%s{\"seed\": %llu, \"n\": \"%llu\", \"v\": [", first ? "" : ", ",
                        (unsigned long long)s, (unsigned long long)n);
            first = false;
            for (int k = 0; k < 16; ++k) std::printf("%s\"%llu\"", k ? ", " : "", (unsigned long long)r.below(n));
            std::printf("], \"draws\": %llu}", (unsigned long long)r.draw_count());
        }
    std::printf("],\n");
    // uniform_pm1 sequences (raw bits)
    std::printf("\"uniform_pm1\": [");
    first = true;
    for (uint64_t s : seeds) {
        ltgp::Rng r(s);
        std::printf("%s{\"seed\": %llu, \"bits\": [", first ? "" : ", ", (unsigned long long)s);
        first = false;
        for (int k = 0; k < 48; ++k) std::printf("%s%u", k ? ", " : "", bits(r.uniform_pm1()));
        std::printf("]}");
    }
    std::printf("],\n");
    // interleaved stream: below(255) x5 then uniform x3
    std::printf("\"interleaved\": [");
    first = true;
    for (uint64_t s : seeds) {
        ltgp::Rng r(s);
        std::printf("%s{\"seed\": %llu, \"below255\": [", first ? "" : ", ", (unsigned long long)s);
        first = false;
        for (int k = 0; k < 5; ++k) std::printf("%s%llu", k ? ", " : "", (unsigned long long)r.below(255));
        std::printf("], \"pm1_bits\": [");
        for (int k = 0; k < 3; ++k) std::printf("%s%u", k ? ", " : "", bits(r.uniform_pm1()));
        std::printf("], \"draws\": %llu}", (unsigned long long)r.draw_count());
    }
    std::printf("],\n");
    // protected_div / apply_op over special values (raw bits)
    const uint32_t vals[] = {0x00000000u, 0x80000000u, 0x3f800000u, 0xbf800000u, 0x40400000u, 0xc0600000u,
                             0x3dcccccdu, 0x0000b27au, 0x8000b27au, 0x7f7fffffu, 0x00800000u, 0x7f800000u,
                             0xff800000u, 0x7fc00000u, 0x7e967699u, 0x0d0ee41cu, 0x3f400000u, 0xbe99999au,
                             0x00000001u, 0x3eaaaaabu};
    const size_t nv = sizeof vals / sizeof vals[0];
    std::printf("\"values\": [");
    for (size_t i = 0; i < nv; ++i) std::printf("%s%u", i ? ", " : "", vals[i]);
    std::printf("],\n\"apply_op\": [");
    for (int op = 0; op < 4; ++op) {
        std::printf("%s[", op ? ", " : "");
        for (size_t i = 0; i < nv; ++i)
            for (size_t j = 0; j < nv; ++j)
                std::printf("%s%u", (i || j) ? ", " : "",
                            bits(ltgp::apply_op((uint8_t)op, fbits(vals[i]), fbits(vals[j]))));
        std::printf("]");
    }
    std::printf("],\n\"protected_div\": [");
    for (size_t i = 0; i < nv; ++i)
        for (size_t j = 0; j < nv; ++j)
            std::printf("%s%u", (i || j) ? ", " : "", bits(ltgp::protected_div(fbits(vals[i]), fbits(vals[j]))));
    std::printf("],\n\"fitness_better\": [");
    for (size_t i = 0; i < nv; ++i)
        for (size_t j = 0; j < nv; ++j)
            std::printf("%s%d", (i || j) ? ", " : "", (int)ltgp::fitness_better(fbits(vals[i]), fbits(vals[j])));
    std::printf("],\n\"fitness_tied\": [");
    for (size_t i = 0; i < nv; ++i)
        for (size_t j = 0; j < nv; ++j)
            std::printf("%s%d", (i || j) ? ", " : "", (int)ltgp::fitness_tied(fbits(vals[i]), fbits(vals[j])));
    std::printf("],\n");
    // layouts the C ABI mirrors
    std::printf("\"layout\": {\"CrossoverPlan\": [%zu, %zu, %zu, %zu, %zu], \"kLaneWidth\": %zu, "
                "\"kConstantCount\": %d, \"kPrimitiveCount\": %d}\n",
                sizeof(ltgp::CrossoverPlan), offsetof(ltgp::CrossoverPlan, mum_index),
                offsetof(ltgp::CrossoverPlan, dad_index), offsetof(ltgp::CrossoverPlan, mum_pt),
                offsetof(ltgp::CrossoverPlan, dad_pt), ltgp::kLaneWidth, ltgp::kConstantCount,
                ltgp::kPrimitiveCount);
    std::printf("}\n");
    return 0;
}
