// ltgp_pack.h — host-side packing of an opcode byte range for the PCIe
// transfer of a streamed evaluation (ltgp_evaluate_packed), and its layout.
//
// The streamed path copies every slice of the caller's host buffer to the
// device; at 1 B per node that copy is the bound of the end-to-end call
// (config 3: 856 MB, 15.4 ms at the pinned-copy ceiling). Opcodes are mostly
// the 5 small values (0-3 functions, 4 = X; opcodes.hpp:8-35), so each byte
// becomes a 3-bit code and only the others travel as literal bytes:
//
//   code 0-3  the function opcode itself      code 5  literal byte follows
//   code 4    X (opcode 4)                    code 6  0xFF (padding byte)
//
// The codes of a 16-byte packet are three 16-bit planes (bit k of plane j =
// bit j of byte k's code); literals follow in byte order. Lossless for all
// 256 byte values. Per slice the device buffer is
//
//   [plane0 u16 x npk][plane1 u16 x npk][plane2 u16 x npk]  (each padded to whole blocks)
//   [block literal base u32 x nblk]                         (padded to 64 B)
//   [literals]
//
// with npk = ceil(len / 16) packets and nblk = ceil(npk / 256) blocks of 256
// packets; block b's literals start at base[b]. k_decode's packed mode
// (ltgp_kernels.cuh) rebuilds the bytes, one CTA per block.
#pragma once
#include <stdint.h>
#include <string.h>

namespace ltgp_pack {

constexpr uint64_t kBlockPackets = 256;

inline uint64_t ceil16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

inline uint64_t ceil64(uint64_t x) { return (x + 63) & ~uint64_t(63); }

struct Layout {
    uint64_t npk, nblk;
    uint64_t plane_bytes;   // one plane, padded to whole blocks (512 B: a block's plane words)
    uint64_t base_off;      // block literal bases
    uint64_t lit_off;       // literals
    explicit Layout(uint64_t len) {
        npk = (len + 15) / 16;
        nblk = (npk + kBlockPackets - 1) / kBlockPackets;
        plane_bytes = nblk * kBlockPackets * 2;
        base_off = 3 * plane_bytes;
        lit_off = base_off + ceil64(nblk * 4);
    }
    // bytes of the packed slice for `literals` literal bytes
    uint64_t bytes(uint64_t literals) const { return lit_off + literals; }
    // worst case: every byte a literal
    uint64_t max_bytes() const { return lit_off + npk * 16 + 64; }
};

// Code of one byte.
inline uint32_t code_of(uint8_t b) { return b < 5 ? b : b == 0xff ? 6u : 5u; }

// Scalar encoder of blocks [b0, b1) of src[0, len): writes the three plane
// words of every packet of those blocks (packets past the end encode 0xFF
// bytes, so whole blocks are written), literals at lit (returns how many) and
// block b's literal count into blk_count[b - b0].
inline uint64_t encode_scalar(const uint8_t* src, uint64_t len, const Layout& L, uint8_t* dst, uint64_t b0,
                              uint64_t b1, uint8_t* lit, uint32_t* blk_count) {
    uint16_t* p0 = reinterpret_cast<uint16_t*>(dst);
    uint16_t* p1 = reinterpret_cast<uint16_t*>(dst + L.plane_bytes);
    uint16_t* p2 = reinterpret_cast<uint16_t*>(dst + 2 * L.plane_bytes);
    uint64_t n = 0;
    for (uint64_t b = b0; b < b1; ++b) {
        uint32_t nb = 0;
        for (uint64_t pk = b * kBlockPackets; pk < (b + 1) * kBlockPackets; ++pk) {
            uint32_t a = 0, bb = 0, c = 0;
            for (uint32_t k = 0; k < 16; ++k) {
                const uint64_t i = pk * 16 + k;
                const uint8_t v = i < len ? src[i] : 0xff;
                const uint32_t cd = code_of(v);
                a |= (cd & 1u) << k;
                bb |= ((cd >> 1) & 1u) << k;
                c |= ((cd >> 2) & 1u) << k;
                if (cd == 5u) lit[n + nb++] = v;
            }
            p0[pk] = (uint16_t)a;
            p1[pk] = (uint16_t)bb;
            p2[pk] = (uint16_t)c;
        }
        blk_count[b - b0] = nb;
        n += nb;
    }
    return n;
}

}  // namespace ltgp_pack

namespace ltgp_pack {

// Multi-threaded packer (ltgp_pack.cpp).
struct Pool;
Pool* pool_create(int nthreads);
void pool_destroy(Pool* p);
int pool_threads(const Pool* p);
bool have_avx512();
// Packs src[0, len) into dst (64-B aligned, Layout(len).max_bytes() bytes);
// returns the packed size. pack_start returns at once (the worker threads
// pack; the caller is free) and pack_wait waits for it: a streamed
// evaluation launches one slice's kernels while the next slice is packed.
// With caller_helps, pack_wait also packs a share on the calling thread.
uint64_t pack(Pool* p, const uint8_t* src, uint64_t len, uint8_t* dst);
void pack_start(Pool* p, const uint8_t* src, uint64_t len, uint8_t* dst, bool caller_helps);
uint64_t pack_wait(Pool* p);

// Reference decoder of one packed slice (tests and tools).
inline void unpack_scalar(const uint8_t* pk, uint64_t len, uint8_t* out) {
    const Layout L(len);
    const uint16_t* p0 = reinterpret_cast<const uint16_t*>(pk);
    const uint16_t* p1 = reinterpret_cast<const uint16_t*>(pk + L.plane_bytes);
    const uint16_t* p2 = reinterpret_cast<const uint16_t*>(pk + 2 * L.plane_bytes);
    const uint32_t* base = reinterpret_cast<const uint32_t*>(pk + L.base_off);
    const uint8_t* lit = pk + L.lit_off;
    uint64_t li = 0;
    for (uint64_t p = 0; p < L.npk; ++p) {
        if (p % kBlockPackets == 0) li = base[p / kBlockPackets];
        for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t c = ((p0[p] >> k) & 1u) | (((p1[p] >> k) & 1u) << 1) | (((p2[p] >> k) & 1u) << 2);
            const uint8_t v = c < 5 ? (uint8_t)c : c == 6 ? (uint8_t)0xff : lit[li++];
            if (p * 16 + k < len) out[p * 16 + k] = v;
        }
    }
}

}  // namespace ltgp_pack
