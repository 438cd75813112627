// ltgp_splice.cuh — device-side subtree crossover.
//
// k_extent replaces subtree_extent (/root/reference/proj/include/ltgp/
// genome.hpp:49-57): counter scan from the crossover point until the need
// count reaches zero, one warp per query, 512 opcode bytes per step.
// k_splice replaces crossover (genome.hpp:80-84):
// child = mum[0,ms) ++ dad[ds,de) ++ mum[me,n), one CTA per child, written as
// aligned 16-byte chunks assembled with funnel shifts from two aligned
// 16-byte loads of the (unaligned) parent bytes, which may live on a peer GPU
// (read over NVLink by UVA).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ltgp_dev {

struct DirEntry {          // one population slot
    const uint8_t* ptr;    // device address of the genome (any GPU, UVA)
    uint64_t size;
};

struct PlanDev {
    uint32_t mum, dad, mum_pt, dad_pt;
};

struct Extent {            // per child: mum [ms, me), dad [ds, de)
    uint32_t ms, me, ds, de;
};

// One warp per query q: child q/2, parent = mum (q even) or dad (q odd).
__global__ void __launch_bounds__(128) k_extent(const PlanDev* plans, uint32_t count,
                                                const DirEntry* dir, Extent* ext,
                                                uint64_t* child_size, uint32_t* err) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (q >= 2 * count) return;
    const uint32_t c = q >> 1;
    const bool is_dad = q & 1;
    const PlanDev p = plans[c];
    const DirEntry d = dir[is_dad ? p.dad : p.mum];
    const uint64_t pt = is_dad ? p.dad_pt : p.mum_pt;
    const uint64_t n = d.size;
    if (pt >= n) {  // std::out_of_range in the reference
        if (lane == 0) atomicOr(err, 4u);
        return;
    }
    int64_t need = 1;  // children still expected when reaching byte pos
    uint64_t base = pt & ~uint64_t(15);
    uint64_t end = 0;
    bool found = false;
    // the next 512-byte block is loaded while this one is scanned (long
    // subtrees of deep evolved trees take hundreds of dependent steps)
    auto load = [&](uint64_t b) {
        const uint64_t l = b + 16ull * lane;
        return l < n ? *reinterpret_cast<const uint4*>(d.ptr + l) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint4 wnext = load(base);
    while (!found && base < n) {
        const uint64_t lb = base + 16ull * lane;  // this lane's 16 bytes
        const uint4 w = wnext;
        wnext = load(base + 512);
        int delta[16];
        int tot = 0;
        if (lb < n) {
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t pos = lb + k;
                const uint32_t b = (ws[k >> 2] >> (8 * (k & 3))) & 0xffu;
                const int dk = (pos < pt || pos >= n) ? 0 : (b < 4u ? 1 : -1);
                delta[k] = dk;
                tot += dk;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) delta[k] = 0;
        }
        // exclusive warp scan of lane totals
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += v;
        }
        int run = (int)need + incl - tot;
        int hit = -1;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            run += delta[k];
            if (hit < 0 && delta[k] != 0 && run == 0) hit = k;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hit >= 0);
        if (m) {
            const int src = __ffs(m) - 1;
            const int h = __shfl_sync(0xffffffffu, hit, src);
            end = base + 16ull * src + (uint64_t)h + 1;
            found = true;
        } else {
            need += __shfl_sync(0xffffffffu, incl, 31);
            base += 512;
        }
    }
    if (!found) {
        if (lane == 0) atomicOr(err, 2u);
        return;
    }
    if (lane == 0) {
        if (is_dad) { ext[c].ds = (uint32_t)pt; ext[c].de = (uint32_t)end; }
        else { ext[c].ms = (uint32_t)pt; ext[c].me = (uint32_t)end; }
    }
}

// child size from both extents (crossover_child_size, genome.hpp:76-78)
__global__ void k_child_size(const PlanDev* plans, uint32_t count, const DirEntry* dir,
                             const Extent* ext, uint64_t* child_size) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    const Extent x = ext[c];
    const uint64_t mn = dir[plans[c].mum].size;
    child_size[c] = mn - (uint64_t)(x.me - x.ms) + (uint64_t)(x.de - x.ds);
}

// 16 bytes of a parent starting at src (any alignment): the two aligned
// 16-byte blocks that cover them, read through the non-coherent path (the
// block shared with the neighbouring thread's chunk hits in L1), then funnel
// shifts. ws/bs (word and bit offset of src within its block) are the same for
// every chunk of a segment, so the switch is warp-uniform.
__device__ __forceinline__ uint4 ld16_unaligned(const uint8_t* src) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uint4* al = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uint32_t off = (uint32_t)(a & 15);
    const uint4 x = __ldg(al);
    if (off == 0) return x;
    const uint4 y = __ldg(al + 1);
    const uint32_t bs = (off & 3) * 8;
    uint32_t w0, w1, w2, w3, w4;
    switch (off >> 2) {
        case 0: w0 = x.x; w1 = x.y; w2 = x.z; w3 = x.w; w4 = y.x; break;
        case 1: w0 = x.y; w1 = x.z; w2 = x.w; w3 = y.x; w4 = y.y; break;
        case 2: w0 = x.z; w1 = x.w; w2 = y.x; w3 = y.y; w4 = y.z; break;
        default: w0 = x.w; w1 = y.x; w2 = y.y; w3 = y.z; w4 = y.w; break;
    }
    return make_uint4(__funnelshift_r(w0, w1, bs), __funnelshift_r(w1, w2, bs), __funnelshift_r(w2, w3, bs),
                      __funnelshift_r(w3, w4, bs));
}

// One CTA per child; dst offsets are 16-aligned, bytes past the child up to
// the next 16-byte boundary are set to 0xff (never read as nodes). Each
// thread writes 16-byte chunks; a chunk inside one segment is one unaligned
// 16-byte copy, a chunk that straddles a segment boundary or the child's end
// (at most three per child) is assembled byte by byte.
__global__ void __launch_bounds__(256) k_splice(const PlanDev* plans, uint32_t count,
                                                const DirEntry* dir, const Extent* ext,
                                                const uint64_t* child_off, const uint64_t* child_size,
                                                uint8_t* arena, const uint32_t* skip) {
    if (skip && *skip) return;  // device-resident generation: a limit or capacity check failed
    for (uint32_t c = blockIdx.x; c < count; c += gridDim.x) {
        const PlanDev p = plans[c];
        const Extent x = ext[c];
        const uint8_t* mum = dir[p.mum].ptr;
        const uint8_t* dad = dir[p.dad].ptr;
        const uint64_t b1 = x.ms;                      // end of segment A
        const uint64_t b2 = b1 + (x.de - x.ds);        // end of segment B
        const uint64_t cn = child_size[c];
        uint4* dst = reinterpret_cast<uint4*>(arena + child_off[c]);
        const uint64_t nchunks = (cn + 15) / 16;
        for (uint64_t w = threadIdx.x; w < nchunks; w += blockDim.x) {
            const uint64_t q = 16 * w;
            const bool edge = (q < b1 && b1 < q + 16) || (q < b2 && b2 < q + 16) || (q + 16 > cn);
            uint4 v;
            if (!edge) {
                const uint8_t* src = q < b1 ? mum + q : q < b2 ? dad + x.ds + (q - b1) : mum + x.me + (q - b2);
                v = ld16_unaligned(src);
            } else {
                uint32_t t[4];
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    uint32_t word = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t pos = q + 4 * k4 + k;
                        uint32_t b = 0xffu;
                        if (pos < cn) b = pos < b1 ? mum[pos] : pos < b2 ? dad[x.ds + (pos - b1)]
                                                                        : mum[x.me + (pos - b2)];
                        word |= b << (8 * k);
                    }
                    t[k4] = word;
                }
                v = make_uint4(t[0], t[1], t[2], t[3]);
            }
            dst[w] = v;
        }
    }
}

}  // namespace ltgp_dev
