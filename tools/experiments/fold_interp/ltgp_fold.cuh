// ltgp_fold.cuh — the folded-leaf interpreter: k_fold (per-item pre-pass)
// and k_eval2 (the warp interpreter of its micro-ops).
//
// Same computation as eval_batch_raw (/root/reference/proj/include/ltgp/
// eval.hpp:70-79): a reverse scan of the prefix buffer in
// which every function node applies apply_op (eval.hpp:54-63) to its left
// operand (the top) and right operand (below it), once, in scan order. What
// changes is who does the bookkeeping.
//
// k_fold (one THREAD per work item) replays the item's reverse scan on a
// stack of operand REFERENCES instead of values: a leaf pushes its opcode, a
// function pops two references and pushes "computed". For every function
// node it emits one 32-bit micro-op naming its operand kinds, so leaves are
// never pushed as values: a leaf operand is read straight from the leaf
// table by the function that consumes it (leaf folding). The kinds are
//   LL   both operands leaves      T' = op(A, B), the old T pushed first
//   LL0  both leaves, nothing live T' = op(A, B)
//   CL   left computed (= T)       T' = op(T, B)      (also the commuted
//   LC   left leaf, right = T      T' = op(A, T)       ADD/MUL of LC)
//   CC   both computed             T' = op(T, pop)
// where T is the top computed value, kept in registers by the interpreter;
// computed values below it live in a per-warp shared window of kWin2 frames,
// spilled to / refilled from global memory by SPILL / FILL micro-ops that
// k_fold plans exactly (it simulates the window). The same pass computes
// every node's depth as an exact integer (genome.hpp:45-46), sizes chunk
// summaries exactly and claims them from the pool, and flags malformed
// input (underflow, leftovers, opcode 255).
//
// k_eval2 (one WARP per item, persistent grid) runs the micro-ops with the
// generated direct-threaded fast path (ltgp_interp2_gen.cuh): one dispatch
// per function node, which covers the node and its leaf operands, i.e. about
// two tree nodes per dispatch, with no per-node depth or leaf-push work.
// Rare events (chunk spine steps, the item's end) exit to C++.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ltgp_interp2_gen.cuh"

namespace ltgp_dev {

constexpr int kWin2 = 24;              // shared window frames per warp
constexpr uint32_t kFS2 = 192;         // window frame: 24 value lanes x float2
constexpr uint32_t kRing2 = 256;       // micro-op ring: 2 groups of 32 words

// micro-op handler indices (word bits 0-4; bit 5: the word ends a 32-word group)
enum : uint32_t {
    U_LL = 0, U_LL0 = 4, U_CL = 8, U_CC = 12, U_LCSUB = 16, U_LCDIV = 17,
    U_SPILL = 18, U_FILL = 19, U_EXIT = 20
};
// EXIT codes (word byte 1)
enum : uint32_t { X_END = 0, X_SPINE_T = 1, X_SPINE_L = 2, X_SPINE_B = 3 };

struct FoldItem {
    uint32_t flags;    // bit0: capacity (needs the worst-case tier), bit1: malformed
    uint32_t nwords;
    uint32_t spill;    // most frames this item spills
    uint32_t pad;
};

struct FoldArgs {
    const uint8_t* arena;
    const uint64_t* off;
    const Item* items;
    uint32_t n_items;
    const uint64_t* wbase;   // per item: word offset of its micro-op stream (a multiple of 32)
    uint32_t* words;
    FoldItem* fitem;
    uint32_t* kstack;        // reference-stack scratch: kcap entries per thread, interleaved
    uint32_t kcap;
    uint32_t kstride;        // threads sharing the interleaved scratch (entry j of thread t at j*kstride + t)
    uint32_t spill_cap;      // per-warp spill frames of k_eval2
    PlanPool pool;           // chunk summaries (exactly sized here)
    float* rec;              // records: depth of whole trees (k_eval2 writes the rest)
    uint32_t* counters;      // [1] flags, [2] capacity items, [5] window adjusts
};

// word capacity of an item of n nodes (host and device agree): <= one word
// per function node or spine step, window adjusts, the end list (<= n + 2)
__host__ __device__ __forceinline__ uint64_t fold_word_cap(uint32_t n, bool chunk) {
    const uint64_t c = chunk ? (uint64_t)n + n / 4 : (uint64_t)(n / 2) + n / 8;
    return (c + 96 + 31) & ~uint64_t(31);
}

constexpr uint32_t kLeafMark = 0x80000000u;  // stack entry: computed | depth (else a leaf opcode)

// One work item's reverse scan on references. Thread-serial; written so
// that the common node (a leaf push, or a function with two local operands
// and no window adjust) is branch-light: the threads of a warp walk
// different items. The stack's top two entries stay in registers (top,
// nos); deeper ones live in the interleaved scratch ks[j * stride]. K-frame
// depths are kept from the scratch's far end downwards.
__device__ void fold_item(const FoldArgs& a, uint32_t i, uint32_t* ks, uint32_t kst) {
    const Item it = a.items[i];
    const bool chunk = it.chunk != kWholeTree;
    const uint8_t* tb = a.arena + a.off[it.tree];
    uint32_t* w = a.words + a.wbase[i];
    const uint32_t wcap = (uint32_t)fold_word_cap(it.hi - it.lo, chunk);
    const uint32_t S = (uint32_t)kWin2;
    const uint32_t kcap = a.kcap;
    uint32_t nw = 0, flags = 0, nadj = 0;
    uint32_t h = 0, top = 0, nos = 0;
    uint32_t vcnt = 0, nwin = 0, spilled = 0, spill_max = 0;  // computed values: T + window + spilled
    uint32_t nsteps = 0, nkf = 0;
    auto emit = [&](uint32_t x) {  // a dispatched word: bit 5 marks the end of a 32-word group
        if (nw < wcap) w[nw] = x | ((nw & 31u) == 31u ? 32u : 0u);
        ++nw;
    };
    for (int64_t pos = (int64_t)it.hi - 1; pos >= (int64_t)it.lo && !(flags & 3u); ) {
        const int64_t pbase = pos & ~int64_t(15);
        const uint4 pk = *reinterpret_cast<const uint4*>(tb + pbase);
        const int64_t stop = max(pbase, (int64_t)it.lo);
        for (; pos >= stop; --pos) {
            const uint32_t k = (uint32_t)(pos - pbase);
            const uint32_t wd = k < 8u ? (k < 4u ? pk.x : pk.y) : (k < 12u ? pk.z : pk.w);
            const uint32_t b = (wd >> (8u * (k & 3u))) & 0xffu;
            const bool leaf = b >= 4u;
            if (leaf && b == 255u) { flags |= 2u; break; }
            if (!leaf && h < 2) {  // a spine step (chunk) or underflow (malformed)
                if (!chunk) { flags |= 2u; break; }
                if (h == 1) {  // form A: the one local value is the K frame
                    const bool tl = top < kLeafMark;
                    if (nkf + 1 >= kcap) { flags |= 1u; break; }
                    ks[(kcap - 1 - nkf) * kst] = tl ? 1u : (top & ~kLeafMark);  // K frame depth
                    ++nkf;
                    emit(tl ? (U_EXIT | (X_SPINE_L << 8) | (top << 16) | (b << 24)) : (U_EXIT | (X_SPINE_T << 8) | (b << 24)));
                    if (!tl) vcnt = 0;  // T was the only live value
                    h = 0;
                } else {
                    emit(U_EXIT | (X_SPINE_B << 8) | (b << 24));
                }
                ++nsteps;
                continue;
            }
            // push (leaf) or pop-two-push-one (function): memory traffic
            // predicated, register updates by selects
            if (leaf && h >= 2) {
                if (h - 2 + nkf >= kcap) { flags |= 1u; break; }
                ks[(h - 2) * kst] = nos;
            }
            const uint32_t deeper = (!leaf && h >= 3) ? ks[(h - 3) * kst] : 0u;
            const uint32_t x = top, y = nos;
            nos = leaf ? top : deeper;
            h = leaf ? h + 1 : h - 1;
            if (leaf) {
                top = b;
                continue;
            }
            const bool xl = x < kLeafMark, yl = y < kLeafMark;
            const uint32_t dx = xl ? 1u : (x & ~kLeafMark), dy = yl ? 1u : (y & ~kLeafMark);
            top = kLeafMark | (max(dx, dy) + 1u);
            uint32_t word;
            if (xl && yl) {
                if (vcnt >= 1) {
                    if (nwin == S) {  // the window is full: spill its bottom half
                        emit(U_SPILL | ((S / 2) << 24));
                        spilled += S / 2;
                        nwin -= S / 2;
                        ++nadj;
                        spill_max = max(spill_max, spilled);
                    }
                    ++nwin;
                }
                word = (vcnt >= 1 ? U_LL : U_LL0) + b;
                word |= (x << 8) | (y << 16);
                ++vcnt;
            } else if (!xl && yl) {
                word = (U_CL + b) | (y << 16);
            } else if (xl) {  // LC: commutative ops run as CL with the leaf as B
                word = (b == 0u || b == 2u) ? ((U_CL + b) | (x << 16)) : ((b == 1u ? U_LCSUB : U_LCDIV) | (x << 8));
            } else {          // CC: the right operand is the window's top frame
                if (nwin == 0) {
                    const uint32_t k2 = min(spilled, S / 2);
                    emit(U_FILL | (k2 << 24));
                    spilled -= k2;
                    nwin += k2;
                    ++nadj;
                }
                --nwin;
                --vcnt;
                word = U_CC + b;
            }
            emit(word);
        }
    }
    // end list: the remaining references bottom to top (computed | leaf opcode)
    if (!(flags & 3u)) {
        if (!chunk && h != 1) flags |= 2u;
        emit(U_EXIT | (X_END << 8));
        if (nw + 1 + h <= wcap) {
            w[nw] = h;
            for (uint32_t j = 0; j < h; ++j) {
                const uint32_t e = j + 1 == h ? top : j + 2 == h ? nos : ks[j * kst];
                w[nw + 1 + j] = e < kLeafMark ? e : kLeafMark;
            }
        }
        nw += 1 + h;
        if (nw > wcap) flags |= 1u;
    }
    if (spill_max > a.spill_cap) flags |= 1u;
    if (nadj) atomicAdd(&a.counters[5], nadj);
    if (flags & 2u) atomicOr(&a.counters[1], 2u);
    if (!(flags & 3u)) {
        if (!chunk) {
            const uint32_t d = top < kLeafMark ? 1u : (top & ~kLeafMark);
            a.rec[(size_t)it.tree * 4 + 3] = __uint_as_float(d);
        } else if (a.pool.hdr) {  // claim the exact summary: K frames, then the outputs
            const unsigned long long nf = (unsigned long long)nkf + h, ns = nsteps;
            const unsigned long long f0 = atomicAdd(&a.pool.used[0], nf), s0 = atomicAdd(&a.pool.used[1], ns);
            if (f0 + nf <= a.pool.cap_frames && s0 + ns <= a.pool.cap_steps) {
                ChunkHdr hd{};
                hd.n_steps = (uint32_t)ns;
                hd.n_kframes = nkf;
                hd.n_out = h;
                float2* fr = a.pool.frames + f0 * 32;
                hd.frames = fr;
                hd.steps = a.pool.steps + s0;
                // depths ride in lane 24's .x of every summary frame (the spine
                // combine's integer depth chain reads them there)
                for (uint32_t j = 0; j < nkf; ++j) fr[(size_t)j * 32 + 24].x = __uint_as_float(ks[(kcap - 1 - j) * kst]);
                for (uint32_t j = 0; j < h; ++j) {
                    const uint32_t e = j + 1 == h ? top : j + 2 == h ? nos : ks[j * kst];
                    fr[(size_t)(nkf + j) * 32 + 24].x = __uint_as_float(e < kLeafMark ? 1u : (e & ~kLeafMark));
                }
                a.pool.hdr[it.chunk] = hd;
            } else {
                flags |= 1u;  // the pool is full: this chunk goes to the worst-case tier
            }
        }
    }
    if ((flags & 3u) && chunk && a.pool.hdr) {  // nothing usable for the spine combine
        ChunkHdr hd{};
        hd.flags = flags;
        a.pool.hdr[it.chunk] = hd;
    }
    if (flags & 1u) atomicAdd(&a.counters[2], 1u);
    a.fitem[i] = FoldItem{flags, nw, spill_max, 0u};
}

// A persistent grid of threads, each folding items i = tid, tid + nthreads, ...
// with its own reference-stack scratch (entries interleaved across threads
// so a warp's stack accesses at equal depths share cache lines).
__global__ void __launch_bounds__(128) k_fold(FoldArgs a) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nth = gridDim.x * blockDim.x;
    uint32_t* ks = a.kstack + tid;
    for (uint32_t i = tid; i < a.n_items; i += nth) fold_item(a, i, ks, a.kstride);
}

// ---------------------------------------------------------------------------
// k_eval2: the warp interpreter.
// ---------------------------------------------------------------------------
struct Eval2Args {
    const Item* items;
    uint32_t n_items;
    const uint64_t* wbase;
    const uint32_t* words;
    const FoldItem* fitem;
    ChunkHdr* hdr;
    float2* spill;             // per resident warp: spill_frames frames of 256 B
    uint32_t spill_frames;
    float* rec;
    float* outs;
    uint32_t* counters;        // [4] exits
    uint32_t* queue;
};

template <int WARPS>
struct Eval2Layout {
    // per warp: micro-op ring (256 B), the window (kWin2 x 192 B) and 64 B
    // of slack (lanes 24..31 read 64 bytes past the top frame)
    static constexpr uint32_t kWarpBytes = kRing2 + kWin2 * kFS2 + 64;
    static constexpr uint32_t kBytes = kTableBytes + (WARPS + 1) * kWarpBytes;
};

__device__ __forceinline__ float2 u64_to_f2(uint64_t t) {
    return make_float2(__uint_as_float((uint32_t)t), __uint_as_float((uint32_t)(t >> 32)));
}

// fitness / hits / size of a whole tree (depth: written by k_fold)
__device__ __forceinline__ void write_record2(uint32_t lane, float2 tv, float2 o, uint32_t size, float* rec,
                                              float* outs) {
    if (outs && lane < 24) {
        outs[2 * lane] = o.x;
        outs[2 * lane + 1] = o.y;
    }
    const bool vl = lane < 24;
    const float dx = fabsf(__fsub_rn(o.x, tv.x));
    const float dy = fabsf(__fsub_rn(o.y, tv.y));
    const uint32_t hx = __ballot_sync(0xffffffffu, vl && dx <= 0.01f);
    const uint32_t hy = __ballot_sync(0xffffffffu, vl && dy <= 0.01f);
    float sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 24; ++j) {  // fitness (eval.hpp:81-84): cases 0..47 in order, then / 48
        sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, dx, j));
        sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, dy, j));
    }
    float fit = __fdiv_rn(sum, 48.0f);
    if (fit != fit) fit = __int_as_float(0x7fc00000);
    if (lane == 0) {
        rec[0] = fit;
        rec[1] = __int_as_float((int)(__popc(hx) + __popc(hy)));
        rec[2] = __uint_as_float(size);
    }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_eval2(Eval2Args a, SuiteArgs s) {
    extern __shared__ __align__(1024) unsigned char smem2[];
    using L = Eval2Layout<WARPS>;
    const uint32_t s0 = smem_addr(smem2);
    const uint32_t tab = (s0 + 0xffffu) & ~0xffffu;  // 64 KB aligned leaf table
    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    // leaf table: row = opcode, column l < 24: (x or c) for cases 2l, 2l+1
    for (uint32_t i = threadIdx.x; i < 256u * 32u; i += blockDim.x) {
        const uint32_t row = i >> 5, col = i & 31u;
        float2 v = make_float2(0.0f, 0.0f);
        if (col < 24u) v = row == 4u ? s.x[col] : make_float2(s.c[row], s.c[row]);
        sts2(tab + row * 256u + col * 8u, v);
    }
    __syncthreads();
    const uint32_t n_low = (tab - s0) / L::kWarpBytes;  // warp regions that fit below the table
    const uint32_t wstart = warp < n_low ? s0 + warp * L::kWarpBytes : tab + kTableBytes + (warp - n_low) * L::kWarpBytes;
    if (wstart + L::kWarpBytes > s0 + L::kBytes) {
        if (lane == 0) atomicOr(&a.counters[1], 8u);
        return;
    }
    const uint32_t ring = wstart;
    const uint32_t lane8 = lane * 8u;
    const uint32_t wslot0 = wstart + kRing2 + lane8;  // window slot 0, this lane's column
    const uint32_t lb = tab | lane8;
    const float2 tv = lane < 24 ? s.t[lane] : make_float2(0.0f, 0.0f);
    const uint32_t pv = lane < 24 ? 1u : 0u;
    float2* spill = a.spill + ((size_t)(blockIdx.x * WARPS + warp) * a.spill_frames) * 32 + lane;
    uint32_t nexit = 0;
    while (true) {
        uint32_t i = 0;
        if (lane == 0) i = atomicAdd(a.queue, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= a.n_items) break;
        const FoldItem fi = a.fitem[i];
        if (fi.flags & 3u) continue;  // malformed (reported) or left to the worst-case tier
        const Item it = a.items[i];
        const bool chunk = it.chunk != kWholeTree;
        const uint32_t* ws = a.words + a.wbase[i];
        float2* kfr = nullptr;
        uint8_t* stp = nullptr;
        if (chunk) {
            const ChunkHdr h = a.hdr[it.chunk];
            kfr = const_cast<float2*>(h.frames) + lane;
            stp = const_cast<uint8_t*>(h.steps);
        }
        uint64_t T = 0;
        uint32_t sp = wslot0, spilled = 0, nA = 0, ns = 0;
        int wi = 0;
        while (true) {
            run_uops(T, sp, wi, spilled, ring, lane * 4u, lb, ws, wslot0, spill, pv);
            ++nexit;
            const uint32_t wd = ws[wi];
            const uint32_t code = (wd >> 8) & 0xffu;
            if (code == X_END) break;
            const uint32_t op = wd >> 24;
            if (code == X_SPINE_B) {
                if (lane == 0) stp[ns] = (uint8_t)(op | 4u);
            } else {  // form A: the one local value is the K frame
                const float2 v = code == X_SPINE_T ? u64_to_f2(T) : lds2(lb | (((wd >> 16) & 0xffu) << 8));
                if (lane < 24) kfr[(size_t)nA * 32] = v;
                if (lane == 0) stp[ns] = (uint8_t)op;
                ++nA;
            }
            ++ns;
            ++wi;
        }
        // the end list: remaining references bottom to top
        const uint32_t n_out = ws[wi + 1];
        if (!chunk) {
            const uint32_t e = ws[wi + 2];
            const float2 v = e == kLeafMark ? u64_to_f2(T) : lds2(lb | (e << 8));
            write_record2(lane, tv, v, it.hi, a.rec + (size_t)it.tree * 4,
                          a.outs ? a.outs + (size_t)it.tree * kLanes : nullptr);
            continue;
        }
        // computed outputs in stack order: spilled frames, window frames, T
        const uint32_t nwin = (sp - wslot0) / kFS2;
        uint32_t c = 0;
        for (uint32_t j = 0; j < n_out; ++j) {
            const uint32_t e = ws[wi + 2 + j];
            float2 v;
            if (e != kLeafMark) {
                v = lds2(lb | (e << 8));
            } else {
                v = c < spilled ? spill[(size_t)c * 32] : c < spilled + nwin ? lds2(wslot0 + (c - spilled) * kFS2)
                                                                            : u64_to_f2(T);
                ++c;
            }
            if (lane < 24) kfr[(size_t)(nA + j) * 32] = v;
        }
    }
    if (lane == 0 && nexit) atomicAdd(&a.counters[4], nexit);
}

}  // namespace ltgp_dev
