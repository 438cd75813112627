// ltgp_gen.cuh — device-resident generation control (single-shard engines).
//
// execute_generation (/root/reference/proj/include/ltgp/evolve.hpp:111-117)
// as one launch sequence with one readback: the parents' slot directory, the
// children's sizes (crossover_child_size, genome.hpp:76-78), the
// MemoryBudgetExceeded / SizeLimitHit checks (evolve.hpp:89-93,
// genome.hpp:71-84), the children's arena layout and
// the evaluation work list are computed here, on the device, between
// k_extent and k_splice / k_plan_warp / k_eval. The host path of the engine
// (ltgp_engine.cu: build_directory, set_layout, launch_eval's work list) is
// the same algorithm; this is its device restatement, so the host waits once
// per generation instead of three times and builds nothing per child.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ltgp_kernels.cuh"
#include "ltgp_splice.cuh"

namespace ltgp_dev {

constexpr uint32_t kGenBuckets = 33;  // log2 size buckets (bucket(n) = 32 - clz(n))

// Written by k_gen_control, read by the kernels after it and by the host.
struct GenStatus {
    uint32_t fatal;       // nothing is spliced: bit0 child >= node_limit, bit1 planned bytes > budget,
                          // bit2 child > 2^32-1 nodes, bit3 child arena too small, bit5 extent scan error
    uint32_t flags;       // fatal | bit4: work list beyond its buffers (children spliced, not evaluated)
    uint32_t n_items;     // work list length (0 when flags != 0)
    uint32_t n_trees;     // chunked trees  } CombineArgs::counts_dev
    uint32_t n_chunks;    // chunks         }
    uint32_t max_chunks;  // most chunks of one tree
    uint32_t chunk;       // chunk length C
    uint32_t lpt;         // items longest first (1) or chunks in tree order first (0)
    uint32_t need_items;  // the work list's length and chunks, also when bit4 is set
    uint32_t need_chunks;
    unsigned long long child_bytes;    // children's arena bytes (16-B aligned each)
    unsigned long long nodes;          // sum of child sizes
    unsigned long long planned_bytes;  // parents' + children's genome bytes (the budget's measure)
    unsigned long long max_child;      // largest child
    uint32_t wpos[kGenBuckets];  // k_gen_items: next slot of a whole tree of bucket b
    uint32_t cpos[kGenBuckets];  // next slot of an LPT-ordered chunk of bucket b
};

struct GenArgs {
    const PlanDev* plans;
    const DirEntry* dir;        // parents
    const Extent* ext;
    const uint32_t* ext_err;    // k_extent's error word
    uint32_t M;
    unsigned long long node_limit, budget, arena_cap;  // budget 0: no check
    uint64_t* csize;            // children: sizes (u64, k_splice)
    uint64_t* child_off;        //   arena offsets (the child TreeSet's off)
    uint32_t* child_size;       //   sizes (the child TreeSet's size)
    uint32_t* tree_chunk0;      // per child: first chunk id (chunked trees)
    uint32_t* tree_ct;          // per child: combine-tree index (chunked trees)
    Item* items;
    uint32_t items_cap;
    CombineTree* ctrees;
    uint32_t chunks_cap;        // chunk summaries the per-chunk buffers hold
    uint32_t fixed_chunk;       // 0: automatic chunk length
    uint32_t default_chunk, max_chunk, max_wave_chunk;
    uint32_t grid_warps;        // k_eval's persistent warps
    GenStatus* st;
};

// parents' directory: slot i at arena + off[i]
__global__ void k_gen_dir(const uint8_t* arena, const uint64_t* off, const uint32_t* size, uint32_t M,
                          DirEntry* dir) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M) dir[i] = DirEntry{arena + off[i], size[i]};
}

__device__ __forceinline__ uint32_t gen_bucket(uint32_t n) { return 32u - (uint32_t)__clz(n); }

// Block-wide exclusive scan (1024 threads = 32 warps) with the block total.
template <class T>
__device__ __forceinline__ T gen_scan(T v, T& total, T* wsum) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const T w = wsum[lane];
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(0xffffffffu, wi, o);
            if ((int)lane >= o) wi += t;
        }
        wsum[lane] = wi - w;         // exclusive warp offsets
        if (lane == 31) wsum[32] = wi;
    }
    __syncthreads();
    const T r = wsum[warp] + incl - v;
    total = wsum[32];
    __syncthreads();
    return r;
}

template <class T>
__device__ __forceinline__ T gen_sum(T v, T* wsum) {
    T total;
    gen_scan<T>(v, total, wsum);
    return total;
}

__device__ __forceinline__ unsigned long long gen_max(unsigned long long v, unsigned long long* wm) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) wm[warp] = v;
    __syncthreads();
    unsigned long long r = 0;
    for (int w = 0; w < 32; ++w) r = max(r, wm[w]);
    __syncthreads();
    return r;
}

// One block of 1024 threads. Children sizes and layout, the limit checks,
// the chunk length and the work list's counts and bucket bases. On a failed
// check the status says why and every later kernel of the generation does
// nothing (k_splice, k_gen_items, k_plan_warp, k_eval and the combine read
// the status).
__global__ void __launch_bounds__(1024) k_gen_control(GenArgs a) {
    __shared__ unsigned long long w64[33];
    __shared__ uint32_t w32[33];
    __shared__ uint32_t wcnt[kGenBuckets], ccnt[kGenBuckets];
    GenStatus* st = a.st;
    const uint32_t M = a.M;
    // 1. child sizes, offsets, limits (crossover_child_size: genome.hpp:76-78)
    unsigned long long carry = 0, nodes = 0, planned = 0, biggest = 0;
    uint32_t fatal = 0;
    for (uint32_t t0 = 0; t0 < M; t0 += 1024) {
        const uint32_t t = t0 + threadIdx.x;
        unsigned long long n = 0, pb = 0;
        if (t < M) {
            const PlanDev p = a.plans[t];
            const Extent x = a.ext[t];
            n = a.dir[p.mum].size - (unsigned long long)(x.me - x.ms) + (unsigned long long)(x.de - x.ds);
            pb = a.dir[t].size;
            a.csize[t] = n;
            if (n >= a.node_limit) fatal |= 1u;
            if (n > 0xffffffffull) fatal |= 4u;
        }
        unsigned long long tot;
        const unsigned long long o = gen_scan<unsigned long long>((n + 15) & ~15ull, tot, w64);
        if (t < M) {
            a.child_off[t] = carry + o;
            a.child_size[t] = (uint32_t)n;
        }
        carry += tot;
        nodes += n;
        planned += pb + n;
        biggest = max(biggest, n);
    }
    nodes = gen_sum<unsigned long long>(nodes, w64);
    planned = gen_sum<unsigned long long>(planned, w64);
    biggest = gen_max(biggest, w64);
    {   // the OR of every thread's bits
        __shared__ uint32_t fsh;
        if (threadIdx.x == 0) fsh = 0;
        __syncthreads();
        if (fatal) atomicOr(&fsh, fatal);
        __syncthreads();
        fatal = fsh;
    }
    if (a.budget && planned > a.budget) fatal |= 2u;   // MemoryBudgetExceeded (evolve.hpp:89-93)
    if (carry + 64 > a.arena_cap) fatal |= 8u;
    if (*a.ext_err) fatal |= 32u;
    if (threadIdx.x == 0) {
        st->fatal = fatal;
        st->child_bytes = carry;
        st->nodes = nodes;
        st->planned_bytes = planned;
        st->max_child = biggest;
        st->n_items = st->n_trees = st->n_chunks = st->max_chunks = 0;
        st->flags = fatal;
    }
    if (fatal) return;
    // 2. chunk length: launch_eval's rule (ltgp_engine.cu), restated
    uint32_t C = a.fixed_chunk;
    if (!C) {
        const unsigned long long W = a.grid_warps;
        const unsigned long long per = nodes / (W + 1);
        C = 1024;
        while (C < a.default_chunk && (unsigned long long)C * 4 <= per * 3) C *= 2;
        const double want = pow(1.25 * (double)biggest, 2.0 / 3.0);
        while (C < a.max_chunk && (double)C < want) C *= 2;
        auto chunks_of = [&](uint32_t c, uint32_t* big, unsigned long long* bign) {
            unsigned long long k = 0, bn = 0;
            uint32_t b = 0;
            for (uint32_t t = threadIdx.x; t < M; t += 1024) {
                const uint32_t n = a.child_size[t];
                if (n > c) { k += (n + c - 1) / c; ++b; bn += n; }
            }
            k = gen_sum<unsigned long long>(k, w64);
            if (big) *big = gen_sum<uint32_t>(b, w32);
            if (bign) *bign = gen_sum<unsigned long long>(bn, w64);
            return k;
        };
        uint32_t big_trees = 0;
        unsigned long long big_nodes = 0;
        const unsigned long long k0 = chunks_of(C, &big_trees, &big_nodes);
        const unsigned long long waves = (k0 + W - 1) / W;
        if ((k0 > W / 2 || big_nodes * 2 >= nodes) && waves <= 8 && C >= 2048 && big_trees <= 512) {
            // one chunk per warp where max_wave_chunk allows it, else the fewest waves
            const unsigned long long kw = chunks_of(a.max_wave_chunk, nullptr, nullptr);
            const unsigned long long w = max(1ull, (kw + W - 1) / W);
            uint32_t lo = 1, hi = a.max_wave_chunk / 1024;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) / 2;
                if (chunks_of(mid * 1024, nullptr, nullptr) <= w * W) hi = mid; else lo = mid + 1;
            }
            C = max(hi * 1024, max(1024u, C / 2));
        }
    }
    // 3. counts per bucket, chunk ids and combine-tree indices in tree order
    if (threadIdx.x < kGenBuckets) { wcnt[threadIdx.x] = 0; ccnt[threadIdx.x] = 0; }
    __syncthreads();
    uint32_t ch_carry = 0, ct_carry = 0, maxk = 0;
    for (uint32_t t0 = 0; t0 < M; t0 += 1024) {
        const uint32_t t = t0 + threadIdx.x;
        uint32_t k = 0;
        if (t < M) {
            const uint32_t n = a.child_size[t];
            if (n <= C) {
                atomicAdd(&wcnt[gen_bucket(n)], 1u);
            } else {
                k = (n + C - 1) / C;
                atomicAdd(&ccnt[gen_bucket(C)], k - 1);
                atomicAdd(&ccnt[gen_bucket(n - (k - 1) * C)], 1u);
                maxk = max(maxk, k);
            }
        }
        uint32_t tk, tc;
        const uint32_t ok = gen_scan<uint32_t>(k, tk, w32);
        const uint32_t oc = gen_scan<uint32_t>(k ? 1u : 0u, tc, w32);
        if (t < M && k) {
            a.tree_chunk0[t] = ch_carry + ok;
            a.tree_ct[t] = ct_carry + oc;
        }
        ch_carry += tk;
        ct_carry += tc;
    }
    maxk = (uint32_t)gen_max(maxk, w64);
    if (threadIdx.x == 0) {
        uint32_t whole = 0;
        for (uint32_t b = 0; b < kGenBuckets; ++b) whole += wcnt[b];
        const uint32_t nitems = ch_carry + whole;
        st->chunk = C;
        st->max_chunks = maxk;
        st->need_items = nitems;
        st->need_chunks = ch_carry;
        if (nitems > a.items_cap || ch_carry > a.chunks_cap) {
            st->flags = fatal | 16u;  // the host evaluates these children after growing the buffers
        } else {
            // resident evaluations of <= 8 waves take all items longest first
            // (chunks before whole trees within a bucket); longer work lists
            // keep the chunks in tree order, then whole trees by bucket
            const bool lpt = (unsigned long long)nitems <= 8ull * a.grid_warps;
            uint32_t pos = 0;
            if (lpt) {
                for (int b = kGenBuckets - 1; b >= 0; --b) {
                    st->cpos[b] = pos; pos += ccnt[b];
                    st->wpos[b] = pos; pos += wcnt[b];
                }
            } else {
                pos = ch_carry;
                for (int b = kGenBuckets - 1; b >= 0; --b) { st->cpos[b] = 0; st->wpos[b] = pos; pos += wcnt[b]; }
            }
            st->lpt = lpt ? 1u : 0u;
            st->n_items = nitems;
            st->n_chunks = ch_carry;
            st->n_trees = ct_carry;
            st->flags = fatal;
        }
    }
}

// A warp per child: its work items (whole tree, or chunks [q C, (q+1) C))
// and its combine tree, at the slots k_gen_control's bases give.
__global__ void __launch_bounds__(256) k_gen_items(GenArgs a) {
    GenStatus* st = a.st;
    if (st->flags) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= a.M) return;
    const uint32_t C = st->chunk;
    const uint32_t n = a.child_size[t];
    if (n <= C) {
        if (lane == 0) a.items[atomicAdd(&st->wpos[gen_bucket(n)], 1u)] = Item{t, kWholeTree, 0, n};
        return;
    }
    const uint32_t k = (n + C - 1) / C;
    const uint32_t c0 = a.tree_chunk0[t];
    const bool lpt = st->lpt != 0;
    uint32_t full0 = 0, last = 0;  // LPT slots: k - 1 full chunks, then the last one
    if (lane == 0) {
        a.ctrees[a.tree_ct[t]] = CombineTree{t, c0, k, n};
        if (lpt) {
            full0 = atomicAdd(&st->cpos[gen_bucket(C)], k - 1);
            last = atomicAdd(&st->cpos[gen_bucket(n - (k - 1) * C)], 1u);
        }
    }
    full0 = __shfl_sync(0xffffffffu, full0, 0);
    last = __shfl_sync(0xffffffffu, last, 0);
    for (uint32_t q = lane; q < k; q += 32) {
        const uint32_t lo = q * C, hi = min(n, lo + C);
        const uint32_t slot = !lpt ? c0 + q : q + 1 < k ? full0 + q : last;
        a.items[slot] = Item{t, c0 + q, lo, hi};
    }
}

}  // namespace ltgp_dev
