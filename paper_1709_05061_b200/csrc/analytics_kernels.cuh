// analytics_kernels.cuh — sweeps over the gapped slot array shared by the
// whole-graph analytics (graph.cu) and the sharded ones (shard.cu); internal
// linkage, one copy per translation unit.
#pragma once

#include "block_ops.cuh"

namespace gpma {

// Sweeps over the slot array in warp steps of 256 slots: lane l loads the
// slot pairs (64 q + 2 l, 64 q + 2 l + 1), q = 0..3 — every load instruction
// of the warp is one contiguous 512-B key run (16 B per lane) plus a 64-B
// state run, and all eight loads are in flight before any is used.  `f(key)`
// runs for every Valid non-guard slot.  cap is a multiple of 16; a partial
// last step is masked.
template <class F>
__device__ __forceinline__ void sweep_edges8(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap, F f) {
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 base = warp * 256; base < cap; base += nwarps * 256) {
        ulonglong2 kk[4];
        unsigned short ss[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u64 t = base + 64 * q + 2 * lane;
            if (t < cap) {
                ss[q] = __ldcs(reinterpret_cast<const unsigned short*>(st + t));
                kk[q] = __ldcs(reinterpret_cast<const ulonglong2*>(keys + t));
            } else {
                ss[q] = 0;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((ss[q] & 0xFF) == kValid && !is_guard(kk[q].x)) f(kk[q].x);
            if ((ss[q] >> 8) == kValid && !is_guard(kk[q].y)) f(kk[q].y);
        }
    }
}

// The same sweep, but the Valid non-guard keys of each 256-slot step are
// first packed into the warp's shared queue (ballot + popc ranks), then `f`
// runs over the queue with every lane busy.  With C/E ~ 4.5 most slots are
// gaps or guards: calling `f` straight from the slot lanes leaves ~1/3 of
// them active, which is what bounds an `f` with real work (PageRank's
// hot-table probe + atomics).  `queue` = 256 keys per warp of the block.
template <class F>
__device__ __forceinline__ void sweep_edges8_packed(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                    u64* queue, F f) {
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    u64* q = queue + (threadIdx.x >> 5) * 256;
    const unsigned below = lanemask_lt();
    for (u64 base = warp * 256; base < cap; base += nwarps * 256) {
        ulonglong2 kk[4];
        unsigned short ss[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const u64 t = base + 64 * j + 2 * lane;
            if (t < cap) {
                ss[j] = __ldcs(reinterpret_cast<const unsigned short*>(st + t));
                kk[j] = __ldcs(reinterpret_cast<const ulonglong2*>(keys + t));
            } else {
                ss[j] = 0;
            }
        }
        unsigned n = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool a = (ss[j] & 0xFF) == kValid && !is_guard(kk[j].x);
            const bool b = (ss[j] >> 8) == kValid && !is_guard(kk[j].y);
            const unsigned ma = __ballot_sync(FULL, a), mb = __ballot_sync(FULL, b);
            if (a) q[n + __popc(ma & below)] = kk[j].x;
            n += __popc(ma);
            if (b) q[n + __popc(mb & below)] = kk[j].y;
            n += __popc(mb);
        }
        __syncwarp();
        for (unsigned i = lane; i < n; i += 32) f(q[i]);
        __syncwarp();
    }
}

// out-degree: Valid non-guard slots per row.  Rows are contiguous slot runs,
// so lanes holding the same source (match_any) add their count once — one
// atomic per source per 32 slots, never one per edge of a hub row.
static __global__ void __launch_bounds__(256) k_outdeg(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                       u32* __restrict__ outdeg) {
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 base = warp * 256; base < cap; base += nwarps * 256) {
        ulonglong2 kk[4];
        unsigned short ss[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u64 t = base + 64 * q + 2 * lane;
            if (t < cap) {
                ss[q] = __ldcs(reinterpret_cast<const unsigned short*>(st + t));
                kk[q] = __ldcs(reinterpret_cast<const ulonglong2*>(keys + t));
            } else {
                ss[q] = 0;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool e0 = (ss[q] & 0xFF) == kValid && !is_guard(kk[q].x);
            const bool e1 = (ss[q] >> 8) == kValid && !is_guard(kk[q].y);
            const u32 s0 = e0 ? src_of(kk[q].x) : 0xFFFFFFFFu, s1 = e1 ? src_of(kk[q].y) : 0xFFFFFFFFu;
            // the lane's own pair first: one source (the common case) counts 2
            const u32 mine = e0 ? s0 : s1;
            const u32 c = (e0 && e1 && s0 == s1) ? 2u : ((e0 || e1) ? 1u : 0u);
            const u32 rest = (e0 && e1 && s0 != s1) ? s1 : 0xFFFFFFFFu;  // a row boundary inside the pair
            const unsigned grp = __match_any_sync(FULL, c ? mine : 0xFFFFFFFFu);
            const u32 tot = __reduce_add_sync(grp, c);
            if (c && lane == unsigned(__ffs(grp) - 1)) atomicAdd(&outdeg[mine], tot);
            const unsigned g2 = __match_any_sync(FULL, rest);
            if (rest != 0xFFFFFFFFu && lane == unsigned(__ffs(g2) - 1)) atomicAdd(&outdeg[rest], u32(__popc(g2)));
        }
    }
}

// push sweep over the gapped array: src comes from the key, so no row
// offsets are read; red.global.add.f64 into y (L2-resident for |V| <= ~16M).
// Hot destinations (power-law hubs) would serialise thousands of
// red.global.add.f64 on one address; each CTA accumulates them in shared
// memory instead and flushes one atomic per touched hub.  The hot set = the
// vertices of largest out-degree (<= kHotMax, picked once per PageRank call
// by k_hot_hist/k_hot_select — a performance heuristic only: every edge lands
// in exactly one of the two accumulators), looked up through an
// open-addressing table of kHotTable slots staged in smem.
constexpr u32 kHotMax = 1024;
constexpr u32 kHotTable = 2048;  // power of two, >= 2 kHotMax
constexpr u32 kHotEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ u32 hot_hash(u32 v) { return (v * 2654435761u) >> 21; }  // 11 bits = kHotTable

static __global__ void k_hot_hist(const u32* __restrict__ outdeg, u64 n, u32* __restrict__ hist) {
    __shared__ u32 s_h[33];
    if (threadIdx.x < 33) s_h[threadIdx.x] = 0;
    __syncthreads();
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x) {
        const u32 od = outdeg[u];
        if (od) atomicAdd(&s_h[32 - __clz(od)], 1u);  // bucket = bit length
    }
    __syncthreads();
    if (threadIdx.x < 33 && s_h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], s_h[threadIdx.x]);
}

// vertices with bit_length(outdeg) >= min_bits into the hash table (key = id, value = slot index)
static __global__ void k_hot_select(const u32* __restrict__ outdeg, u64 n, u32 min_bits, u32* __restrict__ table,
                                    u32* __restrict__ ids, u32* __restrict__ count) {
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x) {
        const u32 od = outdeg[u];
        if (!od || u32(32 - __clz(od)) < min_bits) continue;
        const u32 i = atomicAdd(count, 1u);
        if (i >= kHotMax) continue;
        ids[i] = u32(u);
        for (u32 h = hot_hash(u32(u));; h = (h + 1) & (kHotTable - 1)) {
            if (atomicCAS(&table[2 * h], kHotEmpty, u32(u)) == kHotEmpty) {
                table[2 * h + 1] = i;
                break;
            }
        }
    }
}

// push sweep over the gapped array: src comes from the key, so no row
// offsets are read; red.global.add.f64 into y (L2-resident for |V| <= ~16M),
// hot destinations through the CTA's shared accumulators.
static __global__ void __launch_bounds__(256) k_pr_push(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                        const double* __restrict__ share, double* __restrict__ y,
                                                        const u32* __restrict__ hot_table, const u32* __restrict__ hot_ids,
                                                        u32 nhot, const u32* done = nullptr) {
    if (done && *done) return;  // converged earlier in this window of iterations
    __shared__ u32 s_tab[2 * kHotTable];
    __shared__ double s_acc[kHotMax];
    __shared__ u64 s_q[8 * 256];  // the block's 8 warp queues
    if (nhot) {
        for (u32 i = threadIdx.x; i < 2 * kHotTable; i += blockDim.x) s_tab[i] = hot_table[i];
        for (u32 i = threadIdx.x; i < nhot; i += blockDim.x) s_acc[i] = 0.0;
        __syncthreads();
    }
    sweep_edges8_packed(keys, st, cap, s_q, [&](u64 k) {
        const u32 v = dst_of(k);
        const double sh = __ldg(&share[src_of(k)]);
        if (nhot) {
            for (u32 h = hot_hash(v);; h = (h + 1) & (kHotTable - 1)) {
                const u32 key = s_tab[2 * h];
                if (key == v) {
                    atomicAdd(&s_acc[s_tab[2 * h + 1]], sh);
                    return;
                }
                if (key == kHotEmpty) break;
            }
        }
        atomicAdd(&y[v], sh);
    });
    if (nhot) {
        __syncthreads();
        for (u32 i = threadIdx.x; i < nhot; i += blockDim.x)
            if (s_acc[i] != 0.0) atomicAdd(&y[hot_ids[i]], s_acc[i]);
    }
}

// -------- SpMV (analytics.hpp:147-158): warp per row; products in parallel,
// accumulation serial in ascending slot order with explicit round-to-nearest
// multiply and add (no FMA contraction) — bit-exact with the reference.
static __global__ void __launch_bounds__(256) k_spmv(const u64* __restrict__ ro, u64 nv, const u64* __restrict__ keys,
                                              const u64* __restrict__ vals, const u8* __restrict__ st,
                                              const double* __restrict__ x, double* __restrict__ y) {
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 u = warp; u < nv; u += nwarps) {
        const u64 b = ro[u], e = ro[u + 1];
        double acc = 0.0;
        for (u64 t0 = b; t0 < e; t0 += 32) {
            const u64 t = t0 + lane;
            double prod = 0.0;
            bool ok = false;
            if (t < e && st[t] == kValid) {
                const u64 k = keys[t];
                if (!is_guard(k)) {
                    ok = true;
                    prod = __dmul_rn(__longlong_as_double((long long)vals[t]), x[dst_of(k)]);
                }
            }
            unsigned m = __ballot_sync(FULL, ok);
            while (m) {
                const int i = __ffs(m) - 1;
                acc = __dadd_rn(acc, __shfl_sync(FULL, prod, i));
                m &= m - 1;
            }
        }
        if (lane == 0) y[u] = acc;
    }
}


}  // namespace gpma
