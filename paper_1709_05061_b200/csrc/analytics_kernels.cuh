// analytics_kernels.cuh — sweeps over the gapped slot array shared by the
// whole-graph analytics (graph.cu) and the sharded ones (shard.cu); internal
// linkage, one copy per translation unit.
#pragma once

#include "block_ops.cuh"

namespace gpma {

// out-degree: Valid non-guard slots per row, warp-segmented by source.
static __global__ void k_outdeg(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap, u32* __restrict__ outdeg) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 t0 = (blockIdx.x * u64(blockDim.x) + threadIdx.x) & ~31ull; t0 < cap; t0 += stride) {
        const u64 t = t0 + (threadIdx.x & 31u);
        bool e = false;
        u32 s = 0xFFFFFFFFu;
        if (t < cap && st[t] == kValid) {
            const u64 k = keys[t];
            e = !is_guard(k);
            s = src_of(k);
        }
        const unsigned grp = __match_any_sync(FULL, e ? s : 0xFFFFFFFFu);
        const unsigned leader = __ffs(grp) - 1;
        if (e && (threadIdx.x & 31u) == leader) atomicAdd(&outdeg[s], u32(__popc(grp)));
    }
}

// push sweep over the gapped array: src comes from the key, so no row
// offsets are read; red.global.add.f64 into y (L2-resident for |V| <= ~16M).
static __global__ void __launch_bounds__(256) k_pr_push(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                 const double* __restrict__ share, double* __restrict__ y) {
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < cap; t += u64(gridDim.x) * blockDim.x) {
        if (st[t] != kValid) continue;
        const u64 k = keys[t];
        if (is_guard(k)) continue;
        atomicAdd(&y[dst_of(k)], share[src_of(k)]);
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
