// block_ops.cuh — CTA-cooperative building blocks shared by the CTA/grid
// merge tier, the sequential single-key ops and the refresh kernels.
#pragma once

#include "common.cuh"

namespace gpma {



// Exclusive scan of one u32 per thread across the CTA.  All threads call it.
// s_w needs blockDim.x/32 entries.
__device__ __forceinline__ u32 block_excl_scan(u32 v, u32* total, u32* s_w) {
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u32 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 o = __shfl_up_sync(FULL, inc, d);
        if (lane >= unsigned(d)) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        u32 x = lane < nw ? s_w[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 o = __shfl_up_sync(FULL, x, d);
            if (lane >= unsigned(d)) x += o;
        }
        if (lane < nw) s_w[lane] = x;
    }
    __syncthreads();
    const u32 base = warp ? s_w[warp - 1] : 0;
    *total = s_w[nw - 1];
    __syncthreads();
    return base + inc - v;
}

__device__ __forceinline__ ull block_sum(ull v, ull* s_w) {
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    ull t = 0;
    for (unsigned w = 0; w < nw; ++w) t += s_w[w];
    __syncthreads();
    return t;
}

__device__ __forceinline__ u64 lower_bound_dev(const u64* a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ u64 upper_bound_u32(const u32* a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (u64(a[mid]) <= key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ u64 lower_bound_u32(const u32* a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (u64(a[mid]) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Leaf search over backward-filled headers == binary_search_leaf
// (pma.hpp:234-245): last leaf whose first non-Empty key <= key, else 0.
__device__ __forceinline__ u64 leaf_of_key(const u64* hdr, u64 L, const u8* st, u64 leaf, u64 key) {
    if (key != ~0ull) {
        u64 lo = 0, hi = L;
        while (lo < hi) {
            const u64 mid = (lo + hi) >> 1;
            if (__ldg(&hdr[mid]) <= key) lo = mid + 1;
            else hi = mid;
        }
        return lo ? lo - 1 : 0;
    }
    u64 lo = 0, hi = L;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (hdr[mid] < ~0ull) lo = mid + 1;
        else hi = mid;
    }
    if (lo < L) {
        for (u64 s = lo * leaf; s < (lo + 1) * leaf; ++s)
            if (st[s] != kEmpty) return lo;
    }
    return lo ? lo - 1 : 0;
}

// Block-wide sum of a per-thread double, one atomicAdd per CTA (same-address
// atomics serialise in L2, so per-warp atomics on one counter cost ~us each).
__device__ __forceinline__ void block_atomic_add(double v, double* dst) {
    __shared__ double s_part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const unsigned w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) s_part[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (unsigned i = 0; i < (blockDim.x >> 5); ++i) a += s_part[i];
        if (a != 0.0) atomicAdd(dst, a);
    }
    __syncthreads();
}

// N leaf searches at once (keys < 2^64-1; pma.hpp:234-289 through the
// backward-filled headers): uniform power-of-two descent (L = C/leaf is a
// power of two) to the last header <= key, else 0 — the same leaf as
// leaf_of_key — with the N searches interleaved so every level issues N
// independent loads instead of one dependent chain per key.
template <int N>
__device__ __forceinline__ void leaf_search_interleaved(const u64* __restrict__ hdr, u64 L, unsigned act,
                                                        const u64 (&key)[N], u64 (&pos)[N]) {
#pragma unroll
    for (int j = 0; j < N; ++j) pos[j] = 0;
    for (u64 s = L >> 1; s; s >>= 1) {
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (((act >> j) & 1u) && __ldg(&hdr[pos[j] + s]) <= key[j]) pos[j] += s;
    }
}

// Destination-driven even placement (pma.hpp:440-467): slot t of the
// segment holds entry j = ceil(t*k/m) iff floor(j*m/k) == t.
__device__ __forceinline__ bool placement_target(u64 t, u64 k, u64 m, u64* j_out) {
    if (k == 0) return false;
    const u64 j = (t * k + m - 1) / m;
    *j_out = j;
    return j < k && (j * m) / k == t;
}

}  // namespace gpma
