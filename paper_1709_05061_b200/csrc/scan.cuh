// scan.cuh — single-pass ordered compaction / exclusive scan with decoupled
// look-back (Merrill & Garland), the primitive under every order-preserving
// step of the batch pipeline: duplicate resolution, per-round grouping
// (unique_segments = RLE + exclusive scan, segment_engine.hpp:78-86),
// advance_round (segment_engine.hpp:90-105) and the touched-range list.
//
// One pass: every element is read once by `flag(i)` and handed to
// `emit(i, f, exclusive_prefix)`; tiles of 2048 elements are claimed in order
// through an atomic ticket so the look-back never waits on an unscheduled
// tile, and the grid is persistent (<= 4 CTAs per SM).
#pragma once

#include "common.cuh"

namespace gpma {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr ull kStatusShift = 62;
constexpr ull kValueMask = (1ull << kStatusShift) - 1;

struct ScanWorkspace {
    DevBuf<ull> tiles;
    DevBuf<unsigned> ticket;
};

__device__ __forceinline__ ull ld_volatile(const ull* p) { return *reinterpret_cast<const volatile ull*>(p); }
__device__ __forceinline__ void st_volatile(ull* p, ull v) { *reinterpret_cast<volatile ull*>(p) = v; }

template <class Flag, class Emit, class Fin>
__global__ void __launch_bounds__(kScanThreads) compact_kernel(const ull* n_dev, ull n_host, Flag flag, Emit emit,
                                                               Fin fin, ull* tiles, unsigned* ticket) {
    __shared__ unsigned s_tile;
    __shared__ ull s_warp[kScanThreads / 32];
    __shared__ ull s_prefix;
    const ull n = n_dev ? *n_dev : n_host;
    const ull ntiles = (n + kScanTile - 1) / kScanTile;
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const ull tile = s_tile;
        if (tile >= ntiles) break;
        const ull base = tile * kScanTile + ull(threadIdx.x) * kScanItems;
        unsigned f[kScanItems];
        unsigned cnt = 0;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const ull i = base + j;
            f[j] = i < n ? (flag(i) ? 1u : 0u) : 0u;
            cnt += f[j];
        }
        // block exclusive scan of per-thread counts
        unsigned inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= unsigned(d)) inc += o;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        ull warp_base = 0, block_total = 0;
#pragma unroll
        for (int w = 0; w < kScanThreads / 32; ++w) {
            if (w < int(warp)) warp_base += s_warp[w];
            block_total += s_warp[w];
        }
        const ull excl = warp_base + inc - cnt;
        // decoupled look-back by warp 0
        if (warp == 0) {
            ull prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_volatile(&tiles[0], (2ull << kStatusShift) | block_total);
            } else {
                if (lane == 0) st_volatile(&tiles[tile], (1ull << kStatusShift) | block_total);
                long long t = (long long)tile - 1 - lane;
                for (;;) {
                    ull st = t >= 0 ? ld_volatile(&tiles[t]) : (2ull << kStatusShift);
                    while (__any_sync(0xffffffffu, (st >> kStatusShift) == 0)) {
                        if ((st >> kStatusShift) == 0) st = ld_volatile(&tiles[t]);
                    }
                    const unsigned incl_mask = __ballot_sync(0xffffffffu, (st >> kStatusShift) == 2);
                    const int first = incl_mask ? __ffs(incl_mask) - 1 : 32;
                    ull v = (int(lane) <= first) ? (st & kValueMask) : 0;
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                    prefix += v;
                    if (incl_mask) break;
                    t -= 32;
                }
                if (lane == 0) st_volatile(&tiles[tile], (2ull << kStatusShift) | (prefix + block_total));
            }
            if (lane == 0) s_prefix = prefix;
        }
        __syncthreads();
        ull run = s_prefix + excl;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const ull i = base + j;
            if (i < n) emit(i, f[j], run);
            run += f[j];
        }
        if (tile == ntiles - 1 && threadIdx.x == 0) fin(s_prefix + block_total);
        __syncthreads();
    }
}

// Launch helper: n is either device-resident (n_dev) or host-known (n_host);
// n_bound is a host-known upper bound used to size the workspace and grid.
// If n can be 0 at run time, `fin` is not called (callers pre-set totals).
template <class Flag, class Emit, class Fin>
void run_compact(cudaStream_t s, ScanWorkspace& ws, const ull* n_dev, ull n_host, ull n_bound, Flag flag, Emit emit,
                 Fin fin) {
    const ull ntiles = (n_bound + kScanTile - 1) / kScanTile;
    if (ntiles == 0) return;
    ws.tiles.reserve(ntiles);
    ws.ticket.reserve(1);
    GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ntiles * sizeof(ull), s));
    GPMA_CUDA(cudaMemsetAsync(ws.ticket.ptr, 0, sizeof(unsigned), s));
    const unsigned grid = static_cast<unsigned>(ntiles < ull(kNumSMs) * 4 ? ntiles : ull(kNumSMs) * 4);
    compact_kernel<<<grid, kScanThreads, 0, s>>>(n_dev, n_host, flag, emit, fin, ws.tiles.ptr, ws.ticket.ptr);
    GPMA_LAUNCH_CHECK();
}

struct NoFin {
    __device__ void operator()(ull) const {}
};

}  // namespace gpma
