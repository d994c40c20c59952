// scan.cuh — single-pass ordered compaction / exclusive scan with decoupled
// look-back (Merrill & Garland), the primitive under every order-preserving
// step of the batch pipeline: duplicate resolution, per-round grouping
// (unique_segments = RLE + exclusive scan, segment_engine.hpp:78-86),
// advance_round (segment_engine.hpp:90-105) and the touched-range list.
//
// One pass: every element is read once by `flag(i)` and handed to
// `emit(i, f, exclusive_prefix)`.  A tile is 2048 elements, one CTA of 256
// threads, items STRIPED (item j of thread t is element base + 256 j + t) so
// every flag/emit access of a warp is one contiguous run; ranks come from warp
// ballots, the 8 x 8 (item row, warp) counts are scanned by one warp, and that
// warp runs the look-back.  Tile ids are block ids (blocks are dispatched in
// order, as CUB's single-pass scans assume), and tile status words carry a
// launch epoch, so no memset / ticket is needed between launches.
#pragma once

#include "common.cuh"

namespace gpma {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kScanTile = kScanThreads * kScanItems;
static_assert(kScanItems * kScanWarps == 64, "compact_kernel's warp-0 scan takes two (row, warp) counts per lane");
// status word: [63:36] epoch | [35:34] flag (1 aggregate, 2 inclusive) | [33:0] value
constexpr int kEpochShift = 36;
constexpr int kFlagShift = 34;
constexpr ull kValueMask = (1ull << kFlagShift) - 1;
constexpr ull kEpochMask = (1ull << (64 - kEpochShift)) - 1;

struct ScanWorkspace {
    DevBuf<ull> tiles;
    ull epoch = 0;
};

__device__ __forceinline__ ull ld_volatile(const ull* p) { return *reinterpret_cast<const volatile ull*>(p); }
__device__ __forceinline__ void st_volatile(ull* p, ull v) { *reinterpret_cast<volatile ull*>(p) = v; }

// emit_tile(i0, n, fm, x[]) handles the thread's kScanItems items i0 + 256 j
// (j < kScanItems, i < n) at once: bit j of fm = flag, x[j] = exclusive prefix.
// Lets a caller interleave independent per-item work (e.g. 8 binary searches).
template <class Flag, class EmitTile, class Fin>
__global__ void __launch_bounds__(kScanThreads, 7) compact_kernel(const ull* n_dev, ull n_host, Flag flag,
                                                               EmitTile emit_tile, Fin fin, ull* tiles, ull epoch,
                                                               ull* stamp) {
    __shared__ unsigned s_off[kScanItems * kScanWarps];  // (item row, warp) counts -> exclusive offsets
    __shared__ ull s_prefix, s_total;
    pdl_enter();
    stamp_first(stamp);
    const ull n = n_dev ? *n_dev : n_host;
    const ull ntiles = (n + kScanTile - 1) / kScanTile;
    const ull tile = blockIdx.x;
    if (tile >= ntiles) {
        if (ntiles == 0 && tile == 0 && threadIdx.x == 0) fin(0);  // empty input: fin(0) all the same
        return;
    }
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const ull base = tile * kScanTile + threadIdx.x;
    const unsigned below = lanemask_lt();
    unsigned fm = 0;
    unsigned char pre[kScanItems];
    bool fl[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {  // all flags first: their loads overlap
        const ull i = base + ull(j) * kScanThreads;
        fl[j] = i < n && flag(i);
    }
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const bool f = fl[j];
        const unsigned bal = __ballot_sync(FULL, f);
        pre[j] = (unsigned char)__popc(bal & below);
        if (lane == 0) s_off[j * kScanWarps + warp] = __popc(bal);
        fm |= (f ? 1u : 0u) << j;
    }
    __syncthreads();
    if (warp == 0) {
        // counts in element order: (row j, warp w) -> index j * 8 + w; two per lane
        const unsigned a0 = s_off[2 * lane], a1 = s_off[2 * lane + 1];
        const unsigned sum = a0 + a1;
        unsigned inc = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned o = __shfl_up_sync(FULL, inc, d);
            if (lane >= unsigned(d)) inc += o;
        }
        const unsigned ex = inc - sum;
        s_off[2 * lane] = ex;
        s_off[2 * lane + 1] = ex + a0;
        const ull total = __shfl_sync(FULL, inc, 31);
        const ull ep = (epoch & kEpochMask) << kEpochShift;
        ull prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile(&tiles[0], ep | (2ull << kFlagShift) | total);
        } else {
            if (lane == 0) st_volatile(&tiles[tile], ep | (1ull << kFlagShift) | total);
            long long t = (long long)tile - 1 - lane;
            for (;;) {
                ull st = t >= 0 ? ld_volatile(&tiles[t]) : (ep | (2ull << kFlagShift));
                auto ready = [&](ull x) { return (x & ~((1ull << kEpochShift) - 1)) == ep && ((x >> kFlagShift) & 3ull); };
                while (__any_sync(FULL, !ready(st))) {
                    if (!ready(st)) st = ld_volatile(&tiles[t]);
                }
                const unsigned incl_mask = __ballot_sync(FULL, ((st >> kFlagShift) & 3ull) == 2);
                const int first = incl_mask ? __ffs(incl_mask) - 1 : 32;
                ull v = (int(lane) <= first) ? (st & kValueMask) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
                prefix += v;
                if (incl_mask) break;
                t -= 32;
            }
            if (lane == 0) st_volatile(&tiles[tile], ep | (2ull << kFlagShift) | (prefix + total));
        }
        if (lane == 0) {
            s_prefix = prefix;
            s_total = total;
        }
    }
    __syncthreads();
    const ull pfx = s_prefix;
    ull xs[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) xs[j] = pfx + s_off[j * kScanWarps + warp] + pre[j];
    emit_tile(base, n, fm, xs);
    if (tile == ntiles - 1 && threadIdx.x == 0) fin(pfx + s_total);
}

// Launch helper: n is either device-resident (n_dev) or host-known (n_host);
// n_bound is a host-known upper bound used to size the workspace and grid.
// `fin(total)` runs exactly once, also for an empty input (n_bound > 0).
template <class Emit>
struct PerItemEmit {
    Emit emit;
    __device__ __forceinline__ void operator()(ull i0, ull n, unsigned fm, const ull* xs) const {
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const ull i = i0 + ull(j) * kScanThreads;
            if (i < n) emit(i, (fm >> j) & 1u, xs[j]);
        }
    }
};

template <class Flag, class EmitTile, class Fin>
void run_compact_tile(cudaStream_t s, ScanWorkspace& ws, const ull* n_dev, ull n_host, ull n_bound, Flag flag,
                      EmitTile emit_tile, Fin fin, ull* stamp = nullptr) {
    const ull ntiles = (n_bound + kScanTile - 1) / kScanTile;
    if (ntiles == 0) return;
    if (ntiles > ws.tiles.cap) {
        ws.tiles.reserve(ntiles);
        GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ws.tiles.cap * sizeof(ull), s));  // epoch 0 never issued
    }
    ws.epoch = (ws.epoch + 1) & kEpochMask;
    if (ws.epoch == 0) {  // wrapped: stale words could carry any epoch again
        GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ws.tiles.cap * sizeof(ull), s));
        ws.epoch = 1;
    }
    launch_k(compact_kernel<Flag, EmitTile, Fin>, dim3(unsigned(ntiles)), dim3(kScanThreads), 0, s, n_dev, n_host, flag,
             emit_tile, fin, ws.tiles.ptr, ws.epoch, stamp);
}

template <class Flag, class Emit, class Fin>
void run_compact(cudaStream_t s, ScanWorkspace& ws, const ull* n_dev, ull n_host, ull n_bound, Flag flag, Emit emit,
                 Fin fin, ull* stamp = nullptr) {
    run_compact_tile(s, ws, n_dev, n_host, n_bound, flag, PerItemEmit<Emit>{emit}, fin, stamp);
}

struct NoFin {
    __device__ void operator()(ull) const {}
};

}  // namespace gpma
