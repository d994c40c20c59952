// radix.cuh — hand-written onesweep LSD radix sort of 64-bit keys (optional
// u32 payload) and a single-pass exclusive sum, the sort under every batch,
// bulk load and window build of the library.
//
// The reference's sort_by_key (primitives.hpp:21-56) is a stable LSD radix
// sort with 8-bit digits over the live key bits; this is the same algorithm
// restated for the GPU as a onesweep sort (Adinets & Merrill 2022):
//
//   1. k_radix_hist   — ONE read of the keys builds the 256-bin histogram of
//                       every digit pass at once (shared-memory bins, one
//                       global add per bin per CTA).
//   2. k_radix_pass   — per 8-bit digit: a CTA ranks a 4096-key tile (warp
//                       match_any over per-warp digit counters: stable by
//                       construction), publishes its per-digit counts, walks
//                       back over the earlier tiles' status words (decoupled
//                       look-back, one digit per thread) for its global digit
//                       offsets, reorders the tile by digit in shared memory
//                       and writes it out in digit runs (coalesced).
//   3. k_radix_small  — n <= 4096: every pass inside one CTA's shared memory,
//                       one launch (the small-batch latency path).
//
// Stability: within a warp, item i of lane l is element chunk + 32 i + l and
// ranks are taken in (i, l) order; warps own consecutive chunks and are
// combined in warp order; tiles in tile order.  So equal digits keep their
// input order in every pass, and the LSD composition is the stable sort the
// reference performs (equal keys keep arrival order: "last insert wins").
//
// Status words carry a launch epoch (as scan.cuh), so no memset runs between
// passes or calls; tile ids are block ids (in-order dispatch, as the
// single-pass scans assume).
#pragma once

#include <cstdlib>

#include "block_ops.cuh"
#include "scan.cuh"

namespace gpma {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixIpt = 16;
constexpr int kRadixTile = kRadixThreads * kRadixIpt;  // 4096 keys
constexpr int kRadixBins = 256;
constexpr int kRadixMaxPasses = 8;
constexpr u32 kNoDigit = 0x100u;  // past-the-end items of a partial tile

struct RadixWorkspace {
    DevBuf<ull> status;  // look-back mode: per pass launch, ntiles x 256 epoch-tagged words
    DevBuf<u32> hist;    // kRadixMaxPasses x 256 global digit counts
    DevBuf<u32> thist, toff;  // reduce-then-scan mode: 256 x ntiles digit counts / offsets
    ScanWorkspace scan;
    ull epoch = 0;
};

__device__ __forceinline__ u32 radix_digit(u64 k, int shift, u32 mask) { return u32(k >> shift) & mask; }

// Lanes holding the same 9-bit value d (8-bit digit or kNoDigit) as this
// lane: nine ballots, one per bit — a few cycles each, where match.any's cost
// grows with the number of distinct values in the warp (a random 8-bit digit
// has ~30 of them).
__device__ __forceinline__ unsigned warp_match9(u32 d) {
    unsigned peers = FULL;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(FULL, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

// Shared-memory layout of a rank/scatter tile (dynamic smem): the per-warp
// digit counters alias the key/value staging (they are dead by then).
template <bool kVals>
struct RadixSmem {
    static constexpr size_t kKeyBytes = size_t(kRadixTile) * 8;
    static constexpr size_t kValBytes = kVals ? size_t(kRadixTile) * 4 : 0;
    static constexpr size_t kStage = kKeyBytes + kValBytes;
    static constexpr size_t kWarpHist = size_t(kRadixWarps) * kRadixBins * 4;
    static constexpr size_t kUnion = kStage > kWarpHist ? kStage : kWarpHist;
    // + s_start[256] u32, s_gbase[256] u64, s_w[8] u32
    static constexpr size_t kBytes = kUnion + kRadixBins * 4 + kRadixBins * 8 + 64;
};

// Rank the thread's kRadixIpt items inside the tile: on return pos[i] is the
// tile-local destination of item i (digits ascending, input order inside a
// digit) and s_start[d] the tile-local start of digit d; *count (thread t =
// digit t) is the tile's count of digit t.  All threads call it.
// Item i of this thread is valid iff 32 i + lane < wvalid (the warp's valid
// items); its digit is recomputed from the key wherever needed, so only keys,
// payloads and positions occupy registers.
__device__ __forceinline__ u32 item_digit(const u64 (&k)[kRadixIpt], int i, u32 wvalid, int shift, u32 mask) {
    return (u32(i) * 32u + (threadIdx.x & 31u)) < wvalid ? radix_digit(k[i], shift, mask) : kNoDigit;
}

__device__ __forceinline__ void radix_rank_tile(const u64 (&k)[kRadixIpt], u32 wvalid, int shift, u32 mask,
                                                u32 (&pos)[kRadixIpt], u32* wh, u32* s_start, u32* s_w,
                                                u32* count) {
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    u32* h = wh + warp * kRadixBins;
#pragma unroll
    for (int j = 0; j < kRadixBins / 32; ++j) h[lane + 32 * j] = 0;
    __syncwarp();
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u32 d = item_digit(k, i, wvalid, shift, mask);
        const unsigned peers = warp_match9(d);
        const int leader = __ffs(peers) - 1;
        // the group's leader claims popc(peers) slots of digit d; shared
        // atomics of one warp retire in program order, so item row i gets
        // lower slots than row i + 1 (stability)
        u32 c = 0;
        if (int(lane) == leader && d < kNoDigit) c = atomicAdd(&h[d], u32(__popc(peers)));
        c = __shfl_sync(FULL, c, leader);
        pos[i] = c + __popc(peers & lt);
    }
    __syncwarp();
    __syncthreads();
    // thread t = digit t: exclusive over warps (warp order = input order)
    const unsigned t = threadIdx.x;
    u32 run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
        const u32 c = wh[w * kRadixBins + t];
        wh[w * kRadixBins + t] = run;
        run += c;
    }
    *count = run;
    u32 total;
    s_start[t] = block_excl_scan(run, &total, s_w);
    __syncthreads();  // every digit's start visible before the positions read them
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u32 d = item_digit(k, i, wvalid, shift, mask);
        if (d < kNoDigit) pos[i] += s_start[d] + wh[warp * kRadixBins + d];
    }
    __syncthreads();  // wh is dead from here: the staging area may be written
}

// One read of the keys -> the 256-bin histogram of every pass.
static __global__ void __launch_bounds__(256) k_radix_hist(const u64* __restrict__ keys, u64 n, int begin, int end,
                                                    u32* __restrict__ hist) {
    __shared__ u32 sh[kRadixMaxPasses * kRadixBins];
    pdl_enter();
    const int npass = (end - begin + 7) / 8;
    for (int i = threadIdx.x; i < npass * kRadixBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const u64 stride = u64(gridDim.x) * blockDim.x * 2;
    for (u64 i = (u64(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
        u64 k0 = 0, k1 = 0;
        bool two = i + 1 < n;
        if (two && ((reinterpret_cast<uintptr_t>(keys + i) & 15) == 0)) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(keys + i);
            k0 = v.x;
            k1 = v.y;
        } else {
            k0 = keys[i];
            if (two) k1 = keys[i + 1];
        }
        for (int p = 0; p < npass; ++p) {
            const int sh_ = begin + 8 * p;
            const int bits = min(8, end - sh_);
            const u32 m = (1u << bits) - 1u;
            atomicAdd(&sh[p * kRadixBins + radix_digit(k0, sh_, m)], 1u);
            if (two) atomicAdd(&sh[p * kRadixBins + radix_digit(k1, sh_, m)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * kRadixBins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Reduce-then-scan form of a digit pass, step 1: every tile's count of every
// digit, digit-major (tile_hist[d * ntiles + tile]), so one exclusive scan
// gives each (digit, tile) its global output offset — no look-back chains
// (whose first wave walks back across every resident tile).  Per-warp
// counters with match_any aggregation (skewed digits would serialise plain
// shared atomics).
static __global__ void __launch_bounds__(kRadixThreads) k_radix_upsweep(const u64* __restrict__ kin, u64 n, int shift,
                                                                 u32 mask, const u32* __restrict__ ghist,
                                                                 u32* __restrict__ tile_hist) {
    __shared__ u32 wh[kRadixWarps][kRadixBins];
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, t = threadIdx.x;
    if (__syncthreads_or(ghist[t] == n)) return;  // constant digit: the pass copies through
#pragma unroll
    for (int j = 0; j < kRadixBins / 32; ++j) wh[warp][lane + 32 * j] = 0;
    __syncwarp();
    const u64 base = u64(blockIdx.x) * kRadixTile;
    u64 k[kRadixIpt];
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u64 idx = base + u64(i) * kRadixThreads + t;
        k[i] = idx < n ? __ldcs(reinterpret_cast<const unsigned long long*>(kin + idx)) : 0;
    }
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u64 idx = base + u64(i) * kRadixThreads + t;
        const u32 d = idx < n ? radix_digit(k[i], shift, mask) : kNoDigit;
        const unsigned peers = warp_match9(d);
        if (d < kNoDigit && (peers & lanemask_lt()) == 0) atomicAdd(&wh[warp][d], u32(__popc(peers)));
    }
    __syncthreads();
    u32 c = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) c += wh[w][t];
    tile_hist[u64(t) * gridDim.x + blockIdx.x] = c;
}

// One digit pass over the whole array (a tile per CTA, tile id = block id).
template <bool kVals>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_radix_pass(const u64* __restrict__ kin, u64* __restrict__ kout, const u32* __restrict__ vin,
                 u32* __restrict__ vout, u64 n, int shift, u32 mask, const u32* __restrict__ ghist, ull* status,
                 ull epoch, const u32* __restrict__ tile_off) {
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_enter();
    using S = RadixSmem<kVals>;
    u64* sk = reinterpret_cast<u64*>(smem);
    u32* sv = reinterpret_cast<u32*>(smem + S::kKeyBytes);
    u32* wh = reinterpret_cast<u32*>(smem);
    u32* s_start = reinterpret_cast<u32*>(smem + S::kUnion);
    u64* s_gbase = reinterpret_cast<u64*>(smem + S::kUnion + kRadixBins * 4);
    u32* s_w = reinterpret_cast<u32*>(smem + S::kUnion + kRadixBins * 12);

    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, t = threadIdx.x;
    const u64 tile = blockIdx.x;
    const u64 base = tile * kRadixTile;
    // a digit every key shares leaves the order unchanged: the reference skips
    // the pass (primitives.hpp:38-46); here the tile is copied through so the
    // ping-pong parity the host planned stays fixed
    if (__syncthreads_or(ghist[t] == n)) {
        for (u64 i = base + t; i < n && i < base + kRadixTile; i += kRadixThreads) {
            kout[i] = __ldcs(reinterpret_cast<const unsigned long long*>(kin + i));
            if (kVals) vout[i] = __ldcs(vin + i);
        }
        return;
    }
    const u64 chunk = base + u64(warp) * (32 * kRadixIpt);
    u64 k[kRadixIpt];
    u32 v[kRadixIpt];
    u32 pos[kRadixIpt];
    const u32 wvalid = chunk >= n ? 0u : u32(min(n - chunk, u64(32 * kRadixIpt)));
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u64 idx = chunk + u64(i) * 32 + lane;
        if (idx < n) {
            k[i] = __ldcs(reinterpret_cast<const unsigned long long*>(kin + idx));
            if (kVals) v[i] = __ldcs(vin + idx);
        } else {
            k[i] = 0;
            v[i] = 0;
        }
    }
    u32 count;
    radix_rank_tile(k, wvalid, shift, mask, pos, wh, s_start, s_w, &count);

    // publish this tile's count of digit t, then look back for the counts of
    // digit t in all earlier tiles (look-back mode; with tile_off the digit
    // offsets of every tile were scanned beforehand)
    const ull ep = (epoch & kEpochMask) << kEpochShift;
    ull* my = status + tile * kRadixBins + t;
    if (!tile_off) {
        if (tile == 0) st_volatile(my, ep | (2ull << kFlagShift) | count);
        else st_volatile(my, ep | (1ull << kFlagShift) | count);
    }
    // stage the tile in digit order while earlier tiles finish
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        if (u32(i) * 32u + lane < wvalid) {
            sk[pos[i]] = k[i];
            if (kVals) sv[pos[i]] = v[i];
        }
    }
    ull excl = 0;
    if (tile > 0 && !tile_off) {
        // walk back kLook tiles per step with the loads of a step in flight
        // together (a serial walk costs one L2 round trip per tile, and the
        // first wave of tiles has no inclusive predecessor nearby)
        constexpr int kLook = 32;
        const ull inclusive0 = ep | (2ull << kFlagShift);  // "tile -1": inclusive prefix 0
        auto ready = [&](ull w) { return (w & ~((1ull << kEpochShift) - 1)) == ep && ((w >> kFlagShift) & 3ull); };
        long long j = (long long)tile - 1;
        bool found = false;
        while (!found) {
            ull w[kLook];
#pragma unroll
            for (int q = 0; q < kLook; ++q)
                w[q] = j - q >= 0 ? ld_volatile(status + u64(j - q) * kRadixBins + t) : inclusive0;
#pragma unroll
            for (int q = 0; q < kLook; ++q) {
                if (found) continue;
                while (!ready(w[q])) w[q] = ld_volatile(status + u64(j - q) * kRadixBins + t);
                excl += w[q] & kValueMask;
                found = ((w[q] >> kFlagShift) & 3ull) == 2;
            }
            j -= kLook;
        }
        st_volatile(my, ep | (2ull << kFlagShift) | (excl + count));
    }
    // global start of digit t = digits below t over the whole array + digit t
    // in earlier tiles; minus the tile-local start so out = gbase[d] + j
    if (tile_off) {
        s_gbase[t] = u64(tile_off[u64(t) * gridDim.x + tile]) - s_start[t];
    } else {
        u32 gtot;
        const u32 gex = block_excl_scan(ghist[t], &gtot, s_w);
        s_gbase[t] = u64(gex) + excl - s_start[t];
    }
    __syncthreads();
    const u64 nv = n - base < u64(kRadixTile) ? n - base : u64(kRadixTile);
#pragma unroll 4
    for (int i = 0; i < kRadixIpt; ++i) {
        const u32 j = t + u32(i) * kRadixThreads;
        if (j < nv) {
            const u64 key = sk[j];
            const u64 o = s_gbase[radix_digit(key, shift, mask)] + j;
            __stcs(reinterpret_cast<unsigned long long*>(kout + o), key);
            if (kVals) __stcs(vout + o, sv[j]);
        }
    }
}

// n <= kRadixTile: all passes inside one CTA (one launch).
template <bool kVals>
__global__ void __launch_bounds__(kRadixThreads, 1)
    k_radix_small(const u64* __restrict__ kin, u64* __restrict__ kout, const u32* __restrict__ vin,
                  u32* __restrict__ vout, u32 n, const ull* n_dev, int begin, int end) {
    if (n_dev) n = u32(*n_dev);  // device-resident count (graph-captured small batches)
    extern __shared__ __align__(16) unsigned char smem[];
    using S = RadixSmem<kVals>;
    u64* sk = reinterpret_cast<u64*>(smem);
    u32* sv = reinterpret_cast<u32*>(smem + S::kKeyBytes);
    u32* wh = reinterpret_cast<u32*>(smem);
    u32* s_start = reinterpret_cast<u32*>(smem + S::kUnion);
    u32* s_w = reinterpret_cast<u32*>(smem + S::kUnion + kRadixBins * 12);
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const u32 chunk = warp * (32 * kRadixIpt);
    u64 k[kRadixIpt];
    u32 v[kRadixIpt];
    u32 pos[kRadixIpt];
    const u32 wvalid = chunk >= n ? 0u : min(n - chunk, u32(32 * kRadixIpt));
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u32 idx = chunk + u32(i) * 32 + lane;
        k[i] = idx < n ? kin[idx] : 0;
        v[i] = (kVals && idx < n) ? vin[idx] : 0;
    }
    for (int sh_ = begin; sh_ < end; sh_ += 8) {
        const u32 m = (1u << min(8, end - sh_)) - 1u;
        u32 count;
        radix_rank_tile(k, wvalid, sh_, m, pos, wh, s_start, s_w, &count);
#pragma unroll
        for (int i = 0; i < kRadixIpt; ++i) {
            if (u32(i) * 32u + lane < wvalid) {
                sk[pos[i]] = k[i];
                if (kVals) sv[pos[i]] = v[i];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kRadixIpt; ++i) {
            const u32 idx = chunk + u32(i) * 32 + lane;
            if (idx < n) {
                k[i] = sk[idx];
                if (kVals) v[i] = sv[idx];
            }
        }
        __syncthreads();  // the next pass's counters alias the staging area
    }
#pragma unroll
    for (int i = 0; i < kRadixIpt; ++i) {
        const u32 idx = chunk + u32(i) * 32 + lane;
        if (idx < n) {
            kout[idx] = k[i];
            if (kVals) vout[idx] = v[i];
        }
    }
}

// ---- single-pass exclusive sum (decoupled look-back) ----------------------
// out[i] = sum of in[0..i) for n values (u32 in, u32 out; totals must fit).
// A tile is 256 threads x 8 consecutive values; warp 0 runs the look-back
// over epoch-tagged tile words exactly as compact_kernel does.
constexpr int kSumItems = 16;  // 4096-word tiles: half the look-back chain of 2048 (measured on 4M counters)
constexpr int kSumTile = kScanThreads * kSumItems;

static __global__ void __launch_bounds__(kScanThreads) k_exclusive_sum(const u32* __restrict__ in, u32* __restrict__ out,
                                                                u64 n, ull* tiles, ull epoch, u32* clear) {
    pdl_enter();
    __shared__ u32 s_w[kScanWarps];
    __shared__ ull s_prefix;
    const u64 tile = blockIdx.x;
    const u64 i0 = tile * kSumTile + u64(threadIdx.x) * kSumItems;
    u32 x[kSumItems];
    static_assert(kSumItems % 4 == 0, "vector loads of 4 words");
    if (i0 + kSumItems <= n && ((reinterpret_cast<uintptr_t>(in + i0) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < kSumItems / 4; ++q) {
            const uint4 a = *reinterpret_cast<const uint4*>(in + i0 + 4 * q);
            x[4 * q] = a.x, x[4 * q + 1] = a.y, x[4 * q + 2] = a.z, x[4 * q + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kSumItems; ++j) x[j] = i0 + j < n ? in[i0 + j] : 0u;
    }
    if (clear) {  // the counters read here are zeroed for their next use (no separate memset)
        if (i0 + kSumItems <= n && ((reinterpret_cast<uintptr_t>(clear + i0) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < kSumItems / 4; ++q) *reinterpret_cast<uint4*>(clear + i0 + 4 * q) = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll
            for (int j = 0; j < kSumItems; ++j)
                if (i0 + j < n) clear[i0 + j] = 0;
        }
    }
    u32 sum = 0;
#pragma unroll
    for (int j = 0; j < kSumItems; ++j) sum += x[j];
    u32 total;
    const u32 ex = block_excl_scan(sum, &total, s_w);
    if (threadIdx.x < 32) {
        const unsigned lane = threadIdx.x;
        const ull ep = (epoch & kEpochMask) << kEpochShift;
        ull prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile(&tiles[0], ep | (2ull << kFlagShift) | total);
        } else {
            if (lane == 0) st_volatile(&tiles[tile], ep | (1ull << kFlagShift) | total);
            long long t = (long long)tile - 1 - lane;
            for (;;) {
                ull st = t >= 0 ? ld_volatile(&tiles[t]) : (ep | (2ull << kFlagShift));
                auto ready = [&](ull w) {
                    return (w & ~((1ull << kEpochShift) - 1)) == ep && ((w >> kFlagShift) & 3ull);
                };
                while (__any_sync(FULL, !ready(st))) {
                    if (!ready(st)) st = ld_volatile(&tiles[t]);
                }
                const unsigned incl = __ballot_sync(FULL, ((st >> kFlagShift) & 3ull) == 2);
                const int first = incl ? __ffs(incl) - 1 : 32;
                ull v = (int(lane) <= first) ? (st & kValueMask) : 0;
#pragma unroll
                for (int dd = 16; dd > 0; dd >>= 1) v += __shfl_xor_sync(FULL, v, dd);
                prefix += v;
                if (incl) break;
                t -= 32;
            }
            if (lane == 0) st_volatile(&tiles[tile], ep | (2ull << kFlagShift) | (prefix + total));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    u32 run = u32(s_prefix) + ex;
    u32 y[kSumItems];
#pragma unroll
    for (int j = 0; j < kSumItems; ++j) {
        y[j] = run;
        run += x[j];
    }
    if (i0 + kSumItems <= n && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < kSumItems / 4; ++q)
            *reinterpret_cast<uint4*>(out + i0 + 4 * q) = make_uint4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < kSumItems; ++j)
            if (i0 + j < n) out[i0 + j] = y[j];
    }
}

// clear (optional) = in: the input counters are left zeroed
inline void exclusive_sum(cudaStream_t s, ScanWorkspace& ws, const u32* in, u32* out, u64 n, u32* clear = nullptr) {
    if (n == 0) return;
    const u64 ntiles = (n + kSumTile - 1) / kSumTile;
    if (ntiles > ws.tiles.cap) {
        ws.tiles.reserve(ntiles);
        GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ws.tiles.cap * sizeof(ull), s));
    }
    ws.epoch = (ws.epoch + 1) & kEpochMask;
    if (ws.epoch == 0) {
        GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ws.tiles.cap * sizeof(ull), s));
        ws.epoch = 1;
    }
    launch_k(k_exclusive_sum, dim3(unsigned(ntiles)), dim3(kScanThreads), 0, s, in, out, n, ws.tiles.ptr, ws.epoch,
             clear);
}

// Dynamic shared memory beyond 48 KB for the rank/scatter kernels, once per
// device (the attribute is per function and device).
inline void radix_prepare() {
    static unsigned long long attr_set = 0;
    int dev = 0;
    GPMA_CUDA(cudaGetDevice(&dev));
    if ((attr_set >> (dev & 63)) & 1ull) return;
    GPMA_CUDA(cudaFuncSetAttribute(k_radix_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(RadixSmem<true>::kBytes)));
    GPMA_CUDA(cudaFuncSetAttribute(k_radix_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(RadixSmem<false>::kBytes)));
    GPMA_CUDA(cudaFuncSetAttribute(k_radix_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(RadixSmem<true>::kBytes)));
    GPMA_CUDA(cudaFuncSetAttribute(k_radix_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(RadixSmem<false>::kBytes)));
    attr_set |= 1ull << (dev & 63);
}

// Stable sort of n keys (+ payload when v0 != nullptr) by key bits
// [begin, end).  Double-buffer contract: the input is in k0/v0, k1/v1 are the
// alternate buffers (both may be overwritten); returns 1 when the result is
// in k1/v1, 0 when in k0/v0.  *launches (optional) counts kernel launches.
inline int radix_sort(cudaStream_t s, RadixWorkspace& ws, u64* k0, u64* k1, u32* v0, u32* v1, u64 n, int begin,
                      int end, u64* launches = nullptr) {
    if (n <= 1 || end <= begin) return 0;
    const bool vals = v0 != nullptr;
    const int npass = (end - begin + 7) / 8;
    if (npass > kRadixMaxPasses) throw ApiError(PMA_EINVAL, "radix_sort: more than 64 key bits");
    radix_prepare();
    if (n <= u64(kRadixTile)) {
        if (vals)
            k_radix_small<true><<<1, kRadixThreads, RadixSmem<true>::kBytes, s>>>(k0, k1, v0, v1, u32(n), nullptr, begin,
                                                                                  end);
        else
            k_radix_small<false><<<1, kRadixThreads, RadixSmem<false>::kBytes, s>>>(k0, k1, nullptr, nullptr, u32(n),
                                                                                   nullptr, begin, end);
        GPMA_LAUNCH_CHECK();
        if (launches) *launches += 1;
        return 1;
    }
    const u64 ntiles = (n + kRadixTile - 1) / kRadixTile;
    if (ntiles > 0x7fffffffull) throw ApiError(PMA_EINVAL, "radix_sort: too many keys");
    if (ntiles * kRadixBins > ws.status.cap) {
        ws.status.reserve(ntiles * kRadixBins);
        GPMA_CUDA(cudaMemsetAsync(ws.status.ptr, 0, ws.status.cap * sizeof(ull), s));  // epoch 0 never issued
    }
    ws.hist.reserve(kRadixMaxPasses * kRadixBins);
    // decoupled look-back (default) or reduce-then-scan (GPMA_RADIX_SCAN=1):
    // measured on 2M-16M keys, the look-back form is 20-25% faster
    static const bool lookback = [] {
        const char* e = std::getenv("GPMA_RADIX_SCAN");
        return !(e && e[0] == '1');
    }();
    if (!lookback) {
        ws.thist.reserve(ntiles * kRadixBins);
        ws.toff.reserve(ntiles * kRadixBins);
    }
    GPMA_CUDA(cudaMemsetAsync(ws.hist.ptr, 0, size_t(npass) * kRadixBins * sizeof(u32), s));
    static const unsigned hist_grid = resident_grid(k_radix_hist, 256);
    const unsigned hg = unsigned(std::min<u64>(hist_grid, (n + 511) / 512));
    launch_k(k_radix_hist, dim3(hg), dim3(256), 0, s, static_cast<const u64*>(k0), n, begin, end, ws.hist.ptr);
    u64* ki = k0;
    u64* ko = k1;
    u32* vi = v0;
    u32* vo = v1;
    for (int p = 0; p < npass; ++p) {
        ws.epoch = (ws.epoch + 1) & kEpochMask;
        if (ws.epoch == 0) {
            GPMA_CUDA(cudaMemsetAsync(ws.status.ptr, 0, ws.status.cap * sizeof(ull), s));
            ws.epoch = 1;
        }
        const int sh_ = begin + 8 * p;
        const u32 m = (1u << std::min(8, end - sh_)) - 1u;
        const u32* gh = ws.hist.ptr + p * kRadixBins;
        const u32* toff = nullptr;
        if (!lookback) {  // reduce-then-scan: per-tile digit counts -> offsets
            k_radix_upsweep<<<unsigned(ntiles), kRadixThreads, 0, s>>>(ki, n, sh_, m, gh, ws.thist.ptr);
            GPMA_LAUNCH_CHECK();
            exclusive_sum(s, ws.scan, ws.thist.ptr, ws.toff.ptr, ntiles * kRadixBins);
            toff = ws.toff.ptr;
        }
        if (vals)
            launch_k(k_radix_pass<true>, dim3(unsigned(ntiles)), dim3(kRadixThreads), RadixSmem<true>::kBytes, s,
                     static_cast<const u64*>(ki), ko, static_cast<const u32*>(vi), vo, n, sh_, m, gh, ws.status.ptr,
                     ws.epoch, toff);
        else
            launch_k(k_radix_pass<false>, dim3(unsigned(ntiles)), dim3(kRadixThreads), RadixSmem<false>::kBytes, s,
                     static_cast<const u64*>(ki), ko, static_cast<const u32*>(nullptr), static_cast<u32*>(nullptr), n,
                     sh_, m, gh, ws.status.ptr, ws.epoch, toff);
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    if (launches) *launches += 1 + npass * (lookback ? 1 : 3);
    return ki == k1 ? 1 : 0;
}

}  // namespace gpma
