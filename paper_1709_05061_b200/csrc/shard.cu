// shard.cu — key-range sharding of the GPMA+ store across GPUs.
//
// Keys are src << 32 | dst, so a source-vertex range [lo, hi) is a key
// range: one GPMA+ per GPU holds the edges of its sources plus their guards,
// segments never cross shards and every round / decision / rebalance is local.
// What crosses GPUs is (a) each batch's updates, routed to their owners by one
// variable-size all-to-all (the caller's NCCL), after the stable owner
// partition below, and (b) the per-level / per-iteration exchanges of the
// analytics.  This file holds the device side of both; the collectives run in
// the caller (torch.distributed over NCCL), between these synchronous calls.
#include "analytics_kernels.cuh"
#include "block_ops.cuh"
#include "graph_impl.cuh"

namespace gpma {

// ------------------------------------------------------------ routing
// Stable multi-way partition of a batch slice by owner rank (bounds[r] <=
// src < bounds[r+1]).  Tiles of kRouteTile elements: (1) per-tile owner
// histograms, (2) one CTA scans them owner-major into write offsets, (3) each
// tile ranks its elements per owner with warp ballots (arrival order kept) and
// scatters.  Inserts and deletes are partitioned as separate slices.
constexpr int kRouteThreads = 256;
constexpr int kRouteItems = 8;
constexpr int kRouteTile = kRouteThreads * kRouteItems;
constexpr int kMaxWorld = 64;

// One rank's share of a batch: inserts then deletes (graph.hpp:133-147).
struct RouteIn {
    const u32* is;
    const u32* id;
    const double* iw;
    u64 ni;
    const u32* ds;
    const u32* dd;
    u64 nd;
    u32 nv;  // |V| <= 2^31
    __device__ __forceinline__ u32 src(u64 i) const { return i < ni ? is[i] : ds[i - ni]; }
    // An insert naming a vertex >= |V| rejects the whole batch (check_ids,
    // graph.hpp:133-137, before any mutation): counted by the senders, the
    // caller rejects the batch on every rank before any shard applies.
    __device__ __forceinline__ bool bad_insert(u64 i) const { return i < ni && (is[i] >= nv || id[i] >= nv); }
    // EdgeKey on the wire; bit 63 marks a delete.  A delete whose source is
    // >= |V| can never match (graph.hpp:140-145 counts it missed).  Sources
    // in [|V|, 2^31) travel as they are (the last rank counts them missed);
    // a source in [2^31, 2^32) would alias (src - 2^31, dst) through the
    // delete bit, so it travels as source 2^31 - 1 with a destination no
    // graph holds (top bit set, >= |V|; a guard delete stays a guard delete:
    // dropped, counted missed, not in batch_size, graph.hpp:141-147).  Such
    // deletes differing only in their source's top bit or in the top bit of
    // their destination count as one missed delete.
    __device__ __forceinline__ u64 key(u64 i) const {
        if (i < ni) return pack_edge(is[i], id[i]);
        const u32 s_ = ds[i - ni], d_ = dd[i - ni];
        if (s_ >= 0x80000000u) {
            const u32 d2 = d_ == u32(kGuardDst) ? d_ : min(d_ | 0x80000000u, 0xFFFFFFFEu);
            return pack_edge(0x7FFFFFFFu, d2) | (1ull << 63);
        }
        return pack_edge(s_, d_) | (1ull << 63);
    }
};

__device__ __forceinline__ int owner_of(u32 s, const u32* __restrict__ b, int world) {
    int lo = 0, hi = world;  // last r with b[r] <= s (ids >= |V| go to the last rank)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b[mid] <= s) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_route_hist(RouteIn in, const u32* __restrict__ bounds, int world, u32* __restrict__ tile_counts,
                             u64* __restrict__ bad) {
    const u64 n = in.ni + in.nd;
    __shared__ u32 s_b[kMaxWorld + 1];
    __shared__ u32 s_c[kMaxWorld];
    for (int i = threadIdx.x; i <= world; i += blockDim.x) s_b[i] = bounds[i];
    for (int i = threadIdx.x; i < world; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    const u64 base = u64(blockIdx.x) * kRouteTile;
    unsigned nbad = 0;
    for (int j = 0; j < kRouteItems; ++j) {
        const u64 i = base + u64(j) * kRouteThreads + threadIdx.x;
        if (i < n) {
            atomicAdd(&s_c[owner_of(in.src(i), s_b, world)], 1u);
            nbad += in.bad_insert(i);
        }
    }
    if (__any_sync(FULL, nbad != 0)) {
        for (int d = 16; d > 0; d >>= 1) nbad += __shfl_xor_sync(FULL, nbad, d);
        if ((threadIdx.x & 31u) == 0 && nbad) atomicAdd(reinterpret_cast<ull*>(bad), ull(nbad));
    }
    __syncthreads();
    for (int r = threadIdx.x; r < world; r += blockDim.x) tile_counts[u64(r) * gridDim.x + blockIdx.x] = s_c[r];
}

// exclusive scan of tile_counts in (owner, tile) order -> tile_offsets; totals
__global__ void k_route_scan(const u32* __restrict__ tile_counts, u64 ntiles, int world, u64* __restrict__ tile_offsets,
                             u64* __restrict__ totals) {
    __shared__ u64 s_part[1024];
    const u64 m = ntiles * u64(world);
    const u64 per = (m + blockDim.x - 1) / blockDim.x;
    const u64 a = min(m, u64(threadIdx.x) * per), b = min(m, a + per);
    u64 sum = 0;
    for (u64 i = a; i < b; ++i) sum += tile_counts[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 run = 0;
        for (unsigned t = 0; t < blockDim.x; ++t) {
            const u64 v = s_part[t];
            s_part[t] = run;
            run += v;
        }
    }
    __syncthreads();
    u64 run = s_part[threadIdx.x];
    for (u64 i = a; i < b; ++i) {
        tile_offsets[i] = run;
        run += tile_counts[i];
    }
    __syncthreads();
    // owner r's updates = start of owner r + 1 - start of owner r (owner-major scan)
    for (int r = threadIdx.x; r < world; r += blockDim.x) {
        const u64 st = tile_offsets[u64(r) * ntiles];
        const u64 en = u64(r + 1) < u64(world) ? tile_offsets[u64(r + 1) * ntiles]
                                                : tile_offsets[m - 1] + tile_counts[m - 1];
        totals[r] = en - st;
    }
}

// Destinations: okeys/ow (owner-major, for an all-to-all), or — fused
// routing — straight into every owner's receive buffer (peer memory over
// NVLink / IPC): owner r's element lands at dst_keys[r][dst_off[r] + its rank
// among this sender's elements for r], i.e. the position an all-to-all in
// sender-rank order would give it.
struct RouteDst {
    u64* okeys;
    double* ow;
    u64* const* dst_keys;   // [world] receive buffers (device pointers), or null
    double* const* dst_w;   // [world] or null
    const u64* dst_off;     // [world] this sender's first slot in each receive buffer
};

__global__ void k_route_scatter(RouteIn in, const u32* __restrict__ bounds, int world,
                                const u64* __restrict__ tile_offsets, RouteDst dst) {
    u64* __restrict__ okeys = dst.okeys;
    double* __restrict__ ow = dst.ow;
    const u64 n = in.ni + in.nd;
    constexpr int kWarps = kRouteThreads / 32;
    __shared__ u32 s_b[kMaxWorld + 1];
    // (item row j, warp, owner) counts -> owner-local exclusive offsets; rows
    // then warps then lanes is element order inside the tile (striped items)
    __shared__ u32 s_wc[kRouteItems * kWarps * kMaxWorld];
    for (int i = threadIdx.x; i <= world; i += blockDim.x) s_b[i] = bounds[i];
    for (int i = threadIdx.x; i < kRouteItems * kWarps * world; i += blockDim.x) s_wc[i] = 0;
    __syncthreads();
    const unsigned warp = threadIdx.x >> 5;
    const u64 base = u64(blockIdx.x) * kRouteTile;
    int own[kRouteItems];
    unsigned rank[kRouteItems];
#pragma unroll
    for (int j = 0; j < kRouteItems; ++j) {
        const u64 i = base + u64(j) * kRouteThreads + threadIdx.x;
        own[j] = i < n ? owner_of(in.src(i), s_b, world) : -1;
        const unsigned peers = __match_any_sync(FULL, own[j]);
        rank[j] = __popc(peers & lanemask_lt());
        if (own[j] >= 0 && rank[j] == 0) s_wc[(j * kWarps + warp) * world + own[j]] = __popc(peers);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < world; r += blockDim.x) {
        u32 run = 0;
        for (int jw = 0; jw < kRouteItems * kWarps; ++jw) {
            const u32 c = s_wc[jw * world + r];
            s_wc[jw * world + r] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRouteItems; ++j) {
        if (own[j] < 0) continue;
        const u64 i = base + u64(j) * kRouteThreads + threadIdx.x;
        const u64 o = tile_offsets[u64(own[j]) * gridDim.x + blockIdx.x] + s_wc[(j * kWarps + warp) * world + own[j]] +
                      rank[j];
        const u64 key = in.key(i);  // EdgeKey (graph.hpp:27-37) + delete bit: one 8-B word on the wire
        const double wt = (i < in.ni && in.iw) ? in.iw[i] : 1.0;
        if (dst.dst_keys) {
            const u64 q = dst.dst_off[own[j]] + (o - tile_offsets[u64(own[j]) * gridDim.x]);
            dst.dst_keys[own[j]][q] = key;
            if (dst.dst_w) dst.dst_w[own[j]][q] = wt;
        } else {
            okeys[o] = key;
            if (ow) ow[o] = wt;
        }
    }
}

// ------------------------------------------------------- sharded analytics
// BFS (analytics.hpp:22-48) owner-computes: each level the owners of the
// frontier mark its out-neighbours in a |V|-byte flag array (global ids);
// the caller max-reduces the flags across shards; each owner then admits its
// unreached flagged vertices at depth + 1 as its next frontier.
__global__ void __launch_bounds__(256) k_shard_bfs_mark(const u32* __restrict__ frontier, u32 nf,
                                                        const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                        const u8* __restrict__ st, u8* __restrict__ flags) {
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 f = warp; f < nf; f += nwarps) {
        const u32 u = frontier[f];
        const u64 b = ro[u], e = ro[u + 1];
        for (u64 t = b + lane; t < e; t += 32) {
            if (st[t] != kValid) continue;
            const u64 k = keys[t];
            if (!is_guard(k)) flags[dst_of(k)] = 1;
        }
    }
}

__global__ void k_shard_bfs_update(const u8* __restrict__ flags, u64 lo, u64 nloc, u32* __restrict__ dist, u32 depth,
                                   u32* __restrict__ next, u32* __restrict__ next_n) {
    const unsigned lane = threadIdx.x & 31u;
    for (u64 i0 = blockIdx.x * u64(blockDim.x); i0 < nloc; i0 += u64(gridDim.x) * blockDim.x) {
        const u64 i = i0 + threadIdx.x;
        const bool win = i < nloc && flags[lo + i] && dist[i] == GPMA_UNREACHED;
        if (win) dist[i] = depth;
        const unsigned wm = __ballot_sync(FULL, win);
        if (wm) {
            u32 base = 0;
            if (lane == 0) base = atomicAdd(next_n, u32(__popc(wm)));
            base = __shfl_sync(FULL, base, 0);
            if (win) next[base + __popc(wm & lanemask_lt())] = u32(lo + i);
        }
    }
}

// CC (analytics.hpp:53-82) as min-label propagation over replicated labels:
// every owned edge hooks the larger label's root under the smaller label;
// the caller min-reduces the labels across shards; pointer jumping then makes
// every label a root.  At the fixpoint each label is its component's minimum
// id — the reference's labels.
__global__ void __launch_bounds__(256) k_shard_cc_hook(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                       u32* labels) {
    __shared__ u64 s_q[8 * 256];
    sweep_edges8_packed(keys, st, cap, s_q, [&](u64 k) {
        const u32 u = src_of(k), v = dst_of(k);
        const u32 a = labels[u], b = labels[v];
        if (a == b) return;
        const u32 hi = a > b ? a : b, lo = a > b ? b : a;
        atomicMin(&labels[hi], lo);
        atomicMin(&labels[u], lo);
        atomicMin(&labels[v], lo);
    });
}

__global__ void k_cc_jump(u32* labels, u64 n, const u32* __restrict__ prev, u32* changed) {
    u32 ch = 0;
    for (u64 v = blockIdx.x * u64(blockDim.x) + threadIdx.x; v < n; v += u64(gridDim.x) * blockDim.x) {
        u32 x = labels[v];
        while (labels[x] != x) x = labels[x];  // labels only decrease along a chain: terminates at a root
        labels[v] = x;
        ch |= x != prev[v];
    }
    if (__any_sync(FULL, ch) && (threadIdx.x & 31u) == 0) atomicOr(changed, 1u);
}

// PageRank (analytics.hpp:84-143): out-degrees of the owned rows; per
// iteration the owners push d x[u] / outdeg[u] over their edges into a
// zeroed |V| vector that the caller sum-reduces; the finish (base term from
// the dangling mass, L1 residual) then runs replicated on identical inputs.
__global__ void k_shard_pr_share(const double* __restrict__ x, const u32* __restrict__ outdeg, u64 lo, u64 hi,
                                 double d, double* __restrict__ share) {
    for (u64 u = lo + blockIdx.x * u64(blockDim.x) + threadIdx.x; u < hi; u += u64(gridDim.x) * blockDim.x) {
        const u32 od = outdeg[u];
        share[u] = od ? __ddiv_rn(__dmul_rn(d, x[u]), double(od)) : 0.0;
    }
}

__global__ void k_pr_dangling(const double* __restrict__ x, const u32* __restrict__ outdeg, u64 n, double* sum) {
    double acc = 0.0;
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x)
        if (outdeg[u] == 0) acc += x[u];
    block_atomic_add(acc, sum);
}

__global__ void k_pr_finish(const double* __restrict__ x, double* __restrict__ y, u64 n, const double* dangling,
                            double d, double* l1) {
    const double nn = double(n);
    const double base = __dadd_rn(__ddiv_rn(1.0 - d, nn), __ddiv_rn(__dmul_rn(d, *dangling), nn));
    double acc = 0.0;
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x) {
        const double v = __dadd_rn(base, y[u]);
        y[u] = v;
        acc += fabs(v - x[u]);
    }
    block_atomic_add(acc, l1);
}

// ================================================================ host side

void Graph::route_partition(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                            u64 nd, const u32* d_bounds, int world, u64* okeys, double* ow, u64* h_counts,
                            u64* d_counts) {
    if (world < 1 || world > kMaxWorld) throw ApiError(PMA_EINVAL, "route: world size must be in [1, 64]");
    if (nv > (1ull << 31)) throw ApiError(PMA_EINVAL, "route: vertex ids must be < 2^31 (bit 63 marks deletes)");
    cudaStream_t s = pma.stream();
    const RouteIn in{is, id, iw, ni, ds, dd, nd, u32(nv)};
    const u64 n = ni + nd;
    // counts: world owners + [world] = inserts naming a vertex >= |V|
    if (n == 0) {
        if (h_counts)
            for (int r = 0; r <= world; ++r) h_counts[r] = 0;
        if (d_counts) GPMA_CUDA(cudaMemsetAsync(d_counts, 0, (world + 1) * sizeof(u64), s));
        return;
    }
    const u64 ntiles = (n + kRouteTile - 1) / kRouteTile;
    rt_counts.reserve(ntiles * world);
    rt_offsets.reserve(ntiles * world);
    rt_totals.reserve(world + 1);
    u64* totals = d_counts ? d_counts : rt_totals.ptr;
    GPMA_CUDA(cudaMemsetAsync(totals + world, 0, sizeof(u64), s));
    k_route_hist<<<unsigned(ntiles), kRouteThreads, 0, s>>>(in, d_bounds, world, rt_counts.ptr, totals + world);
    GPMA_LAUNCH_CHECK();
    k_route_scan<<<1, 1024, 0, s>>>(rt_counts.ptr, ntiles, world, rt_offsets.ptr, totals);
    GPMA_LAUNCH_CHECK();
    if (okeys) {
        k_route_scatter<<<unsigned(ntiles), kRouteThreads, 0, s>>>(in, d_bounds, world, rt_offsets.ptr,
                                                                   RouteDst{okeys, ow, nullptr, nullptr, nullptr});
        GPMA_LAUNCH_CHECK();
    }
    rt_ntiles = ntiles;
    if (h_counts) {  // host counts: one round trip; device counts: stream-ordered, no sync
        GPMA_CUDA(cudaMemcpyAsync(h_counts, totals, (world + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
    }
}

// Fused routing, second half: after route_partition(..., okeys = nullptr)
// counted the same slice, scatter it straight into the owners' receive
// buffers (stream-ordered; the caller makes the owners wait for every sender).
void Graph::route_scatter_peer(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                               u64 nd, const u32* d_bounds, int world, u64* const* dst_keys, double* const* dst_w,
                               const u64* dst_off) {
    const u64 n = ni + nd;
    if (n == 0) return;
    const u64 ntiles = (n + kRouteTile - 1) / kRouteTile;
    if (ntiles != rt_ntiles) throw ApiError(PMA_ELOGIC, "route_scatter_peer: slice differs from the counted one");
    const RouteIn in{is, id, iw, ni, ds, dd, nd, u32(nv)};
    k_route_scatter<<<unsigned(ntiles), kRouteThreads, 0, pma.stream()>>>(
        in, d_bounds, world, rt_offsets.ptr, RouteDst{nullptr, nullptr, dst_keys, dst_w, dst_off});
    GPMA_LAUNCH_CHECK();
}

void Graph::shard_bfs_mark(const u32* frontier, u32 nf, u8* flags) {
    cudaStream_t s = pma.stream();
    GPMA_CUDA(cudaMemsetAsync(flags, 0, nv, s));
    if (nf) {
        k_shard_bfs_mark<<<grid_for(u64(nf) * 32, 256, 148 * 16), 256, 0, s>>>(frontier, nf, pma.ro_base(),
                                                                              pma.d_keys, pma.d_st, flags);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaStreamSynchronize(s));
}

void Graph::shard_bfs_update(const u8* flags, u32* dist_local, u32 depth, u32* next, u32* nf_out) {
    cudaStream_t s = pma.stream();
    qn.reserve(1);
    GPMA_CUDA(cudaMemsetAsync(qn.ptr, 0, 4, s));
    if (nloc()) {
        k_shard_bfs_update<<<grid_for(nloc(), 256, 148 * 16), 256, 0, s>>>(flags, lo, nloc(), dist_local, depth, next,
                                                                          qn.ptr);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaMemcpyAsync(h_nf_, qn.ptr, 4, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    *nf_out = *h_nf_;
}

void Graph::shard_cc_hook(u32* labels) {
    cudaStream_t s = pma.stream();
    const u64 cap = pma.capacity();
    k_shard_cc_hook<<<grid_for(cap / 8, 256, 148 * 16), 256, 0, s>>>(pma.d_keys, pma.d_st, cap, labels);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaStreamSynchronize(s));
}

void Graph::cc_jump(u32* labels, u64 n, const u32* prev, int* changed) {
    cudaStream_t s = pma.stream();
    qn.reserve(1);
    GPMA_CUDA(cudaMemsetAsync(qn.ptr, 0, 4, s));
    if (n) {
        k_cc_jump<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(labels, n, prev, qn.ptr);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaMemcpyAsync(h_nf_, qn.ptr, 4, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    *changed = *h_nf_ != 0;
}

void Graph::shard_outdeg(u32* outdeg) {
    cudaStream_t s = pma.stream();
    hot_ready_ = false;
    GPMA_CUDA(cudaMemsetAsync(outdeg, 0, nv * 4, s));
    const u64 cap = pma.capacity();
    k_outdeg<<<grid_for(cap / 8, 256, 148 * 16), 256, 0, s>>>(pma.d_keys, pma.d_st, cap, outdeg);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaStreamSynchronize(s));
}

void Graph::shard_pr_push(const double* x, const u32* outdeg, double d, double* y) {
    cudaStream_t s = pma.stream();
    pshare.reserve(nv + 1);
    GPMA_CUDA(cudaMemsetAsync(y, 0, nv * 8, s));
    if (nloc()) {
        k_shard_pr_share<<<grid_for(nloc(), 256, 148 * 8), 256, 0, s>>>(x, outdeg, lo, hi, d, pshare.ptr);
        GPMA_LAUNCH_CHECK();
    }
    const u64 cap = pma.capacity();
    if (!hot_ready_) {  // once per PageRank call (the out-degrees are global by now)
        prepare_hot(outdeg, nv);
        hot_ready_ = true;
    }
    k_pr_push<<<148 * 8, 256, 0, s>>>(pma.d_keys, pma.d_st, cap, pshare.ptr, y, hot_table.ptr, hot_ids.ptr, nhot_);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaStreamSynchronize(s));
}

void Graph::pr_finish(const double* x, double* y, u64 n, const u32* outdeg, double d, double* h_l1) {
    cudaStream_t s = pma.stream();
    psc.reserve(2);
    GPMA_CUDA(cudaMemsetAsync(psc.ptr, 0, 16, s));
    k_pr_dangling<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(x, outdeg, n, psc.ptr);
    GPMA_LAUNCH_CHECK();
    k_pr_finish<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(x, y, n, psc.ptr, d, psc.ptr + 1);
    GPMA_LAUNCH_CHECK();
    double l1 = 0.0;
    GPMA_CUDA(cudaMemcpyAsync(&l1, psc.ptr + 1, 8, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    *h_l1 = l1;
}

void Graph::shard_spmv(const double* x, double* y_local) {
    cudaStream_t s = pma.stream();
    if (nloc()) {
        k_spmv<<<grid_for(nloc() * 32, 256, 148 * 16), 256, 0, s>>>(ro.ptr, nloc(), pma.d_keys, pma.d_vals, pma.d_st,
                                                                    x, y_local);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gpma
