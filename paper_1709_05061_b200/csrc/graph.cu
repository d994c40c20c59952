// graph.cu — DynamicGraph on the device PMA (graph.hpp:62-240) and the
// analytics kernels over the gapped slot array (analytics.hpp:17-158).
//
// Row u of the graph is the slot interval [ro[u], ro[u+1]) of the PMA:
// Valid non-guard slots are its edges in ascending destination order, the
// interval also holds gaps, tombstones and the row's guard (graph.hpp:100-114).
// The analytics read keys+states (9 B/slot) and, for SpMV, values (17 B/slot).

#include <cmath>
#include <cstring>

#include "block_ops.cuh"
#include "analytics_kernels.cuh"
#include "graph_impl.cuh"

namespace gpma {

// ---------------------------------------------------------------- kernels

__global__ void k_check_ids(const u32* src, const u32* dst, u64 n, u64 nv, Ctr* ctr) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        if (src[i] >= nv || dst[i] >= nv) atomicMin(&ctr->bad_index, ull(i));
}

// Shard build: edges whose source lies outside the owned range [lo, hi) get
// key 2^64-1 (sorted last, dropped by the dedupe).
__global__ void k_pack_edges_shard(const u32* s, const u32* d, u64 n, u64 lo, u64 hi, u64* keys, u32* idx) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        keys[i] = (s[i] >= lo && s[i] < hi) ? pack_edge(s[i], d[i]) : ~0ull;
        idx[i] = u32(i);
    }
}

__global__ void k_pack_edges(const u32* s, const u32* d, u64 n, u64* keys, u32* idx) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        keys[i] = pack_edge(s[i], d[i]);
        idx[i] = u32(i);
    }
}

// Merge the |V| guards into the sorted unique edge list: edge i lands at
// i + src (guards of smaller rows precede it), guard v lands after every
// edge with src <= v.
__global__ void k_place_guards(const u64* ek, const u64* ev, u64 ne, u64 lo, u64 hi, u64* ok, u64* ov) {
    const u64 total = ne + (hi - lo);
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        if (i < ne) {
            const u64 k = ek[i];
            ok[i + src_of(k) - lo] = k;
            ov[i + src_of(k) - lo] = ev[i];
        } else {
            const u64 v = lo + (i - ne);
            const u64 g = pack_edge(u32(v), u32(kGuardDst));
            const u64 pos = lower_bound_dev(ek, ne, g) + (v - lo);
            ok[pos] = g;
            ov[pos] = 0;
        }
    }
}

__global__ void k_fill_u32(u32* a, u64 n, u32 v) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) a[i] = v;
}
__global__ void k_iota_u32(u32* a, u64 n) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) a[i] = u32(i);
}

// -------- BFS (analytics.hpp:22-48): frontier queues split by row length.
// Light rows (<= kHeavyRow slots): a warp per frontier vertex, lanes stride
// its slot interval (coalesced 8-B keys + 1-B states).  Heavy rows (RMAT
// hubs): kHeavyParts CTAs per vertex, each striding 1/kHeavyParts of the row,
// so one hub never serialises a level on a single warp.  Discovery is a CAS on
// dist; discovered vertices are enqueued (warp-aggregated: ballot + popc + one
// atomic per warp and queue) into the light or heavy next queue by their own
// row length.
constexpr u64 kHeavyRow = 1024;
// fixed grids (levels run back to back with device-side frontier sizes);
// measured on the C2 hub BFS: light 148x32 / heavy 148x64 CTAs beat 148x16 /
// 148x8 by 20% (more heavy-row parts in flight), and more parts per heavy row
// (64, 128) lose
constexpr unsigned kBfsLightGrid = 148 * 32, kBfsHeavyGrid = 148 * 64;
constexpr u32 kHeavyParts = 32;

// Discovery: a visited bitmap (|V| bits: 256 KB at C2, L1/L2-resident) is
// probed first and claimed with atomicOr; only the winner writes dist.  The
// probes of the frontier's edges are the BFS's dominant cost, and the bitmap
// is 32x smaller than dist.  (A stale "unset" bit only costs an atomic.)
__device__ __forceinline__ bool bfs_claim(u32* __restrict__ vis, u32* __restrict__ dist, u32 v, u32 depth) {
    const u32 bit = 1u << (v & 31u);
    if (vis[v >> 5] & bit) return false;
    if (atomicOr(&vis[v >> 5], bit) & bit) return false;
    dist[v] = depth;
    return true;
}

__device__ __forceinline__ void bfs_visit(const u64* __restrict__ ro, const u64* __restrict__ keys,
                                          const u8* __restrict__ st, u32* __restrict__ dist, u32* __restrict__ vis,
                                          u32 depth, u64 t, u64 e,
                                          u32* __restrict__ next, u32* __restrict__ hnext, u32* __restrict__ qn) {
    const unsigned lane = threadIdx.x & 31u;
    bool won = false;
    u32 v = 0;
    if (t < e && st[t] == kValid) {
        const u64 k = keys[t];
        if (!is_guard(k)) {
            v = dst_of(k);
            won = bfs_claim(vis, dist, v, depth);
        }
    }
    const bool heavy = won && (ro[v + 1] - ro[v]) > kHeavyRow;
    const unsigned lm = __ballot_sync(FULL, won && !heavy), hm = __ballot_sync(FULL, heavy);
    if (lm) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&qn[0], u32(__popc(lm)));
        base = __shfl_sync(FULL, base, 0);
        if (won && !heavy) next[base + __popc(lm & lanemask_lt())] = v;
    }
    if (hm) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&qn[1], u32(__popc(hm)));
        base = __shfl_sync(FULL, base, 0);
        if (heavy) hnext[base + __popc(hm & lanemask_lt())] = v;
    }
}

// Valid non-guard neighbours are packed into a per-warp queue (ballot ranks)
// across 128-slot chunks and rows, then probed 32 at a time with every lane
// busy: most slots of a row are gaps and short rows are the norm.
struct BfsWarpQueue {
    u32* q;    // 256 entries of shared memory
    u32 cnt;   // warp-uniform
    __device__ __forceinline__ void drain(const u64* __restrict__ ro, u32* __restrict__ dist, u32* __restrict__ vis,
                                          u32 depth,
                                          u32* __restrict__ next, u32* __restrict__ hnext, u32* __restrict__ qn) {
        const unsigned lane = threadIdx.x & 31u, below = lanemask_lt();
        __syncwarp();
        for (u32 base = 0; base < cnt; base += 32) {
            const bool act = base + lane < cnt;
            const u32 v = act ? q[base + lane] : 0u;
            bool won = false;
            if (act) won = bfs_claim(vis, dist, v, depth);
            const bool heavy = won && (ro[v + 1] - ro[v]) > kHeavyRow;
            const unsigned lm = __ballot_sync(FULL, won && !heavy), hm = __ballot_sync(FULL, heavy);
            if (lm) {
                u32 o = 0;
                if (lane == 0) o = atomicAdd(&qn[0], u32(__popc(lm)));
                o = __shfl_sync(FULL, o, 0);
                if (won && !heavy) next[o + __popc(lm & below)] = v;
            }
            if (hm) {
                u32 o = 0;
                if (lane == 0) o = atomicAdd(&qn[1], u32(__popc(hm)));
                o = __shfl_sync(FULL, o, 0);
                if (heavy) hnext[o + __popc(hm & below)] = v;
            }
        }
        __syncwarp();
        cnt = 0;
    }
    // the 128 slots [t0, t0 + 128) ∩ [., e): lane l reads t0 + 32 j + l
    __device__ __forceinline__ void push128(const u64* __restrict__ keys, const u8* __restrict__ st, u64 t0, u64 e,
                                            const u64* __restrict__ ro, u32* __restrict__ dist, u32* __restrict__ vis,
                                            u32 depth, u32* __restrict__ next, u32* __restrict__ hnext,
                                            u32* __restrict__ qn) {
        const unsigned lane = threadIdx.x & 31u, below = lanemask_lt();
        u32 vv[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const u64 t = t0 + 32 * j + lane;
            ok[j] = false;
            vv[j] = 0;
            if (t < e && st[t] == kValid) {
                const u64 k = keys[t];
                ok[j] = !is_guard(k);
                vv[j] = dst_of(k);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned m = __ballot_sync(FULL, ok[j]);
            if (ok[j]) q[cnt + __popc(m & below)] = vv[j];
            cnt += __popc(m);
        }
        if (cnt >= 128) drain(ro, dist, vis, depth, next, hnext, qn);  // room for the next chunk stays
    }
};

// (frontier sizes are read from the device: levels run back to back, the
// host only syncs once per window of levels)
// four slots per thread per call (t, t + S, t + 2S, t + 3S; S = the
// caller's stride, so each of the four rounds of loads is coalesced across the
// warp): the key/state loads, then the dist probes, then the CASes are each
// issued four at a time — the probes are random L2 reads, latency is the cost
__device__ __forceinline__ void bfs_visit4(const u64* __restrict__ ro, const u64* __restrict__ keys,
                                           const u8* __restrict__ st, u32* __restrict__ dist, u32* __restrict__ vis,
                                           u32 depth, u64 t,
                                           u64 S, u64 e, u32* __restrict__ next, u32* __restrict__ hnext,
                                           u32* __restrict__ qn) {
    const unsigned lane = threadIdx.x & 31u;
    u32 v[4];
    bool cand[4], won[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const u64 tj = t + j * S;
        cand[j] = false;
        v[j] = 0;
        if (tj < e && st[tj] == kValid) {
            const u64 k = keys[tj];
            if (!is_guard(k)) {
                v[j] = dst_of(k);
                cand[j] = true;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) cand[j] = cand[j] && !((vis[v[j] >> 5] >> (v[j] & 31u)) & 1u);
#pragma unroll
    for (int j = 0; j < 4; ++j) won[j] = cand[j] && bfs_claim(vis, dist, v[j], depth);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool heavy = won[j] && (ro[v[j] + 1] - ro[v[j]]) > kHeavyRow;
        const unsigned lm = __ballot_sync(FULL, won[j] && !heavy), hm = __ballot_sync(FULL, heavy);
        if (lm) {
            u32 base = 0;
            if (lane == 0) base = atomicAdd(&qn[0], u32(__popc(lm)));
            base = __shfl_sync(FULL, base, 0);
            if (won[j] && !heavy) next[base + __popc(lm & lanemask_lt())] = v[j];
        }
        if (hm) {
            u32 base = 0;
            if (lane == 0) base = atomicAdd(&qn[1], u32(__popc(hm)));
            base = __shfl_sync(FULL, base, 0);
            if (heavy) hnext[base + __popc(hm & lanemask_lt())] = v[j];
        }
    }
}

__global__ void __launch_bounds__(256) k_bfs_expand(const u32* __restrict__ frontier, const u32* nfp,
                                                    const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                    const u8* __restrict__ st, u32* __restrict__ dist,
                                                    u32* __restrict__ vis, u32 depth, u32* __restrict__ next,
                                                    u32* __restrict__ hnext, u32* __restrict__ qn) {
    __shared__ u32 s_q[8][256];
    const u32 nf = *nfp;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    BfsWarpQueue wq{s_q[threadIdx.x >> 5], 0};
    for (u64 f = warp; f < nf; f += nwarps) {
        const u32 u = frontier[f];
        const u64 b = ro[u], e = ro[u + 1];
        for (u64 t0 = b; t0 < e; t0 += 128) wq.push128(keys, st, t0, e, ro, dist, vis, depth, next, hnext, qn);
    }
    wq.drain(ro, dist, vis, depth, next, hnext, qn);
}

__global__ void __launch_bounds__(256) k_bfs_expand_heavy(const u32* __restrict__ hfrontier, const u32* nhp,
                                                          const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                          const u8* __restrict__ st, u32* __restrict__ dist,
                                                          u32* __restrict__ vis, u32 depth, u32* __restrict__ next,
                                                          u32* __restrict__ hnext, u32* __restrict__ qn) {
    // (a packed warp queue here measured slower: 1.03 vs 0.93 ms on the C2 hub BFS)
    const u32 nh = *nhp;
    for (u64 task = blockIdx.x; task < u64(nh) * kHeavyParts; task += gridDim.x) {
        const u32 u = hfrontier[task / kHeavyParts];
        const u64 p = task % kHeavyParts;
        const u64 b0 = ro[u], e0 = ro[u + 1], len = e0 - b0;
        const u64 b = b0 + (len * p) / kHeavyParts, e = b0 + (len * (p + 1)) / kHeavyParts;
        // whole warps iterate together (ballots inside)
        u64 t0 = b;
        for (; t0 + 3 * blockDim.x < e; t0 += 4 * blockDim.x)
            bfs_visit4(ro, keys, st, dist, vis, depth, t0 + threadIdx.x, blockDim.x, e, next, hnext, qn);
        for (; t0 < e; t0 += blockDim.x)
            bfs_visit(ro, keys, st, dist, vis, depth, t0 + threadIdx.x, e, next, hnext, qn);
    }
}

// -------- CC (analytics.hpp:53-82): min-root union-find over every stored
// edge (undirected closure).  Roots only ever link under smaller roots, so a
// tree's root is its minimum id and the final labels equal the reference's
// min-id-per-component labels bit for bit.
__device__ __forceinline__ u32 cc_find(u32* parent, u32 x) {
    u32 p = parent[x];
    while (p != x) {
        const u32 gp = parent[p];
        if (gp != p) parent[x] = gp;  // path halving (only ever shortcuts to an ancestor)
        x = p;
        p = gp;
    }
    return x;
}

// (over warp-packed edge queues: the pointer chases run with every lane busy)
__global__ void __launch_bounds__(256) k_cc_hook(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                                 u32* parent) {
    __shared__ u64 s_q[8 * 256];
    sweep_edges8_packed(keys, st, cap, s_q, [&](u64 k) {
        u32 a = src_of(k), b = dst_of(k);
        for (;;) {
            a = cc_find(parent, a);
            b = cc_find(parent, b);
            if (a == b) break;
            const u32 hi = a > b ? a : b, lo = a > b ? b : a;
            if (atomicCAS(&parent[hi], hi, lo) == hi) break;
            a = hi;
            b = lo;
        }
    });
}

__global__ void k_cc_flatten(u32* parent, u64 nv) {
    for (u64 v = blockIdx.x * u64(blockDim.x) + threadIdx.x; v < nv; v += u64(gridDim.x) * blockDim.x) {
        u32 x = u32(v);
        while (parent[x] != x) x = parent[x];
        parent[v] = x;
    }
}

// -------- PageRank (analytics.hpp:100-143)
__global__ void k_pr_prep(const double* __restrict__ x, const u32* __restrict__ outdeg, u64 n, double d,
                          double* __restrict__ share, double* dangling_sum) {
    double dang = 0.0;
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x) {
        const u32 od = outdeg[u];
        if (od == 0) {
            dang += x[u];
            share[u] = 0.0;
        } else {
            share[u] = __ddiv_rn(__dmul_rn(d, x[u]), double(od));
        }
    }
    block_atomic_add(dang, dangling_sum);
}

// One |V| pass per iteration after the push (analytics.hpp:112-141): y =
// base + pushed mass (base from the current dangling mass), L1 += |y - x|,
// and already the next iteration's inputs — share = d y / outdeg, the next
// dangling mass.
// Gate of iteration `it` inside a window of iterations launched without a
// host round trip: once the previous iteration's L1 residual fell below
// epsilon (analytics.hpp:136-140 stops there) the sticky `done` flag turns
// every later kernel of the window into a no-op; otherwise it clears the
// push accumulator y and the next dangling sum.
__global__ void k_pr_gate(const double* __restrict__ l1_prev, double eps, u32* done, double* __restrict__ y, u64 n,
                          double* next_dangling) {
    __shared__ bool skip;
    if (threadIdx.x == 0) {
        bool d = *done != 0;
        if (!d && l1_prev && *l1_prev < eps) d = true;
        skip = d;
        if (d && blockIdx.x == 0) *done = 1;
    }
    __syncthreads();
    if (skip) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) *next_dangling = 0.0;
    double2* y2 = reinterpret_cast<double2*>(y);
    const u64 n2 = n / 2;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n2; i += u64(gridDim.x) * blockDim.x)
        y2[i] = make_double2(0.0, 0.0);
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) y[n - 1] = 0.0;
}

__global__ void k_fill_f64(double* __restrict__ x, u64 n, double v) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) x[i] = v;
}

__global__ void k_pr_finish_next(double* __restrict__ x, double* __restrict__ y, const u32* __restrict__ outdeg, u64 n,
                                 double d, const double* dangling, double* next_dangling, double* l1,
                                 double* __restrict__ share, const u32* done = nullptr) {
    if (done && *done) return;
    const double nn = double(n);
    const double base = __dadd_rn(__ddiv_rn(1.0 - d, nn), __ddiv_rn(__dmul_rn(d, *dangling), nn));
    double acc = 0.0, dang = 0.0;
    for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x) {
        const double v = __dadd_rn(base, y[u]);
        y[u] = v;
        acc += fabs(v - x[u]);
        const u32 od = outdeg[u];
        if (od) {
            share[u] = __ddiv_rn(__dmul_rn(d, v), double(od));
        } else {
            share[u] = 0.0;
            dang += v;
        }
    }
    block_atomic_add(acc, l1);
    block_atomic_add(dang, next_dangling);
}

// ---------------------------------------------------------------- Graph

Graph::Graph(const gpma_graph_config* cfg, int device, u64 nv_, u64 lo_, u64 hi_)
    : pma(cfg ? &cfg->profile : nullptr, device), nv(nv_), lo(lo_), hi(hi_ > nv_ ? nv_ : hi_) {
    if (lo > hi) throw ApiError(PMA_EINVAL, "shard: need lo <= hi <= num_vertices");
    if (cfg) {
        if (cfg->engine != 0)
            throw ApiError(PMA_EINVAL, "GraphConfig.engine: only the segment engine (GPMA+) is provided");
        ecfg.eager = cfg->deletion_mode == PMA_EAGER;
        fill_target = cfg->fill_target;
    }
    ro.reserve(nloc() + 1);
    pma.d_row_offsets = ro.ptr;
    pma.num_vertices = nloc();
    pma.ro_lo = lo;
}

// stable (key, arrival index) sort of the edge keys by key bits [0, nbits):
// the result pair of buffers (kin/vin or kout/vout)
static std::pair<const u64*, const u32*> sort_pairs(cudaStream_t s, RadixWorkspace& ws, u64* kin, u64* kout, u32* vin,
                                                    u32* vout, u64 n, int nbits) {
    const int alt = radix_sort(s, ws, kin, kout, vin, vout, n, 0, nbits);
    using R = std::pair<const u64*, const u32*>;
    return alt ? R(kout, vout) : R(kin, vin);
}

static int bits_for(u64 v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

// DynamicGraph::from_edges (graph.hpp:66-92)
void Graph::from_edges_device(const u32* d_src, const u32* d_dst, const double* d_w, u64 n) {
    cudaStream_t s = pma.stream();
    Ctr* ctr = scratch_ctr();
    if (n > 0) {
        ull init = ~0ull;
        GPMA_CUDA(cudaMemcpyAsync(&ctr->bad_index, &init, 8, cudaMemcpyHostToDevice, s));
        k_check_ids<<<grid_for(n, 256), 256, 0, s>>>(d_src, d_dst, n, nv, ctr);
        GPMA_LAUNCH_CHECK();
        ull bad = 0;
        GPMA_CUDA(cudaMemcpyAsync(&bad, &ctr->bad_index, 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        if (bad != ~0ull) {
            u32 bs = 0, bd = 0;
            GPMA_CUDA(cudaMemcpy(&bs, d_src + bad, 4, cudaMemcpyDeviceToHost));
            GPMA_CUDA(cudaMemcpy(&bd, d_dst + bad, 4, cudaMemcpyDeviceToHost));
            throw ApiError(PMA_EINVAL, "edge (" + std::to_string(bs) + ", " + std::to_string(bd) +
                                           ") outside vertex range " + std::to_string(nv));
        }
    }
    DevBuf<u64> k0, k1, uk, uvv, mk, mv;
    DevBuf<u32> i0, i1;
    k0.reserve(n + 1);
    k1.reserve(n + 1);
    i0.reserve(n + 1);
    i1.reserve(n + 1);
    u64 ne = 0;
    uk.reserve(n + 1);
    uvv.reserve(n + 1);
    if (n > 0) {
        int nbits = 32 + bits_for(nv ? nv - 1 : 0);
        if (is_shard()) {
            k_pack_edges_shard<<<grid_for(n, 256), 256, 0, s>>>(d_src, d_dst, n, lo, hi, k0.ptr, i0.ptr);
            nbits = 64;
        } else {
            k_pack_edges<<<grid_for(n, 256), 256, 0, s>>>(d_src, d_dst, n, k0.ptr, i0.ptr);
        }
        GPMA_LAUNCH_CHECK();
        const auto sorted = sort_pairs(s, pma.rws, k0.ptr, k1.ptr, i0.ptr, i1.ptr, n, nbits);
        // dedupe, last arrival wins (stable sort keeps arrival order)
        const u64* sk = sorted.first;
        const u32* si = sorted.second;
        u64* ok_ = uk.ptr;
        u64* ov_ = uvv.ptr;
        Ctr* c = ctr;
        run_compact(
            s, pma.ws, nullptr, n, n,
            [=] __device__(ull i) { return (i + 1 == n || sk[i + 1] != sk[i]) && sk[i] != ~0ull; },
            [=] __device__(ull i, unsigned f, ull x) {
                if (f) {
                    ok_[x] = sk[i];
                    ov_[x] = __double_as_longlong(d_w ? d_w[si[i]] : 1.0);
                }
            },
            [=] __device__(ull total) { c->n_unique = total; });
        GPMA_CUDA(cudaMemcpyAsync(&ne, &ctr->n_unique, 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
    }
    const u64 total = ne + nloc();
    mk.reserve(total + 1);
    mv.reserve(total + 1);
    if (total > 0) {
        k_place_guards<<<grid_for(total, 256), 256, 0, s>>>(uk.ptr, uvv.ptr, ne, lo, hi, mk.ptr, mv.ptr);
        GPMA_LAUNCH_CHECK();
    }
    pma.from_sorted_device(mk.ptr, mv.ptr, total, fill_target);
    GPMA_CUDA(cudaStreamSynchronize(s));
}

Ctr* Graph::scratch_ctr() {
    if (!d_ctr_) GPMA_CUDA(cudaMalloc(&d_ctr_, sizeof(Ctr)));
    GPMA_CUDA(cudaMemsetAsync(d_ctr_, 0, sizeof(Ctr), pma.stream()));
    return d_ctr_;
}

Graph::~Graph() {
    if (d_ctr_) cudaFree(d_ctr_);
}

// DynamicGraph::apply_batch (graph.hpp:130-162)
void Graph::reserve_batch(u64 n) {
    bk.reserve(n + 1);
    bv.reserve(n + 1);
    bo.reserve(n + 1);
    pma.reserve_batch(n);
}

void Graph::apply_batch_device(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                               u64 nd, pma_stats* out) {
    apply_batch_impl(is, id, nullptr, iw, ni, ds, dd, nd, out);
}

void Graph::apply_batch_mixed_device(const u64* keys, const double* w, u64 n, pma_stats* out) {
    if (nv > (1ull << 31)) throw ApiError(PMA_EINVAL, "apply_batch_mixed: vertex ids must be < 2^31");
    apply_batch_impl(nullptr, nullptr, keys, w, n, nullptr, nullptr, 0, out);
}

void Graph::apply_batch_impl(const u32* is, const u32* id, const u64* mk, const double* iw, u64 ni, const u32* ds,
                             const u32* dd, u64 nd, pma_stats* out) {
    const u64 n = ni + nd;
    bk.reserve(n + 1);
    bv.reserve(n + 1);
    bo.reserve(n + 1);
    GraphFront gf{is, id, iw, ni, ds, dd, nd, nv, lo, hi, mk, bk.ptr, bv.ptr, bo.ptr};
    pma_stats st;
    pma.batch_update_device(nullptr, nullptr, nullptr, n, ecfg, &st, &gf);
    if (gf.bad_insert >= 0) {
        u32 bs = 0, bd = 0;
        if (mk) {
            u64 key = 0;
            GPMA_CUDA(cudaMemcpy(&key, mk + gf.bad_insert, 8, cudaMemcpyDeviceToHost));
            bs = src_of(key);
            bd = dst_of(key);
        } else {
            GPMA_CUDA(cudaMemcpy(&bs, is + gf.bad_insert, 4, cudaMemcpyDeviceToHost));
            GPMA_CUDA(cudaMemcpy(&bd, id + gf.bad_insert, 4, cudaMemcpyDeviceToHost));
        }
        if (is_shard() && bd < nv && bs < nv)
            throw ApiError(PMA_EINVAL, "edge (" + std::to_string(bs) + ", " + std::to_string(bd) +
                                           ") outside shard source range [" + std::to_string(lo) + ", " +
                                           std::to_string(hi) + ")");
        throw ApiError(PMA_EINVAL, "edge (" + std::to_string(bs) + ", " + std::to_string(bd) +
                                       ") outside vertex range " + std::to_string(nv));
    }
    st.batch_size = n - gf.guard_deletes;
    st.deletes_missed += gf.guard_deletes;
    if (out) *out = st;
}

void Graph::row_offsets(u64* out) {
    GPMA_CUDA(cudaMemcpyAsync(out, ro.ptr, (nloc() + 1) * 8, cudaMemcpyDeviceToHost, pma.stream()));
    GPMA_CUDA(cudaStreamSynchronize(pma.stream()));
}

u64 Graph::num_edges() const { return pma.valid_count - nloc(); }

void Graph::csr_snapshot(u64* h_ro, u32* h_col, double* h_val) {
    cudaStream_t s = pma.stream();
    const u64 ne = num_edges();
    DevBuf<u64> dro;
    DevBuf<u32> dcol;
    DevBuf<double> dval;
    dro.reserve(nloc() + 1);
    dcol.reserve(ne + 1);
    dval.reserve(ne + 1);
    GPMA_CUDA(cudaMemsetAsync(dro.ptr, 0, 8, s));
    const u64* kk = pma.d_keys;
    const u64* vv = pma.d_vals;
    const u8* ss = pma.d_st;
    u64* r = dro.ptr;
    u32* c = dcol.ptr;
    double* w = dval.ptr;
    const u64 cap = pma.capacity();
    const u64 rlo = lo;
    if (cap > 0) {
        run_compact(
            s, pma.ws, nullptr, cap, cap,
            [=] __device__(ull t) { return ss[t] == kValid && !is_guard(kk[t]); },
            [=] __device__(ull t, unsigned f, ull x) {
                if (f) {
                    c[x] = dst_of(kk[t]);
                    w[x] = __longlong_as_double((long long)vv[t]);
                } else if (ss[t] == kValid) {
                    r[src_of(kk[t]) - rlo + 1] = x;  // guard of row u: entries of rows <= u
                }
            },
            NoFin{});
    }
    if (h_ro) GPMA_CUDA(cudaMemcpyAsync(h_ro, dro.ptr, (nloc() + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (h_col && ne) GPMA_CUDA(cudaMemcpyAsync(h_col, dcol.ptr, ne * 4, cudaMemcpyDeviceToHost, s));
    if (h_val && ne) GPMA_CUDA(cudaMemcpyAsync(h_val, dval.ptr, ne * 8, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------- analytics

void Graph::bfs(u32 root, u32* h_dist, u64* reached) {
    if (is_shard()) throw ApiError(PMA_ELOGIC, "whole-graph analytics on a shard: use the gpma_shard_* entry points");
    if (root >= nv) throw ApiError(PMA_EINVAL, "bfs: root outside vertex range");
    cudaStream_t s = pma.stream();
    GPMA_CUDA(cudaEventRecord(pma_ev(0), s));
    dist.reserve(nv);
    q0.reserve(nv + 1);
    q1.reserve(nv + 1);
    h0.reserve(nv + 1);
    h1.reserve(nv + 1);
    qn.reserve(2);
    k_fill_u32<<<grid_for(nv, 256, 148 * 16), 256, 0, s>>>(dist.ptr, nv, GPMA_UNREACHED);
    GPMA_LAUNCH_CHECK();
    const u32 zero = 0;
    GPMA_CUDA(cudaMemcpyAsync(dist.ptr + root, &zero, 4, cudaMemcpyHostToDevice, s));
    bvis.reserve(nv / 32 + 1);
    GPMA_CUDA(cudaMemsetAsync(bvis.ptr, 0, (nv / 32 + 1) * 4, s));
    const u32 rbit = 1u << (root & 31u);
    GPMA_CUDA(cudaMemcpyAsync(bvis.ptr + root / 32, &rbit, 4, cudaMemcpyHostToDevice, s));
    u64 rr[2] = {0, 0};
    GPMA_CUDA(cudaMemcpyAsync(rr, ro.ptr + root, 16, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    const bool root_heavy = rr[1] - rr[0] > kHeavyRow;
    GPMA_CUDA(cudaMemcpyAsync(root_heavy ? h0.ptr : q0.ptr, &root, 4, cudaMemcpyHostToDevice, s));
    // per level L: (light, heavy) vertices discovered, qn[2L], qn[2L + 1];
    // level 0 = the root.  Levels are launched kBfsWindow at a time with
    // their frontier sizes read on the device; the host syncs once per
    // window and stops at the first empty level (later launches of the
    // window found empty frontiers and did nothing).
    constexpr u32 kBfsWindow = 4;
    u64 cap_levels = 0;
    const u32 first[2] = {root_heavy ? 0u : 1u, root_heavy ? 1u : 0u};
    u64 total = 1;
    u32 depth = 0;
    u32 *cur = q0.ptr, *nxt = q1.ptr, *hcur = h0.ptr, *hnxt = h1.ptr;
    u64 launches = 3;
    for (bool done = false; !done;) {
        if (depth + kBfsWindow + 1 > cap_levels) {  // grow the counter ring (keeps earlier levels)
            const u64 nc = (depth + kBfsWindow + 1) * 2 + 64;
            DevBuf<u32> q2;
            q2.reserve(2 * nc);
            GPMA_CUDA(cudaMemsetAsync(q2.ptr, 0, 2 * nc * 4, s));
            if (cap_levels) GPMA_CUDA(cudaMemcpyAsync(q2.ptr, qn.ptr, 2 * cap_levels * 4, cudaMemcpyDeviceToDevice, s));
            else GPMA_CUDA(cudaMemcpyAsync(q2.ptr, first, 8, cudaMemcpyHostToDevice, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
            std::swap(qn.ptr, q2.ptr);
            std::swap(qn.cap, q2.cap);
            cap_levels = nc;
        }
        const u32 d0 = depth;
        for (u32 w = 0; w < kBfsWindow; ++w) {
            ++depth;
            const u32* cnt_in = qn.ptr + 2 * (depth - 1);
            u32* cnt_out = qn.ptr + 2 * depth;
            k_bfs_expand<<<kBfsLightGrid, 256, 0, s>>>(cur, cnt_in, ro.ptr, pma.d_keys, pma.d_st, dist.ptr, bvis.ptr,
                                                 depth, nxt, hnxt, cnt_out);
            GPMA_LAUNCH_CHECK();
            k_bfs_expand_heavy<<<kBfsHeavyGrid, 256, 0, s>>>(hcur, cnt_in + 1, ro.ptr, pma.d_keys, pma.d_st, dist.ptr,
                                                       bvis.ptr, depth, nxt, hnxt, cnt_out);
            GPMA_LAUNCH_CHECK();
            launches += 2;
            std::swap(cur, nxt);
            std::swap(hcur, hnxt);
        }
        h_lv_.resize(2 * kBfsWindow);
        GPMA_CUDA(cudaMemcpyAsync(h_lv_.data(), qn.ptr + 2 * (d0 + 1), 2 * kBfsWindow * 4, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        for (u32 w = 0; w < kBfsWindow; ++w) {
            const u64 c = u64(h_lv_[2 * w]) + h_lv_[2 * w + 1];
            if (c == 0) {
                done = true;
                break;
            }
            total += c;
        }
    }
    GPMA_CUDA(cudaEventRecord(pma_ev(1), s));
    if (h_dist) GPMA_CUDA(cudaMemcpyAsync(h_dist, dist.ptr, nv * 4, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    if (reached) *reached = total;
    record_timing(launches);
}

void Graph::cc(u32* h_labels) {
    if (is_shard()) throw ApiError(PMA_ELOGIC, "whole-graph analytics on a shard: use the gpma_shard_* entry points");
    cudaStream_t s = pma.stream();
    GPMA_CUDA(cudaEventRecord(pma_ev(0), s));
    dist.reserve(nv + 1);
    k_iota_u32<<<grid_for(nv, 256, 148 * 16), 256, 0, s>>>(dist.ptr, nv);
    GPMA_LAUNCH_CHECK();
    // 8x the resident CTAs (the hooks are pointer chases: more warps queued
    // keep the SMs fed; measured 1x 0.29, 4x 0.24, 8x 0.23 ms on C2)
    static const unsigned cc_res = resident_grid(k_cc_hook, 256) * 8;
    k_cc_hook<<<grid_for(pma.capacity() / 256 * 8, 256, cc_res), 256, 0, s>>>(pma.d_keys, pma.d_st, pma.capacity(), dist.ptr);
    GPMA_LAUNCH_CHECK();
    k_cc_flatten<<<grid_for(nv, 256, 148 * 16), 256, 0, s>>>(dist.ptr, nv);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaEventRecord(pma_ev(1), s));
    if (h_labels) GPMA_CUDA(cudaMemcpyAsync(h_labels, dist.ptr, nv * 4, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    record_timing(3);
}

void Graph::pagerank(double d, double eps, u64 max_iters, const double* h_warm, double* h_ranks, u64* iters,
                     int* converged) {
    if (is_shard()) throw ApiError(PMA_ELOGIC, "whole-graph analytics on a shard: use the gpma_shard_* entry points");
    if (nv == 0) throw ApiError(PMA_EINVAL, "pagerank: empty vertex set");
    cudaStream_t s = pma.stream();
    GPMA_CUDA(cudaEventRecord(pma_ev(0), s));
    px.reserve(nv);
    py.reserve(nv);
    pshare.reserve(nv);
    psc.reserve(2);
    outdeg.reserve(nv);
    if (h_warm) {
        GPMA_CUDA(cudaMemcpyAsync(px.ptr, h_warm, nv * 8, cudaMemcpyHostToDevice, s));
    } else {
        k_fill_f64<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(px.ptr, nv, 1.0 / double(nv));
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaMemsetAsync(outdeg.ptr, 0, nv * 4, s));
    const u64 cap = pma.capacity();
    static const unsigned od_res = resident_grid(k_outdeg, 256);
    k_outdeg<<<grid_for(cap / 8, 256, od_res), 256, 0, s>>>(pma.d_keys, pma.d_st, cap, outdeg.ptr);
    GPMA_LAUNCH_CHECK();
    prepare_hot(outdeg.ptr, nv);
    u64 launches = 3;
    double* x = px.ptr;
    double* y = py.ptr;
    *converged = 0;
    u64 it = 1;
    pr_iter_ms_ = 0.0;
    // psc = [dangling_A, -, dangling_B, -]: iteration parity p reads the
    // dangling sum at psc[2p] and produces the next one at psc[2(1-p)]; the L1
    // residual of iteration i goes to the ring pl1[(i - 1) % kRing].
    // Iterations run in windows of kWin without a host round trip: the gate
    // of each iteration turns the rest of the window into no-ops once an L1
    // fell below epsilon, and the host reads the window's residuals once.
    constexpr u64 kWin = 4, kRing = 16;
    psc.reserve(4);
    pl1.reserve(kRing);
    pdone.reserve(1);
    GPMA_CUDA(cudaMemsetAsync(psc.ptr, 0, 32, s));
    GPMA_CUDA(cudaMemsetAsync(pdone.ptr, 0, 4, s));
    k_pr_prep<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(x, outdeg.ptr, nv, d, pshare.ptr, psc.ptr);
    GPMA_LAUNCH_CHECK();
    ++launches;
    static const unsigned pr_res = resident_grid(k_pr_push, 256);  // measured best vs 0.5x / 2x
    u64 last = 0;  // the iteration whose result is in x
    while (it <= max_iters) {
        const u64 win = std::min(kWin, max_iters - it + 1);
        const u64 r0 = (it - 1) % kRing;
        GPMA_CUDA(cudaMemsetAsync(pl1.ptr + r0, 0, win * 8, s));
        GPMA_CUDA(cudaEventRecord(pma_ev(2), s));
        for (u64 j = 0; j < win; ++j) {
            const u64 i = it + j;
            const int p = int(i & 1) ^ 1;  // i = 1 -> p = 0
            double* cur = psc.ptr + 2 * p;
            double* nxt = psc.ptr + 2 * (1 - p);
            const double* l1_prev = i > 1 ? pl1.ptr + (i - 2) % kRing : nullptr;
            k_pr_gate<<<grid_for(nv / 2 + 1, 256, 148 * 4), 256, 0, s>>>(l1_prev, eps, pdone.ptr, y, nv, nxt);
            k_pr_push<<<pr_res, 256, 0, s>>>(pma.d_keys, pma.d_st, cap, pshare.ptr, y, hot_table.ptr, hot_ids.ptr,
                                             nhot_, pdone.ptr);
            // (148x4 CTAs: fewer per-CTA reductions; measured 1% better than 148x8)
            k_pr_finish_next<<<grid_for(nv, 256, 148 * 4), 256, 0, s>>>(x, y, outdeg.ptr, nv, d, cur, nxt,
                                                                       pl1.ptr + (i - 1) % kRing, pshare.ptr,
                                                                       pdone.ptr);
            GPMA_LAUNCH_CHECK();
            launches += 3;
            std::swap(x, y);  // y (finished) is the next x; the gate clears the next accumulator
        }
        GPMA_CUDA(cudaEventRecord(pma_ev(3), s));
        double l1[kWin] = {};
        GPMA_CUDA(cudaMemcpyAsync(l1, pl1.ptr + r0, win * 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        float ms = 0;
        cudaEventElapsedTime(&ms, pma_ev(2), pma_ev(3));
        pr_iter_ms_ += ms;
        u64 j = 0;
        while (j < win && !(l1[j] < eps)) ++j;
        if (j < win) {  // iteration it + j converged; later ones were no-ops
            *converged = 1;
            last = it + j;
            break;
        }
        last = it + win - 1;
        it += win;
    }
    // iteration i finished into py when i is odd, px when even (x started as px)
    x = last == 0 ? px.ptr : ((last & 1) ? py.ptr : px.ptr);
    it = last;
    *iters = *converged ? it : max_iters;
    GPMA_CUDA(cudaEventRecord(pma_ev(1), s));
    GPMA_CUDA(cudaMemcpyAsync(h_ranks, x, nv * 8, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    record_timing(launches);
    pma.timing.rounds_ms = pr_iter_ms_;
}

// Hot-destination set of the push (analytics_kernels.cuh): the <= kHotMax
// vertices of largest out-degree (>= 64), from a bit-length histogram.
void Graph::prepare_hot(const u32* od, u64 n) {
    cudaStream_t s = pma.stream();
    hot_table.reserve(2 * kHotTable);
    hot_ids.reserve(kHotMax);
    hot_hist.reserve(34);
    GPMA_CUDA(cudaMemsetAsync(hot_hist.ptr, 0, 34 * 4, s));
    k_hot_hist<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(od, n, hot_hist.ptr);
    GPMA_LAUNCH_CHECK();
    u32 h[34] = {};
    GPMA_CUDA(cudaMemcpyAsync(h, hot_hist.ptr, 33 * 4, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    u32 min_bits = 33, total = 0;
    for (int b = 32; b >= 7; --b) {  // bit length >= 7: out-degree >= 64
        if (total + h[b] > kHotMax) break;
        total += h[b];
        if (h[b]) min_bits = u32(b);
    }
    nhot_ = 0;
    if (total == 0) return;
    GPMA_CUDA(cudaMemsetAsync(hot_table.ptr, 0xFF, 2 * kHotTable * 4, s));
    GPMA_CUDA(cudaMemsetAsync(hot_hist.ptr + 33, 0, 4, s));
    k_hot_select<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(od, n, min_bits, hot_table.ptr, hot_ids.ptr,
                                                          hot_hist.ptr + 33);
    GPMA_LAUNCH_CHECK();
    nhot_ = total;
}

void Graph::spmv(const double* h_x, double* h_y) {
    if (is_shard()) throw ApiError(PMA_ELOGIC, "whole-graph analytics on a shard: use the gpma_shard_* entry points");
    cudaStream_t s = pma.stream();
    px.reserve(nv + 1);
    py.reserve(nv + 1);
    if (nv) GPMA_CUDA(cudaMemcpyAsync(px.ptr, h_x, nv * 8, cudaMemcpyHostToDevice, s));
    GPMA_CUDA(cudaEventRecord(pma_ev(0), s));
    if (nv) {
        k_spmv<<<grid_for(nv * 32, 256, 148 * 16), 256, 0, s>>>(ro.ptr, nv, pma.d_keys, pma.d_vals, pma.d_st, px.ptr,
                                                                py.ptr);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaEventRecord(pma_ev(1), s));
    if (nv) GPMA_CUDA(cudaMemcpyAsync(h_y, py.ptr, nv * 8, cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    record_timing(1);
}

cudaEvent_t Graph::pma_ev(int i) {
    if (!evs_[i]) GPMA_CUDA(cudaEventCreate(&evs_[i]));
    return evs_[i];
}

void Graph::record_timing(u64 launches) {
    float ms = 0;
    cudaEventElapsedTime(&ms, pma_ev(0), pma_ev(1));
    pma.timing = pma_timing{};
    pma.timing.device_ms = ms;
    pma.timing.kernel_launches = launches;
}

}  // namespace gpma
