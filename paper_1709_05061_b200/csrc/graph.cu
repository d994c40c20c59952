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
// Light rows (<= kHeavyRow slots): a warp walks up to 32 frontier rows at
// once (k_bfs_expand).  Heavy rows: kHeavyParts warps per row; huge rows
// (hubs): kHugeParts CTAs per row, so one hub never serialises a level
// (k_bfs_expand_heavy).  Discovery claims a visited bit; discovered vertices
// are enqueued (warp-aggregated: ballot + popc + one atomic per warp and
// queue) into the light, heavy or huge next queue by their own row length.
constexpr u64 kHeavyRow = 1024;
// fixed grids (levels run back to back with device-side frontier sizes);
// measured on the C2 hub BFS: light 148x32 / heavy 148x64 CTAs beat 148x16 /
// 148x8 by 20% (more heavy-row parts in flight), and more parts per heavy row
// (64, 128) lose
constexpr unsigned kBfsLightGrid = 148 * 32, kBfsHeavyGrid = 148 * 64;
#ifndef GPMA_BFS_HEAVY_PARTS
#define GPMA_BFS_HEAVY_PARTS 8
#endif
#ifndef GPMA_BFS_HUGE_ROW
#define GPMA_BFS_HUGE_ROW 16384
#endif
constexpr u32 kHeavyParts = GPMA_BFS_HEAVY_PARTS;  // heavy rows (kHeavyRow, kHugeRow]: a warp per part
constexpr u64 kHugeRow = GPMA_BFS_HUGE_ROW;        // huge rows (hubs): a CTA per part
constexpr u32 kHugeParts = 32;
constexpr u32 kBfsQueue = 512;  // per-warp candidate queue (shared memory)

// Discovery: a visited bitmap (|V| bits: 256 KB at C2, L1/L2-resident) is
// probed first and claimed with atomicOr; only the winner writes dist.  The
// probes of the frontier's edges are the BFS's dominant cost, and the bitmap
// is 32x smaller than dist.  (A stale "unset" bit only costs an atomic.)
// Light rows: k_bfs_expand; heavy rows: k_bfs_expand_heavy; both claim
// through bfs_claim4.

// Claim up to 4 candidate neighbours per lane (v[j], cand[j]): the bitmap
// CASes are issued together, then the winners' dist stores and row-bound
// loads (light / heavy by their own row length), then ONE warp-aggregated
// append per queue for all 4 rounds.
__device__ __forceinline__ void bfs_claim4(const u64* __restrict__ ro, u32* __restrict__ dist, u32* __restrict__ vis,
                                           u32 depth, const u32 (&v)[4], const bool (&cand)[4],
                                           u32* __restrict__ next, u32* __restrict__ hnext, u32* __restrict__ gnext,
                                           u32* __restrict__ qn) {
    const unsigned lane = threadIdx.x & 31u, below = lanemask_lt();
    u32 old[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) old[j] = cand[j] ? atomicOr(&vis[v[j] >> 5], 1u << (v[j] & 31u)) : ~0u;
    bool won[4];
    u64 lo[4], hi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        won[j] = !((old[j] >> (v[j] & 31u)) & 1u);
        lo[j] = hi[j] = 0;
        if (won[j]) {
            dist[v[j]] = depth;
            lo[j] = ro[v[j]];
            hi[j] = ro[v[j] + 1];
        }
    }
    unsigned lm[4], hm[4], gm[4];
    u32 nl = 0, nh = 0, ng = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const u64 len = hi[j] - lo[j];
        const bool huge = won[j] && len > kHugeRow, heavy = won[j] && len > kHeavyRow && !huge;
        lm[j] = __ballot_sync(FULL, won[j] && !heavy && !huge);
        hm[j] = __ballot_sync(FULL, heavy);
        gm[j] = __ballot_sync(FULL, huge);
        nl += __popc(lm[j]);
        nh += __popc(hm[j]);
        ng += __popc(gm[j]);
    }
    u32 bl = 0, bh = 0, bg = 0;
    if (lane == 0) {
        if (nl) bl = atomicAdd(&qn[0], nl);
        if (nh) bh = atomicAdd(&qn[1], nh);
        if (ng) bg = atomicAdd(&qn[2], ng);
    }
    bl = __shfl_sync(FULL, bl, 0);
    bh = __shfl_sync(FULL, bh, 0);
    bg = __shfl_sync(FULL, bg, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if ((lm[j] >> lane) & 1u) next[bl + __popc(lm[j] & below)] = v[j];
        if ((hm[j] >> lane) & 1u) hnext[bh + __popc(hm[j] & below)] = v[j];
        if ((gm[j] >> lane) & 1u) gnext[bg + __popc(gm[j] & below)] = v[j];
        bl += __popc(lm[j]);
        bh += __popc(hm[j]);
        bg += __popc(gm[j]);
    }
}

// Unvisited-looking neighbours are packed into a per-warp queue (ballot
// ranks) and claimed 128 at a time (bfs_claim4) with every lane busy.
struct BfsWarpQueue {
    u32* q;    // kBfsQueue entries of shared memory
    u32 cnt;   // warp-uniform
    __device__ __forceinline__ void drain(const u64* __restrict__ ro, u32* __restrict__ dist, u32* __restrict__ vis,
                                          u32 depth, u32* __restrict__ next, u32* __restrict__ hnext,
                                          u32* __restrict__ gnext, u32* __restrict__ qn) {
        const unsigned lane = threadIdx.x & 31u;
        __syncwarp();
        for (u32 base = 0; base < cnt; base += 128) {
            u32 v[4];
            bool c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const u32 i = base + 32 * j + lane;
                c[j] = i < cnt;
                v[j] = c[j] ? q[i] : 0u;
            }
            bfs_claim4(ro, dist, vis, depth, v, c, next, hnext, gnext, qn);
        }
        __syncwarp();
        cnt = 0;
    }
    // 4 candidates per lane (ballot-packed); drains when fewer than 128 slots remain
    __device__ __forceinline__ void push4(const u32 (&v)[4], const bool (&c)[4], const u64* __restrict__ ro,
                                          u32* __restrict__ dist, u32* __restrict__ vis, u32 depth,
                                          u32* __restrict__ next, u32* __restrict__ hnext, u32* __restrict__ gnext,
                                          u32* __restrict__ qn) {
        const unsigned below = lanemask_lt();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned m = __ballot_sync(FULL, c[j]);
            if (c[j]) q[cnt + __popc(m & below)] = v[j];
            cnt += __popc(m);
        }
        if (cnt > kBfsQueue - 128) drain(ro, dist, vis, depth, next, hnext, gnext, qn);
    }
};

// one slot: (neighbour, is it a candidate) — the state and the key are loaded
// together (a key line with no Valid slot is rare at PMA densities), then the
// visited bit is probed
__device__ __forceinline__ void bfs_slot_load(const u64* __restrict__ keys, const u8* __restrict__ st, u64 t, bool in,
                                              u8& s, u64& k) {
    s = in ? st[t] : u8(kEmpty);
    k = in ? keys[t] : 0ull;
}

// Light rows: a warp takes 32 frontier vertices at once (their row bounds load
// together, one per lane), then walks their concatenated slot intervals 128
// slots per step: each lane's 4 slots (state + key, then the visited bit) are
// independent loads instead of one row's chain after another.
__global__ void __launch_bounds__(256) k_bfs_expand(const u32* __restrict__ frontier, const u32* nfp,
                                                    const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                    const u8* __restrict__ st, u32* __restrict__ dist,
                                                    u32* __restrict__ vis, u32 depth, u32* __restrict__ next,
                                                    u32* __restrict__ hnext, u32* __restrict__ gnext,
                                                    u32* __restrict__ qn) {
    __shared__ u32 s_q[8][kBfsQueue];
    const u32 nf = *nfp;
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    BfsWarpQueue wq{s_q[threadIdx.x >> 5], 0};
    // vertices per warp batch: up to 32, fewer while the frontier is too
    // small to give every warp a full batch (parallelism first)
    u32 V = u32((u64(nf) + nwarps - 1) / nwarps);
    V = V < 1 ? 1 : (V > 32 ? 32 : V);
    for (u64 f0 = warp * V; f0 < nf; f0 += nwarps * V) {
        u64 b = 0;
        u32 len = 0;
        if (lane < V && f0 + lane < nf) {
            const u32 u = frontier[f0 + lane];
            b = ro[u];
            len = u32(ro[u + 1] - b);  // <= kHeavyRow
        }
        u32 inc = len;  // inclusive prefix of the row lengths over the lanes
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(FULL, inc, d);
            if (lane >= unsigned(d)) inc += y;
        }
        const u32 total = __shfl_sync(FULL, inc, 31);
        for (u32 s0 = 0; s0 < total; s0 += 128) {
            u8 sv[4];
            u64 kv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const u32 sl = s0 + 32 * j + lane;
                const u32 sc = sl < total ? sl : total - 1;
                u32 r = 0;  // the row holding slot sc: first lane whose prefix exceeds it
#pragma unroll
                for (u32 step = 16; step > 0; step >>= 1)
                    if (__shfl_sync(FULL, inc, r + step - 1) <= sc) r += step;
                const u64 br = __shfl_sync(FULL, b, r);
                const u32 er = __shfl_sync(FULL, inc, r), lr = __shfl_sync(FULL, len, r);
                bfs_slot_load(keys, st, br + (sc - (er - lr)), sl < total, sv[j], kv[j]);
            }
            u32 v[4];
            bool c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[j] = dst_of(kv[j]);
                c[j] = sv[j] == kValid && !is_guard(kv[j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = c[j] && !((vis[v[j] >> 5] >> (v[j] & 31u)) & 1u);
            wq.push4(v, c, ro, dist, vis, depth, next, hnext, gnext, qn);
        }
    }
    wq.drain(ro, dist, vis, depth, next, hnext, gnext, qn);
}

// one step of a row part: 4 slots per lane at stride S (32 for a warp, the
// CTA size for a CTA): state + key loads together, then the visited probes;
// the unvisited-looking neighbours go to the warp's queue (claimed 128 at a
// time when it fills: the claims' round trips no longer gate every step)
__device__ __forceinline__ void bfs_step4(const u64* __restrict__ keys, const u8* __restrict__ st,
                                          u32* __restrict__ vis, u64 t, u64 S, u64 e, BfsWarpQueue& wq,
                                          const u64* __restrict__ ro, u32* __restrict__ dist, u32 depth,
                                          u32* __restrict__ next, u32* __restrict__ hnext, u32* __restrict__ gnext,
                                          u32* __restrict__ qn) {
    u8 sv[4];
    u64 kv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bfs_slot_load(keys, st, t + j * S, t + j * S < e, sv[j], kv[j]);
    u32 v[4];
    bool c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] = dst_of(kv[j]);
        c[j] = sv[j] == kValid && !is_guard(kv[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = c[j] && !((vis[v[j] >> 5] >> (v[j] & 31u)) & 1u);
    wq.push4(v, c, ro, dist, vis, depth, next, hnext, gnext, qn);
}

// Huge rows (hubs, > kHugeRow slots): kHugeParts CTAs per row; then heavy
// rows (kHeavyRow, kHugeRow]: kHeavyParts WARPS per row (a CTA per part left
// most of its threads idle on the shorter heavy rows).  One launch; a
// per-warp candidate queue as in k_bfs_expand (measured 0.63 -> 0.58 ms on
// the C2 BFS).
__global__ void __launch_bounds__(256) k_bfs_expand_heavy(const u32* __restrict__ hfrontier, const u32* nhp,
                                                          const u32* __restrict__ gfrontier, const u32* ngp,
                                                          const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                          const u8* __restrict__ st, u32* __restrict__ dist,
                                                          u32* __restrict__ vis, u32 depth, u32* __restrict__ next,
                                                          u32* __restrict__ hnext, u32* __restrict__ gnext,
                                                          u32* __restrict__ qn) {
    __shared__ u32 s_q[8][kBfsQueue];
    BfsWarpQueue wq{s_q[threadIdx.x >> 5], 0};
    const u32 ng = *ngp, nh = *nhp;
    for (u64 task = blockIdx.x; task < u64(ng) * kHugeParts; task += gridDim.x) {
        const u32 u = gfrontier[task / kHugeParts];
        const u64 p = task % kHugeParts;
        const u64 b0 = ro[u], len = ro[u + 1] - b0;
        const u64 b = b0 + (len * p) / kHugeParts, e = b0 + (len * (p + 1)) / kHugeParts;
        for (u64 t0 = b; t0 < e; t0 += 4 * blockDim.x)  // (whole CTAs: each warp's ballots stay converged)
            bfs_step4(keys, st, vis, t0 + threadIdx.x, blockDim.x, e, wq, ro, dist, depth, next, hnext, gnext, qn);
    }
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 task = warp; task < u64(nh) * kHeavyParts; task += nwarps) {
        const u32 u = hfrontier[task / kHeavyParts];
        const u64 p = task % kHeavyParts;
        const u64 b0 = ro[u], len = ro[u + 1] - b0;
        const u64 b = b0 + (len * p) / kHeavyParts, e = b0 + (len * (p + 1)) / kHeavyParts;
        for (u64 t0 = b; t0 < e; t0 += 128)
            bfs_step4(keys, st, vis, t0 + lane, 32, e, wq, ro, dist, depth, next, hnext, gnext, qn);
    }
    wq.drain(ro, dist, vis, depth, next, hnext, gnext, qn);
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
    NvtxScope nvtx_scope("gpma.bfs");
    if (is_shard()) throw ApiError(PMA_ELOGIC, "whole-graph analytics on a shard: use the gpma_shard_* entry points");
    if (root >= nv) throw ApiError(PMA_EINVAL, "bfs: root outside vertex range");
    cudaStream_t s = pma.stream();
    GPMA_CUDA(cudaEventRecord(pma_ev(0), s));
    dist.reserve(nv);
    q0.reserve(nv + 1);
    q1.reserve(nv + 1);
    h0.reserve(nv + 1);
    h1.reserve(nv + 1);
    g0.reserve(nv + 1);
    g1.reserve(nv + 1);
    qn.reserve(3);
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
    const int root_class = rr[1] - rr[0] > kHugeRow ? 2 : (rr[1] - rr[0] > kHeavyRow ? 1 : 0);
    GPMA_CUDA(cudaMemcpyAsync(root_class == 2 ? g0.ptr : (root_class == 1 ? h0.ptr : q0.ptr), &root, 4,
                              cudaMemcpyHostToDevice, s));
    // per level L: (light, heavy, huge) vertices discovered, qn[3L .. 3L + 2];
    // level 0 = the root.  Levels are launched kBfsWindow at a time with
    // their frontier sizes read on the device; the host syncs once per
    // window and stops at the first empty level (later launches of the
    // window found empty frontiers and did nothing).
    constexpr u32 kBfsWindow = 4;
    u64 cap_levels = 0;
    const u32 first[3] = {root_class == 0 ? 1u : 0u, root_class == 1 ? 1u : 0u, root_class == 2 ? 1u : 0u};
    u64 total = 1;
    u32 depth = 0;
    u32 *cur = q0.ptr, *nxt = q1.ptr, *hcur = h0.ptr, *hnxt = h1.ptr, *gcur = g0.ptr, *gnxt = g1.ptr;
    u64 launches = 3;
    for (bool done = false; !done;) {
        if (depth + kBfsWindow + 1 > cap_levels) {  // grow the counter ring (keeps earlier levels)
            const u64 nc = (depth + kBfsWindow + 1) * 2 + 64;
            DevBuf<u32> q2;
            q2.reserve(3 * nc);
            GPMA_CUDA(cudaMemsetAsync(q2.ptr, 0, 3 * nc * 4, s));
            if (cap_levels) GPMA_CUDA(cudaMemcpyAsync(q2.ptr, qn.ptr, 3 * cap_levels * 4, cudaMemcpyDeviceToDevice, s));
            else GPMA_CUDA(cudaMemcpyAsync(q2.ptr, first, 12, cudaMemcpyHostToDevice, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
            std::swap(qn.ptr, q2.ptr);
            std::swap(qn.cap, q2.cap);
            cap_levels = nc;
        }
        const u32 d0 = depth;
        for (u32 w = 0; w < kBfsWindow; ++w) {
            ++depth;
            const u32* cnt_in = qn.ptr + 3 * (depth - 1);
            u32* cnt_out = qn.ptr + 3 * depth;
            k_bfs_expand<<<kBfsLightGrid, 256, 0, s>>>(cur, cnt_in, ro.ptr, pma.d_keys, pma.d_st, dist.ptr, bvis.ptr,
                                                 depth, nxt, hnxt, gnxt, cnt_out);
            GPMA_LAUNCH_CHECK();
            k_bfs_expand_heavy<<<kBfsHeavyGrid, 256, 0, s>>>(hcur, cnt_in + 1, gcur, cnt_in + 2, ro.ptr, pma.d_keys,
                                                       pma.d_st, dist.ptr, bvis.ptr, depth, nxt, hnxt, gnxt, cnt_out);
            GPMA_LAUNCH_CHECK();
            launches += 2;
            std::swap(cur, nxt);
            std::swap(hcur, hnxt);
            std::swap(gcur, gnxt);
        }
        h_lv_.resize(3 * kBfsWindow);
        GPMA_CUDA(cudaMemcpyAsync(h_lv_.data(), qn.ptr + 3 * (d0 + 1), 3 * kBfsWindow * 4, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        for (u32 w = 0; w < kBfsWindow; ++w) {
            const u64 c = u64(h_lv_[3 * w]) + h_lv_[3 * w + 1] + h_lv_[3 * w + 2];
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
    NvtxScope nvtx_scope("gpma.cc");
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
    NvtxScope nvtx_scope("gpma.pagerank");
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
    NvtxScope nvtx_scope("gpma.spmv");
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
    pma.resolve_all();  // (a batch's deferred record joins the sum first)
    pma.timing = pma_timing{};
    pma.timing.device_ms = ms;
    pma.timing.kernel_launches = launches;
}

}  // namespace gpma
