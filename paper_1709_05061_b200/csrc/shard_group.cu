// shard_group.cu — the key-range sharded GPMA+ across GPUs driven entirely
// from the C ABI (SURVEY §8b gpma_shard_group_*, §8e): one process per GPU,
// one shard per rank, and the collectives issued by the library itself over
// NCCL on the shard's stream — no Python or torch.distributed in the loop.
//
// Per batch the only exchange is routing: the owner
// partition of this rank's share (shard.cu), a count exchange, one
// variable-size all-to-all of 8-B EdgeKeys (+ weights) as grouped
// ncclSend/ncclRecv, then the owner applies its routed batch.  An insert
// naming a vertex outside the graph is counted by its sender and one scalar
// all-reduce makes every rank reject the batch before any shard applies.
//
// Analytics: BFS expands the owned frontier, reduce-scatters the candidate
// flags to their owners (MAX over u8, padded per-rank chunks) and the owners
// admit unreached vertices; CC propagates min labels (all-reduce MIN);
// PageRank all-reduces the pushed contributions (SUM, f64); SpMV and the
// final distance vector are all-gathered.
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): the library loads and
// every single-GPU entry point works without it; in a PyTorch process the
// already loaded NCCL is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "graph_impl.cuh"
#include "pmagraph_cuda.h"

namespace gpma {

struct NcclApi {
    void* h = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclReduceScatter) ReduceScatter = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

static NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.h = h;
#define GPMA_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
            GPMA_NCCL_SYM(GetUniqueId);
            GPMA_NCCL_SYM(CommInitRank);
            GPMA_NCCL_SYM(CommDestroy);
            GPMA_NCCL_SYM(AllReduce);
            GPMA_NCCL_SYM(ReduceScatter);
            GPMA_NCCL_SYM(AllGather);
            GPMA_NCCL_SYM(Send);
            GPMA_NCCL_SYM(Recv);
            GPMA_NCCL_SYM(GroupStart);
            GPMA_NCCL_SYM(GroupEnd);
            GPMA_NCCL_SYM(GetErrorString);
#undef GPMA_NCCL_SYM
        }
    }
    if (!api.h || !api.CommInitRank || !api.Send || !api.GroupEnd)
        throw ApiError(PMA_ECUDA, "shard group: NCCL (libnccl.so.2) is not available");
    return api;
}

#define GPMA_NCCL(call)                                                                                         \
    do {                                                                                                        \
        const ncclResult_t r_ = (call);                                                                         \
        if (r_ != ncclSuccess)                                                                                  \
            throw ApiError(PMA_ECUDA, std::string("NCCL " #call " failed: ") + nccl().GetErrorString(r_));      \
    } while (0)

__device__ __forceinline__ int owner_of_v(u32 v, const u32* b, int world) {
    int lo = 0, hi = world;  // last r with b[r] <= v
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// BFS (analytics.hpp:22-48), one level: the out-neighbours of the owned
// frontier flagged in per-owner chunks (owner r's vertex v at r * chunk +
// v - bounds[r]), ready for a reduce-scatter to the owners.
// Owners' candidate flags for the frontier's out-neighbours (mark only: the
// flags are idempotent stores, reduce-scattered to the owners afterwards).
// Rows up to kGroupHubRow slots: a warp walks up to 32 frontier rows at once
// (row bounds one per lane, then 128-slot steps of lane-parallel loads, as
// graph.cu's k_bfs_expand); longer rows are set aside for
// k_group_bfs_mark_hubs, which splits each over kGroupHubParts CTAs (one warp
// walking an RMAT hub's row serialised the level).
constexpr u64 kGroupHubRow = 4096;
constexpr u32 kGroupHubParts = 32;

__device__ __forceinline__ void group_flag(const u64* __restrict__ keys, const u8* __restrict__ st, u64 t,
                                           const u32* s_b, int world, u64 chunk, u8* __restrict__ flags) {
    if (st[t] != kValid) return;
    const u64 k = keys[t];
    if (is_guard(k)) return;
    const u32 v = dst_of(k);
    const int r = owner_of_v(v, s_b, world);
    flags[u64(r) * chunk + (v - s_b[r])] = 1;
}

__global__ void __launch_bounds__(256) k_group_bfs_mark(const u32* __restrict__ frontier, u32 nf,
                                                        const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                        const u8* __restrict__ st, const u32* __restrict__ bounds,
                                                        int world, u64 chunk, u8* __restrict__ flags,
                                                        u32* __restrict__ hubs, u32* __restrict__ nhubs) {
    __shared__ u32 s_b[65];
    for (int i = threadIdx.x; i <= world; i += blockDim.x) s_b[i] = bounds[i];
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    u32 V = u32((u64(nf) + nwarps - 1) / nwarps);  // rows per warp batch (fewer while the frontier is small)
    V = V < 1 ? 1 : (V > 32 ? 32 : V);
    for (u64 f0 = warp * V; f0 < nf; f0 += nwarps * V) {
        u64 b = 0;
        u32 len = 0;
        if (lane < V && f0 + lane < nf) {
            const u32 u = frontier[f0 + lane];
            b = ro[u];
            const u64 l = ro[u + 1] - b;
            if (l > kGroupHubRow) hubs[atomicAdd(nhubs, 1u)] = u;
            else len = u32(l);
        }
        u32 inc = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(FULL, inc, d);
            if (lane >= unsigned(d)) inc += y;
        }
        const u32 total = __shfl_sync(FULL, inc, 31);
        for (u32 s0 = 0; s0 < total; s0 += 128) {
            u64 tt[4];
            bool in[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const u32 sl = s0 + 32 * j + lane;
                const u32 sc = sl < total ? sl : total - 1;
                u32 r = 0;  // the row holding slot sc
#pragma unroll
                for (u32 step = 16; step > 0; step >>= 1)
                    if (__shfl_sync(FULL, inc, r + step - 1) <= sc) r += step;
                const u64 br = __shfl_sync(FULL, b, r);
                const u32 er = __shfl_sync(FULL, inc, r), lr = __shfl_sync(FULL, len, r);
                tt[j] = br + (sc - (er - lr));
                in[j] = sl < total;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (in[j]) group_flag(keys, st, tt[j], s_b, world, chunk, flags);
        }
    }
}

__global__ void __launch_bounds__(256) k_group_bfs_mark_hubs(const u32* __restrict__ hubs, const u32* nhubs,
                                                             const u64* __restrict__ ro, const u64* __restrict__ keys,
                                                             const u8* __restrict__ st, const u32* __restrict__ bounds,
                                                             int world, u64 chunk, u8* __restrict__ flags) {
    __shared__ u32 s_b[65];
    for (int i = threadIdx.x; i <= world; i += blockDim.x) s_b[i] = bounds[i];
    __syncthreads();
    const u32 nh = *nhubs;
    for (u64 task = blockIdx.x; task < u64(nh) * kGroupHubParts; task += gridDim.x) {
        const u32 u = hubs[task / kGroupHubParts];
        const u64 p = task % kGroupHubParts;
        const u64 b0 = ro[u], len = ro[u + 1] - b0;
        const u64 b = b0 + (len * p) / kGroupHubParts, e = b0 + (len * (p + 1)) / kGroupHubParts;
        for (u64 t = b + threadIdx.x; t < e; t += blockDim.x) group_flag(keys, st, t, s_b, world, chunk, flags);
    }
}

// owners admit their flagged, unreached vertices at `depth` (next frontier,
// global ids); *n counts them
__global__ void k_group_bfs_admit(const u8* __restrict__ flags, u64 nloc, u32* __restrict__ dist, u32 depth, u64 lo,
                                  u32* __restrict__ next, u32* __restrict__ n) {
    const unsigned lane = threadIdx.x & 31u;
    for (u64 i0 = blockIdx.x * u64(blockDim.x); i0 < nloc; i0 += u64(gridDim.x) * blockDim.x) {
        const u64 i = i0 + threadIdx.x;
        const bool win = i < nloc && flags[i] && dist[i] == GPMA_UNREACHED;
        if (win) dist[i] = depth;
        const unsigned wm = __ballot_sync(FULL, win);
        if (wm) {
            u32 base = 0;
            if (lane == 0) base = atomicAdd(n, u32(__popc(wm)));
            base = __shfl_sync(FULL, base, 0);
            if (win) next[base + __popc(wm & lanemask_lt())] = u32(lo + i);
        }
    }
}

__global__ void k_group_fill_u32(u32* __restrict__ x, u64 n, u32 v) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) x[i] = v;
}
__global__ void k_group_iota(u32* __restrict__ x, u64 n) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) x[i] = u32(i);
}
__global__ void k_group_fill_f64(double* __restrict__ x, u64 n, double v) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) x[i] = v;
}

}  // namespace gpma

using namespace gpma;

namespace gpma {
Graph* graph_impl(gpma_graph* g);  // capi.cu
}

struct gpma_shard_group {
    int world = 1, rank = 0, device = 0;
    ncclComm_t comm = nullptr;
    bool own_comm = false;
    gpma_graph* g = nullptr;  // this rank's shard (a regular graph handle)
    std::vector<uint32_t> bounds;
    u64 nv = 0, lo = 0, hi = 0, chunk = 0;
    DevBuf<u32> d_bounds;
    DevBuf<u64> skeys, rkeys, counts, rcounts, bad;
    DevBuf<double> sw, rw;
    DevBuf<u8> flags, myflags;
    DevBuf<u32> dist, frontier, next, nnext, labels, prev, od, gath, hubs;
    DevBuf<double> x, y, gy;
    std::string err;
};

extern "C" {
// declared in pmagraph_cuda.h (shard entry points of capi.cu)
int gpma_shard_from_edges_device(const gpma_graph_config* cfg, int device, size_t num_vertices, uint32_t lo,
                                 uint32_t hi, const uint32_t* d_src, const uint32_t* d_dst, const double* d_weights,
                                 size_t n, gpma_graph** out);
}

namespace {
thread_local std::string g_group_err;

template <class F>
int group_guard(gpma_shard_group* sg, F&& f) {
    try {
        f();
        return PMA_OK;
    } catch (const ApiError& e) {
        (sg ? sg->err : g_group_err) = e.what();
        g_group_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        (sg ? sg->err : g_group_err) = e.what();
        g_group_err = e.what();
        return PMA_ECUDA;
    }
}

void check_rc(int rc, gpma_graph* g) {
    if (rc) throw ApiError(rc, gpma_last_error(g));
}

cudaStream_t group_stream(gpma_shard_group* sg) { return static_cast<cudaStream_t>(gpma_cuda_stream(sg->g)); }
Graph& impl(gpma_shard_group* sg) { return *graph_impl(sg->g); }
}  // namespace

extern "C" {

const char* gpma_shard_group_last_error(const gpma_shard_group* sg) {
    return sg ? sg->err.c_str() : g_group_err.c_str();
}

int gpma_nccl_unique_id(void* id128) {
    return group_guard(nullptr, [&] {
        if (!id128) throw ApiError(PMA_EINVAL, "gpma_nccl_unique_id: id is NULL");
        ncclUniqueId id;
        GPMA_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(id128, &id, sizeof(id));
    });
}

int gpma_nccl_comm_create(const void* id128, int world, int rank, int device, void** comm) {
    return group_guard(nullptr, [&] {
        if (!id128 || !comm) throw ApiError(PMA_EINVAL, "gpma_nccl_comm_create: NULL argument");
        GPMA_CUDA(cudaSetDevice(device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        ncclComm_t c = nullptr;
        GPMA_NCCL(nccl().CommInitRank(&c, world, id, rank));
        *comm = c;
    });
}

int gpma_nccl_comm_destroy(void* comm) {
    return group_guard(nullptr, [&] {
        if (comm) GPMA_NCCL(nccl().CommDestroy(static_cast<ncclComm_t>(comm)));
    });
}

int gpma_shard_group_create(const gpma_graph_config* cfg, int device, size_t num_vertices, const uint32_t* bounds,
                            int world, int rank, const void* nccl_id128, void* nccl_comm, const uint32_t* d_src,
                            const uint32_t* d_dst, const double* d_weights, size_t n, gpma_shard_group** out) {
    gpma_shard_group* sg = nullptr;
    return group_guard(nullptr, [&] {
        if (!out || !bounds) throw ApiError(PMA_EINVAL, "gpma_shard_group_create: NULL argument");
        if (world < 1 || world > 64 || rank < 0 || rank >= world)
            throw ApiError(PMA_EINVAL, "gpma_shard_group_create: world must be in [1, 64], 0 <= rank < world");
        if (num_vertices > (1ull << 31)) throw ApiError(PMA_EINVAL, "shard group: vertex ids must be < 2^31");
        for (int r = 0; r < world; ++r)
            if (bounds[r] > bounds[r + 1]) throw ApiError(PMA_EINVAL, "shard group: bounds must be non-decreasing");
        if (bounds[0] != 0 || bounds[world] != num_vertices)
            throw ApiError(PMA_EINVAL, "shard group: bounds must cover [0, num_vertices)");
        GPMA_CUDA(cudaSetDevice(device));
        sg = new gpma_shard_group;
        try {
            sg->world = world;
            sg->rank = rank;
            sg->device = device;
            sg->bounds.assign(bounds, bounds + world + 1);
            sg->nv = num_vertices;
            sg->lo = bounds[rank];
            sg->hi = bounds[rank + 1];
            for (int r = 0; r < world; ++r) sg->chunk = std::max<u64>(sg->chunk, u64(bounds[r + 1] - bounds[r]));
            if (sg->chunk == 0) sg->chunk = 1;
            if (nccl_comm) {
                sg->comm = static_cast<ncclComm_t>(nccl_comm);
            } else {
                if (!nccl_id128) throw ApiError(PMA_EINVAL, "shard group: an NCCL unique id or communicator is needed");
                ncclUniqueId id;
                std::memcpy(&id, nccl_id128, sizeof(id));
                GPMA_NCCL(nccl().CommInitRank(&sg->comm, world, id, rank));
                sg->own_comm = true;
            }
            check_rc(gpma_shard_from_edges_device(cfg, device, num_vertices, uint32_t(sg->lo), uint32_t(sg->hi), d_src,
                                                  d_dst, d_weights, n, &sg->g),
                     nullptr);
            sg->d_bounds.reserve(world + 1);
            GPMA_CUDA(cudaMemcpy(sg->d_bounds.ptr, bounds, (world + 1) * 4, cudaMemcpyHostToDevice));
            sg->counts.reserve(world + 1);
            sg->rcounts.reserve(world + 1);
            sg->bad.reserve(1);
        } catch (...) {
            if (sg->g) gpma_destroy(sg->g);
            if (sg->own_comm && sg->comm) nccl().CommDestroy(sg->comm);
            delete sg;
            sg = nullptr;
            throw;
        }
        *out = sg;
    });
}

int gpma_shard_group_destroy(gpma_shard_group* sg) {
    if (!sg) return PMA_OK;
    cudaSetDevice(sg->device);
    if (sg->g) gpma_destroy(sg->g);
    if (sg->own_comm && sg->comm && nccl().CommDestroy) nccl().CommDestroy(sg->comm);
    delete sg;
    return PMA_OK;
}

gpma_graph* gpma_shard_group_graph(gpma_shard_group* sg) { return sg ? sg->g : nullptr; }

int gpma_shard_group_apply_batch(gpma_shard_group* sg, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                                 const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                                 const uint32_t* d_del_dst, size_t n_del, pma_stats* stats, uint64_t* routed,
                                 uint64_t* sent) {
    if (!sg) {
        g_group_err = "null handle";
        return PMA_EINVAL;
    }
    return group_guard(sg, [&] {
        GPMA_CUDA(cudaSetDevice(sg->device));
        NcclApi& nc = nccl();
        const int W = sg->world;
        cudaStream_t s = group_stream(sg);
        const u64 n = n_ins + n_del;
        const bool weighted = d_ins_w != nullptr;
        sg->skeys.reserve(n + 1);
        if (weighted) sg->sw.reserve(n + 1);
        // 1. owner partition of this rank's share (counts: W owners + bad inserts)
        check_rc(gpma_route_batch_async(sg->g, d_ins_src, d_ins_dst, d_ins_w, n_ins, d_del_src, d_del_dst, n_del,
                                        sg->d_bounds.ptr, W, sg->skeys.ptr, weighted ? sg->sw.ptr : nullptr,
                                        sg->counts.ptr),
                 sg->g);
        // 2. counts to their owners + the bad-insert total, one round trip
        GPMA_NCCL(nc.GroupStart());
        for (int r = 0; r < W; ++r) {
            GPMA_NCCL(nc.Send(sg->counts.ptr + r, 1, ncclUint64, r, sg->comm, s));
            GPMA_NCCL(nc.Recv(sg->rcounts.ptr + r, 1, ncclUint64, r, sg->comm, s));
        }
        GPMA_NCCL(nc.GroupEnd());
        GPMA_NCCL(nc.AllReduce(sg->counts.ptr + W, sg->bad.ptr, 1, ncclUint64, ncclSum, sg->comm, s));
        std::vector<u64> sc(W + 1), rc(W), bad(1);
        GPMA_CUDA(cudaMemcpyAsync(sc.data(), sg->counts.ptr, (W + 1) * 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaMemcpyAsync(rc.data(), sg->rcounts.ptr, W * 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaMemcpyAsync(bad.data(), sg->bad.ptr, 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        if (bad[0]) {
            // check_ids (graph.hpp:133-137) rejects the batch before any
            // mutation: every rank raises, no shard applied anything
            if (sc[W]) {
                std::vector<uint32_t> hs(n_ins), hd(n_ins);
                GPMA_CUDA(cudaMemcpy(hs.data(), d_ins_src, n_ins * 4, cudaMemcpyDeviceToHost));
                GPMA_CUDA(cudaMemcpy(hd.data(), d_ins_dst, n_ins * 4, cudaMemcpyDeviceToHost));
                for (u64 i = 0; i < n_ins; ++i)
                    if (hs[i] >= sg->nv || hd[i] >= sg->nv)
                        throw ApiError(PMA_EINVAL, "edge (" + std::to_string(hs[i]) + ", " + std::to_string(hd[i]) +
                                                       ") outside vertex range " + std::to_string(sg->nv));
            }
            throw ApiError(PMA_EINVAL, "apply_batch rejected on every shard: an insert names a vertex outside "
                                       "vertex range " + std::to_string(sg->nv));
        }
        // 3. the all-to-all of EdgeKeys (+ weights): owner-major send buffer,
        // receive in sender-rank order (arrival order kept per sender)
        u64 nrecv = 0;
        for (int r = 0; r < W; ++r) nrecv += rc[r];
        sg->rkeys.reserve(nrecv + 1);
        if (weighted) sg->rw.reserve(nrecv + 1);
        GPMA_NCCL(nc.GroupStart());
        u64 so = 0, ro = 0;
        for (int r = 0; r < W; ++r) {
            if (sc[r]) {
                GPMA_NCCL(nc.Send(sg->skeys.ptr + so, sc[r], ncclUint64, r, sg->comm, s));
                if (weighted) GPMA_NCCL(nc.Send(sg->sw.ptr + so, sc[r], ncclFloat64, r, sg->comm, s));
            }
            if (rc[r]) {
                GPMA_NCCL(nc.Recv(sg->rkeys.ptr + ro, rc[r], ncclUint64, r, sg->comm, s));
                if (weighted) GPMA_NCCL(nc.Recv(sg->rw.ptr + ro, rc[r], ncclFloat64, r, sg->comm, s));
            }
            so += sc[r];
            ro += rc[r];
        }
        GPMA_NCCL(nc.GroupEnd());
        // 4. the owner applies its routed batch (stream-ordered after the receives)
        check_rc(gpma_apply_batch_routed_device(sg->g, sg->rkeys.ptr, weighted ? sg->rw.ptr : nullptr, nrecv, stats),
                 sg->g);
        if (routed) *routed = nrecv;
        if (sent) *sent = n - sc[sg->rank];
    });
}

int gpma_shard_group_bfs(gpma_shard_group* sg, uint32_t root, uint32_t* dist_out, uint64_t* reached) {
    if (!sg) {
        g_group_err = "null handle";
        return PMA_EINVAL;
    }
    return group_guard(sg, [&] {
        if (root >= sg->nv) throw ApiError(PMA_EINVAL, "bfs: root out of range");
        GPMA_CUDA(cudaSetDevice(sg->device));
        NcclApi& nc = nccl();
        cudaStream_t s = group_stream(sg);
        Graph& G = impl(sg);
        const int W = sg->world;
        const u64 nloc = sg->hi - sg->lo, C = sg->chunk;
        sg->flags.reserve(W * C);
        sg->myflags.reserve(C);
        sg->dist.reserve(C);
        sg->frontier.reserve(nloc + 1);
        sg->next.reserve(nloc + 1);
        sg->nnext.reserve(3);
        sg->hubs.reserve(nloc + 1);
        k_group_fill_u32<<<grid_for(C, 256, 148 * 4), 256, 0, s>>>(sg->dist.ptr, C, GPMA_UNREACHED);
        u32 nf = 0;
        if (root >= sg->lo && root < sg->hi) {  // the owner seeds the frontier
            const u32 zero = 0;
            GPMA_CUDA(cudaMemcpyAsync(sg->dist.ptr + (root - sg->lo), &zero, 4, cudaMemcpyHostToDevice, s));
            GPMA_CUDA(cudaMemcpyAsync(sg->frontier.ptr, &root, 4, cudaMemcpyHostToDevice, s));
            nf = 1;
        }
        u64 total = 1;
        for (u32 depth = 1;; ++depth) {
            GPMA_CUDA(cudaMemsetAsync(sg->flags.ptr, 0, W * C, s));
            if (nf) {
                GPMA_CUDA(cudaMemsetAsync(sg->nnext.ptr + 2, 0, 4, s));
                k_group_bfs_mark<<<148 * 16, 256, 0, s>>>(
                    sg->frontier.ptr, nf, G.pma.ro_base(), G.pma.d_keys, G.pma.d_st, sg->d_bounds.ptr, W, C,
                    sg->flags.ptr, sg->hubs.ptr, sg->nnext.ptr + 2);
                GPMA_LAUNCH_CHECK();
                k_group_bfs_mark_hubs<<<148 * 8, 256, 0, s>>>(sg->hubs.ptr, sg->nnext.ptr + 2, G.pma.ro_base(),
                                                              G.pma.d_keys, G.pma.d_st, sg->d_bounds.ptr, W, C,
                                                              sg->flags.ptr);
            }
            GPMA_LAUNCH_CHECK();
            GPMA_NCCL(nc.ReduceScatter(sg->flags.ptr, sg->myflags.ptr, C, ncclUint8, ncclMax, sg->comm, s));
            GPMA_CUDA(cudaMemsetAsync(sg->nnext.ptr, 0, 8, s));
            k_group_bfs_admit<<<grid_for(nloc, 256, 148 * 4), 256, 0, s>>>(sg->myflags.ptr, nloc, sg->dist.ptr, depth,
                                                                         sg->lo, sg->next.ptr, sg->nnext.ptr);
            GPMA_LAUNCH_CHECK();
            GPMA_NCCL(nc.AllReduce(sg->nnext.ptr, sg->nnext.ptr + 1, 1, ncclUint32, ncclSum, sg->comm, s));
            u32 h[2] = {0, 0};
            GPMA_CUDA(cudaMemcpyAsync(h, sg->nnext.ptr, 8, cudaMemcpyDeviceToHost, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
            if (h[1] == 0) break;
            total += h[1];
            std::swap(sg->frontier.ptr, sg->next.ptr);
            std::swap(sg->frontier.cap, sg->next.cap);
            nf = h[0];
        }
        if (reached) *reached = total;
        if (dist_out) {  // every owner's range, gathered (padded chunks)
            sg->gath.reserve(W * C);
            GPMA_NCCL(nc.AllGather(sg->dist.ptr, sg->gath.ptr, C, ncclUint32, sg->comm, s));
            // each owner's chunk straight into the caller's array (one DMA per
            // rank; no pageable staging copy)
            for (int r = 0; r < W; ++r)
                GPMA_CUDA(cudaMemcpyAsync(dist_out + sg->bounds[r], sg->gath.ptr + u64(r) * C,
                                          (sg->bounds[r + 1] - sg->bounds[r]) * 4, cudaMemcpyDeviceToHost, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
        }
    });
}

int gpma_shard_group_cc(gpma_shard_group* sg, uint32_t* labels_out) {
    if (!sg) {
        g_group_err = "null handle";
        return PMA_EINVAL;
    }
    return group_guard(sg, [&] {
        GPMA_CUDA(cudaSetDevice(sg->device));
        NcclApi& nc = nccl();
        cudaStream_t s = group_stream(sg);
        const u64 nv = sg->nv;
        sg->labels.reserve(nv + 1);
        sg->prev.reserve(nv + 1);
        k_group_iota<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(sg->labels.ptr, nv);
        GPMA_LAUNCH_CHECK();
        for (;;) {  // min-label propagation to the component minima (analytics.hpp:53-82)
            GPMA_CUDA(cudaMemcpyAsync(sg->prev.ptr, sg->labels.ptr, nv * 4, cudaMemcpyDeviceToDevice, s));
            check_rc(gpma_shard_cc_hook(sg->g, sg->labels.ptr), sg->g);
            GPMA_NCCL(nc.AllReduce(sg->labels.ptr, sg->labels.ptr, nv, ncclUint32, ncclMin, sg->comm, s));
            int changed = 0;  // replicated labels: every rank decides the same
            check_rc(gpma_cc_jump(sg->g, sg->labels.ptr, nv, sg->prev.ptr, &changed), sg->g);
            if (!changed) break;
        }
        if (labels_out) {
            GPMA_CUDA(cudaMemcpyAsync(labels_out, sg->labels.ptr, nv * 4, cudaMemcpyDeviceToHost, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
        }
    });
}

int gpma_shard_group_pagerank(gpma_shard_group* sg, double damping, double eps, size_t max_iters, const double* warm,
                              double* ranks, uint64_t* iterations, int* converged) {
    if (!sg) {
        g_group_err = "null handle";
        return PMA_EINVAL;
    }
    return group_guard(sg, [&] {
        GPMA_CUDA(cudaSetDevice(sg->device));
        NcclApi& nc = nccl();
        cudaStream_t s = group_stream(sg);
        const u64 nv = sg->nv;
        if (nv == 0) throw ApiError(PMA_EINVAL, "pagerank: empty vertex set");
        sg->od.reserve(nv + 1);
        sg->x.reserve(nv + 1);
        sg->y.reserve(nv + 1);
        check_rc(gpma_shard_outdeg(sg->g, sg->od.ptr), sg->g);
        GPMA_NCCL(nc.AllReduce(sg->od.ptr, sg->od.ptr, nv, ncclUint32, ncclSum, sg->comm, s));
        if (warm) GPMA_CUDA(cudaMemcpyAsync(sg->x.ptr, warm, nv * 8, cudaMemcpyHostToDevice, s));
        else k_group_fill_f64<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(sg->x.ptr, nv, 1.0 / double(nv));
        GPMA_LAUNCH_CHECK();
        double* x = sg->x.ptr;
        double* y = sg->y.ptr;
        u64 it = 0;
        int conv = 0;
        while (it < max_iters) {  // analytics.hpp:100-143 (push, owners' rows)
            ++it;
            check_rc(gpma_shard_pr_push(sg->g, x, sg->od.ptr, damping, y), sg->g);
            GPMA_NCCL(nc.AllReduce(y, y, nv, ncclFloat64, ncclSum, sg->comm, s));
            double l1 = 0;
            check_rc(gpma_pr_finish(sg->g, x, y, nv, sg->od.ptr, damping, &l1), sg->g);
            std::swap(x, y);
            if (l1 < eps) {
                conv = 1;
                break;
            }
        }
        if (iterations) *iterations = it;
        if (converged) *converged = conv;
        if (ranks) {
            GPMA_CUDA(cudaMemcpyAsync(ranks, x, nv * 8, cudaMemcpyDeviceToHost, s));
            GPMA_CUDA(cudaStreamSynchronize(s));
        }
    });
}

int gpma_shard_group_spmv(gpma_shard_group* sg, const double* x, double* y) {
    if (!sg) {
        g_group_err = "null handle";
        return PMA_EINVAL;
    }
    return group_guard(sg, [&] {
        GPMA_CUDA(cudaSetDevice(sg->device));
        NcclApi& nc = nccl();
        cudaStream_t s = group_stream(sg);
        const int W = sg->world;
        const u64 nv = sg->nv, C = sg->chunk;
        sg->x.reserve(nv + 1);
        sg->y.reserve(C + 1);
        sg->gy.reserve(W * C + 1);
        GPMA_CUDA(cudaMemcpyAsync(sg->x.ptr, x, nv * 8, cudaMemcpyHostToDevice, s));
        check_rc(gpma_shard_spmv(sg->g, sg->x.ptr, sg->y.ptr), sg->g);
        GPMA_NCCL(nc.AllGather(sg->y.ptr, sg->gy.ptr, C, ncclFloat64, sg->comm, s));
        for (int r = 0; r < W; ++r)
            GPMA_CUDA(cudaMemcpyAsync(y + sg->bounds[r], sg->gy.ptr + u64(r) * C,
                                      (sg->bounds[r + 1] - sg->bounds[r]) * 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
