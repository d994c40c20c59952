// pma.cu — device-resident PMA and the GPMA+ batch-update pipeline for
// sm_100a (the north-star hot path).
//
// Per batch (segment_engine.hpp:365-470):
//   1. varying-bit mask + key compression, stable radix sort of (key, arrival)
//      (primitives.hpp:21-56)
//   2. duplicate resolution = ordered compaction of run ends
//      (segment_engine.hpp:346-363)
//   3. leaf assignment: binary search of the backward-filled leaf headers
//      (pma.hpp:234-289)
//   4. rounds, level by level (segment_engine.hpp:396-465):
//        group  = ordered compaction of segment heads   (unique_segments)
//        commit = decide + merge + even placement, fused  (try_insert_plus)
//                 warp tier (seg <= 32 slots), CTA tier (larger)
//        advance / touched list = ordered compactions   (advance_round)
//      root path with grow / forced merge / eager shrink on device-wide
//      kernels (segment_engine.hpp:435-463, pma.hpp:390-402, 597-601)
//   5. refresh of leaf headers (+ row offsets for graphs) over touched ranges.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <atomic>
#include <cstdlib>

#include <cooperative_groups.h>

#include "block_ops.cuh"
#include "merge.cuh"
#include "pma_impl.cuh"

namespace gpma {

// ===================================================================== layout

u64 Pma::leaf_size_for(u64 cap) {  // pma.hpp:95-101
    int lg = 0;
    while ((1ull << (lg + 1)) <= cap) ++lg;
    u64 leaf = 4;
    while (leaf * 2 <= u64(lg)) leaf *= 2;
    return leaf;
}

int Pma::height_for(u64 cap, u64 leaf) {
    int h = 0;
    for (u64 s = leaf; s < cap; s <<= 1) ++h;
    return h;
}

u64 Pma::max_at_capacity(u64 cap) const {  // pma.hpp:590-595
    const u64 leaf = leaf_size_for(cap);
    const int h = height_for(cap, leaf);
    const u64 mx0 = u64(std::floor(prof_.leaf_upper * double(leaf) + 1e-9));
    return mx0 << h;
}

static void validate_profile(const pma_profile& d) {  // pma.hpp:59-67
    if (!(d.leaf_lower > 0.0 && d.leaf_lower < d.root_lower && d.root_lower < d.root_upper &&
          d.root_upper < d.leaf_upper && d.leaf_upper < 1.0))
        throw ApiError(PMA_EINVAL, "DensityProfile: need 0 < leaf_lower < root_lower < root_upper < leaf_upper < 1");
    if (2.0 * d.root_lower > d.root_upper + 1e-12)
        throw ApiError(PMA_EINVAL, "DensityProfile: need 2*root_lower <= root_upper so a post-shrink root is legal");
}

Pma::Pma(const pma_profile* profile, int device) : device_(device) {
    prof_ = profile ? *profile : pma_profile{0.08, 0.92, 0.40, 0.80, 1, 0};
    validate_profile(prof_);
    GPMA_CUDA(cudaSetDevice(device_));
    GPMA_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
    stream_ = own_stream_;
    GPMA_CUDA(cudaMalloc(&d_ctr, sizeof(Ctr)));
    GPMA_CUDA(cudaMallocHost(&h_ctr, sizeof(Ctr)));
    GPMA_CUDA(cudaMallocHost(&h_desc_, sizeof(GraphFront)));
    GPMA_CUDA(cudaMalloc(&d_desc_, sizeof(GraphFront)));
    if (const char* e = std::getenv("GPMA_NO_GRAPHS")) small_graphs_ = e[0] == '0';
    if (const char* e = std::getenv("GPMA_NO_BUCKETS")) buckets_ = e[0] == '0';
    if (const char* e = std::getenv("GPMA_NO_PDL")) pdl_ = e[0] == '0';
    static const bool early = [] {  // (this TU's kernels; measured slower at B = 1000)
        const char* e = std::getenv("GPMA_PDL_EARLY");
        const int v = (e && *e) ? std::atoi(e) : 0;
        if (v) GPMA_CUDA(cudaMemcpyToSymbol(g_pdl_early, &v, sizeof(int)));
        return v != 0;
    }();
    (void)early;
    if (const char* e = std::getenv("GPMA_NO_POLL")) small_poll_ = e[0] == '0';
    if (const char* e = std::getenv("GPMA_SMALL_ONECTA")) small_onecta_ = std::strtoull(e, nullptr, 10);
    if (const char* e = std::getenv("GPMA_SMALL_CLUSTER")) small_cluster_ = e[0] != '0';
    if (const char* e = std::getenv("GPMA_CHECK_ROUNDS")) check_rounds_ = e[0] == '1';
    if (const char* e = std::getenv("GPMA_NO_DIRECT_TOUCHED")) direct_touched_ = e[0] == '0';
    for (auto& e : ev_) GPMA_CUDA(cudaEventCreate(&e));
    reset_layout(16);
    headers_closed_form(nullptr, 0);
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

Pma::~Pma() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    free_arrays();
    if (d_ctr) cudaFree(d_ctr);
    if (h_ctr) cudaFreeHost(h_ctr);
    for (auto& x : small_exec_)
        if (x) cudaGraphExecDestroy(x);  // (one per front-end variant)
    if (h_desc_) cudaFreeHost(h_desc_);
    if (d_desc_) cudaFree(d_desc_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : lev_ev_)
        if (e) cudaEventDestroy(e);
    if (own_stream_) cudaStreamDestroy(own_stream_);
}

void Pma::free_arrays() {
    if (d_keys) cudaFree(d_keys);
    if (d_vals) cudaFree(d_vals);
    if (d_st) cudaFree(d_st);
    if (d_hdr) cudaFree(d_hdr);
    d_keys = d_vals = d_hdr = nullptr;
    d_st = nullptr;
}

// reset_layout (pma.hpp:561-567) + rebuild_bounds (pma.hpp:577-588)
void Pma::reset_layout(u64 cap) {
    free_arrays();
    cap_ = cap;
    leaf_ = leaf_size_for(cap);
    height_ = height_for(cap, leaf_);
    GPMA_CUDA(cudaMalloc(&d_keys, cap * 8));
    GPMA_CUDA(cudaMalloc(&d_vals, cap * 8));
    GPMA_CUDA(cudaMalloc(&d_st, cap));
    GPMA_CUDA(cudaMalloc(&d_hdr, (cap / leaf_) * 8));
    GPMA_CUDA(cudaMemsetAsync(d_keys, 0, cap * 8, stream_));
    GPMA_CUDA(cudaMemsetAsync(d_vals, 0, cap * 8, stream_));
    GPMA_CUDA(cudaMemsetAsync(d_st, 0, cap, stream_));
    valid_count = 0;
    tombstone_count = 0;
    const double lf = double(leaf_);
    const u64 mn0 = u64(std::ceil(prof_.leaf_lower * lf - 1e-9));
    const u64 mx0 = u64(std::floor(prof_.leaf_upper * lf + 1e-9));
    for (int l = 0; l <= height_; ++l) {
        mn_[l] = mn0 << l;
        mx_[l] = mx0 << l;
    }
}

void Pma::ensure_slot_scratch() {
    const u64 n = cap_ + 1;
    ek.reserve(n);
    ev.reserve(n);
    ok.reserve(n);
    ov.reserve(n);
    es.reserve(n);
    mb.reserve(n);
    mflag.reserve(n);
}

void Pma::sync_ctr() {
    GPMA_CUDA(cudaMemcpyAsync(h_ctr, d_ctr, sizeof(Ctr), cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

void Pma::event(int idx) { GPMA_CUDA(cudaEventRecord(E(idx), stream_)); }

void Pma::accumulate_timing(const pma_timing& t) {
    pma_timing& a = tsum_;
    a.device_ms += t.device_ms;
    a.sort_ms += t.sort_ms;
    a.search_ms += t.search_ms;
    a.rounds_ms += t.rounds_ms;
    a.refresh_ms += t.refresh_ms;
    a.kernel_launches += t.kernel_launches;
    a.merge_slots += t.merge_slots;
    a.tombstone_flips += t.tombstone_flips;
    a.commit_bytes += t.commit_bytes;
    a.front_end += t.front_end;
    a.grid_merges += t.grid_merges;
    for (int l = 0; l < 16; ++l) {
        a.level_ms[l] += t.level_ms[l];
        a.level_groups[l] += t.level_groups[l];
        a.level_big[l] += t.level_big[l];
        a.level_bytes[l] += t.level_bytes[l];
        a.level_max_slice[l] = std::max(a.level_max_slice[l], t.level_max_slice[l]);
    }
    ++tsum_n_;
}

// stage times of the deferred batch recorded in event set `set`
void Pma::resolve_set(int set) {
    pend_[set] = false;
    const cudaEvent_t* e = ev_ + set * 6;
    GPMA_CUDA(cudaEventSynchronize(e[4]));
    pma_timing& t = pend_t_[set];
    float dev03 = 0, d = 0;
    cudaEventElapsedTime(&dev03, e[0], e[3]);
    cudaEventElapsedTime(&d, e[3], e[4]);
    const float a = float(t.sort_ms), b = float(t.search_ms);  // (from the stage stamps, set at the batch's end)
    const float c = std::max(0.f, dev03 - a - b);
    t.rounds_ms = c;
    t.refresh_ms = d;
    t.device_ms = a + b + c + d;
    accumulate_timing(t);
    if (set == ev_set_ && latest_pending_) {  // still the last batch's record: complete it
        timing.sort_ms = a;
        timing.search_ms = b;
        timing.rounds_ms = c;
        timing.refresh_ms = d;
        timing.device_ms = t.device_ms;
        latest_pending_ = false;
    }
}

// ==================================================================== kernels

// Even placement of k sorted entries over [b, b+m) (pma.hpp:440-467),
// destination-driven so every store is coalesced.
__global__ void k_place_evenly(u64* __restrict__ keys, u64* __restrict__ vals, u8* __restrict__ st, u64 b, u64 m,
                               const u64* __restrict__ ek, const u64* __restrict__ ev, const ull* k_dev, u64 k_host) {
    const u64 k = k_dev ? *k_dev : k_host;
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < m; t += u64(gridDim.x) * blockDim.x) {
        u64 j;
        const bool tgt = placement_target(t, k, m, &j);
        keys[b + t] = tgt ? ek[j] : 0;
        vals[b + t] = tgt ? ev[j] : 0;
        st[b + t] = tgt ? kValid : kEmpty;
    }
}

// Leaf headers of an array that is one even placement of k entries:
// hdr[i] = entry ceil(i*leaf*k/C) (the first entry at or after the leaf).
__global__ void k_headers_closed(u64* hdr, u64 L, u64 leaf, u64 cap, const u64* ek, const ull* k_dev, u64 k_host) {
    const u64 k = k_dev ? *k_dev : k_host;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < L; i += u64(gridDim.x) * blockDim.x) {
        const u64 t = i * leaf;
        const u64 j = k ? (t * k + cap - 1) / cap : 0;
        hdr[i] = (k && j < k) ? ek[j] : ~0ull;
    }
}

__global__ void k_validate_sorted(const u64* keys, u64 n, Ctr* ctr) {
    for (u64 i = 1 + blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        if (keys[i] <= keys[i - 1]) atomicMin(&ctr->bad_index, ull(i));
}

__global__ void k_or_mask(const u64* keys, u64 n, Ctr* ctr) {
    stamp_first(&ctr->t_front);
    const u64 k0 = keys[0];
    u64 acc = 0;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        acc |= keys[i] ^ k0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc |= __shfl_xor_sync(FULL, acc, d);
    if ((threadIdx.x & 31) == 0 && acc) atomicOr(&ctr->mask_or, ull(acc));
}

struct BitRuns {
    int n;
    int lo[16];
    int len[16];
    int out[16];
};

// pext of the varying bits: order-preserving and injective on the batch.
// Payload = arrival index << 1 | is_insert, so duplicate resolution never
// gathers the op.
__global__ void k_compress(const u64* keys, const u8* ops, u64 n, BitRuns runs, u64* ck, u32* ci) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        const u64 k = keys[i];
        u64 c = 0;
        for (int r = 0; r < runs.n; ++r)
            c |= ((k >> runs.lo[r]) & ((runs.len[r] == 64) ? ~0ull : ((1ull << runs.len[r]) - 1))) << runs.out[r];
        ck[i] = c;
        ci[i] = (u32(i) << 1) | (ops[i] == kOpInsert ? 1u : 0u);
    }
}

struct PrepAcc {
    ull guards = 0, bad = 0, oor = 0, bigrun = 0;
};

// leaf of a graph key (pma.hpp:234-289 binary_search_leaf): keys of a vertex
// in the row-offset range are bracketed by its guards' slots first, so the
// header search spans only the leaves of that vertex's run
__device__ __forceinline__ u64 leaf_for_key(u64 key, const u64* __restrict__ hdr, u64 L, const u8* __restrict__ st,
                                            u64 leaf, const u64* __restrict__ ro, u64 rlo, u64 rhi) {
    const u64 u = key >> 32;
    if (ro && u >= rlo && u < rhi && !is_guard(key)) {
        const u64 a = __ldg(&ro[u]), b = __ldg(&ro[u + 1]);
        u64 lo = a ? (a - 1) / leaf : 0;  // hdr[lo] <= guard(u - 1) < key (or lo == 0)
        u64 hi = (b - 1) / leaf + 1;      // hdr[hi] > guard(u) > key (or hi == L)
        if (hi > L) hi = L;
        while (hi - lo > 1) {
            const u64 mid = (lo + hi) >> 1;
            if (__ldg(&hdr[mid]) <= key) lo = mid;
            else hi = mid;
        }
        return lo;
    }
    if (key == ~0ull) return leaf_of_key(hdr, L, st, leaf, key);
    const u64 kk[1] = {key};
    u64 pos[1];
    leaf_search_interleaved<1>(hdr, L, 1u, kk, pos);
    return pos[0];
}

// Leaf-bucket front end (graph batches): each update's leaf is found in
// arrival order and counted (the atomic's return = its ordinal in the
// bucket); bucket L holds the guard deletes.  A bucket reaching kRunMax
// raises `bigrun` (the batch is then redone through the radix sort).
constexpr u32 kRunMax = 1024;
struct BucketArgs {
    const u64* hdr;
    u64 L;
    const u8* st;
    u64 leaf;
    const u64* ro;
    u64 rlo, rhi;
    u32* cnt;  // L + 2 bucket counters (zeroed)
    u32* lf;   // per update: bucket
    u32* od;   // per update: ordinal in the bucket
};

// one update of the graph front end: checks + the compressed key; cls = the
// bucket class: -2 outside the layout (or a guard delete: the batch is redone), else 0
__device__ __forceinline__ u64 prep_code(const GraphFront& f, int db, u32 s, u32 d, u64 i, bool ins, PrepAcc& acc,
                                         int& cls) {
    const u64 lim = 1ull << db;
    bool skip = false;
    if (ins) {
        if (s < f.lo || s >= f.hi || d >= f.nv) acc.bad = max(acc.bad, ~ull(i));  // first offending insert
    } else {
        skip = d == u32(kGuardDst);
        acc.guards += skip;
    }
    u64 c;
    cls = 0;
    if (skip) {
        // a guard delete (graph.hpp:141-147 drops it, counted missed): never
        // in a window stream, so instead of a skip bit that costs every batch
        // a wider sort key, the batch takes the generic redo path, which
        // drops guard deletes before the engine
        c = 0;
        acc.oor = 1;
        cls = -2;
    } else if (s >= lim || d >= lim) {
        c = 0;
        acc.oor |= !ins;
        cls = -2;
    } else {
        c = (u64(s) << db) | d;
    }
    return c;
}

// packed word of a graph update with ib index bits (ib > 0)
__device__ __forceinline__ u64 pack_word(const GraphFront& f, int ib, u64 c, u64 i, bool ins) {
    return (c << ib) | (ins ? (f.opbit ? 0ull : i) : ((1ull << ib) - 1));
}

// checks + the sort input of one update (packed word, or key + payload); returns cls
__device__ __forceinline__ int prep_word(const GraphFront& f, int db, int ib, u64* ck, u32* ci, u64 i, u32 s, u32 d,
                                         bool ins, PrepAcc& acc) {
    int cls;
    const u64 c = prep_code(f, db, s, d, i, ins, acc, cls);
    if (ib) {
        // packed: key above the arrival index for inserts, all-ones for
        // deletes — among equal keys the inserts keep arrival order and the
        // deletes sort after them, which is all duplicate resolution needs
        ck[i] = pack_word(f, ib, c, i, ins);
    } else {
        ck[i] = c;
        ci[i] = (u32(i) << 1) | (ins ? 1u : 0u);
    }
    return cls;
}

// bucket N updates at once: the leaf searches advance in lock-step so each
// step has N independent header loads in flight (unsorted keys: the searches
// miss cache, latency is the cost), then N independent counter atomics.
// (an out-of-layout key only occurs with a bad insert or an oor delete: the
// batch is rejected or redone, its bucket is immaterial)
template <int N>
__device__ __forceinline__ void bucket_n(const BucketArgs& ba, const u64* idx, const u32* s, const u32* d,
                                         const int* cls, PrepAcc& acc) {
    u64 lo[N], hi[N], key[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        key[j] = pack_edge(s[j], d[j]);
        lo[j] = cls[j] == -1 ? ba.L : 0;
        hi[j] = lo[j] + 1;  // settled
        if (cls[j] == 0) {
            const u64 u = s[j];
            if (ba.ro && u >= ba.rlo && u < ba.rhi && !is_guard(key[j])) {
                const u64 a = __ldg(&ba.ro[u]), b = __ldg(&ba.ro[u + 1]);
                lo[j] = a ? (a - 1) / ba.leaf : 0;
                hi[j] = (b - 1) / ba.leaf + 1;
                if (hi[j] > ba.L) hi[j] = ba.L;
            } else {
                lo[j] = leaf_for_key(key[j], ba.hdr, ba.L, ba.st, ba.leaf, ba.ro, ba.rlo, ba.rhi);
                hi[j] = lo[j] + 1;
            }
        }
    }
    for (;;) {  // lock-stepped bisections over hdr
        bool more = false;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (hi[j] - lo[j] > 1) {
                const u64 mid = (lo[j] + hi[j]) >> 1;
                if (__ldg(&ba.hdr[mid]) <= key[j]) lo[j] = mid;
                else hi[j] = mid;
                more |= hi[j] - lo[j] > 1;
            }
        }
        if (!more) break;
    }
    u32 o[N];
#pragma unroll
    for (int j = 0; j < N; ++j) o[j] = atomicAdd(&ba.cnt[lo[j]], 1u);
#pragma unroll
    for (int j = 0; j < N; ++j) {
        ba.lf[idx[j]] = u32(lo[j]);
        ba.od[idx[j]] = o[j];
        acc.bigrun |= o[j] == kRunMax && lo[j] != ba.L;
    }
}

template <bool kBucket>
__device__ __forceinline__ void prep_one(const GraphFront& f, int db, int ib, u64* ck, u32* ci, const BucketArgs& ba,
                                         u64 i, u32 s, u32 d, bool ins, PrepAcc& acc) {
    const int cls = prep_word(f, db, ib, ck, ci, i, s, d, ins, acc);
    if constexpr (kBucket) bucket_n<1>(ba, &i, &s, &d, &cls, acc);
}

// one endpoint-array segment (inserts or deletes): 16-byte vector loads when
// both arrays are aligned alike — the arrays may be page-locked host memory
// read in place over PCIe, where wide requests are what keeps the link busy
template <bool kBucket>
__device__ __forceinline__ void prep_segment(const GraphFront& f, int db, int ib, u64* ck, u32* ci,
                                             const BucketArgs& ba, const u32* sa, const u32* da, u64 n, u64 base,
                                             bool ins, PrepAcc& acc) {
    const u64 tid = blockIdx.x * u64(blockDim.x) + threadIdx.x, nt = u64(gridDim.x) * blockDim.x;
    u64 head = 0;
    if ((reinterpret_cast<uintptr_t>(sa) & 15) == (reinterpret_cast<uintptr_t>(da) & 15) &&
        (reinterpret_cast<uintptr_t>(sa) & 3) == 0) {
        head = ((16 - (reinterpret_cast<uintptr_t>(sa) & 15)) & 15) / 4;
        if (head > n) head = n;
        const u64 nq = (n - head) / 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(sa + head);
        const uint4* d4 = reinterpret_cast<const uint4*>(da + head);
        // the next quad's loads are issued before this quad's leaf searches:
        // read in place over PCIe (pinned host batches) the link stays busy
        // while the searches run
        uint4 na = make_uint4(0, 0, 0, 0), nb = na;
        if (tid < nq) {
            na = s4[tid];
            nb = d4[tid];
        }
        for (u64 q = tid; q < nq; q += nt) {
            const uint4 a = na, b = nb;
            if (q + nt < nq) {
                na = s4[q + nt];
                nb = d4[q + nt];
            }
            const u64 i = base + head + 4 * q;
            const u32 ss[4] = {a.x, a.y, a.z, a.w}, dd[4] = {b.x, b.y, b.z, b.w};
            const u64 ii[4] = {i, i + 1, i + 2, i + 3};
            int cls[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) cls[j] = prep_word(f, db, ib, ck, ci, ii[j], ss[j], dd[j], ins, acc);
            if constexpr (kBucket) bucket_n<4>(ba, ii, ss, dd, cls, acc);
        }
        // scalar head and tail
        for (u64 j = tid; j < head; j += nt) prep_one<kBucket>(f, db, ib, ck, ci, ba, base + j, sa[j], da[j], ins, acc);
        for (u64 j = head + 4 * nq + tid; j < n; j += nt)
            prep_one<kBucket>(f, db, ib, ck, ci, ba, base + j, sa[j], da[j], ins, acc);
        return;
    }
    for (u64 j = tid; j < n; j += nt) prep_one<kBucket>(f, db, ib, ck, ci, ba, base + j, sa[j], da[j], ins, acc);
}

// Graph-mode front end (DynamicGraph::apply_batch, graph.hpp:133-147): check
// insert ids, count guard deletes, and emit the sort input with the
// |V|-derived compressed layout (src << db | dst); guard deletes (dropped by
// the reference before the engine) get key 1 << 2db and sort last.  Payload =
// arrival index << 1 | is_insert — or, when key and index fit one word
// (ib > 0), the single u64 (key << ib | index), sorted keys-only on the key
// bits: LSD radix is stable, so this is the same order at 16 instead of 24
// bytes per element per pass.  A non-guard delete outside the layout raises
// `oor` (the batch is then redone on the generic path).  kBucket: also the
// leaf bucket of every update (leaf-bucket front end, see batch_update_device).
template <bool kBucket>
__device__ __forceinline__ void prep_graph_body(const GraphFront& f, int db, int ib, u64* __restrict__ ck,
                                                u32* __restrict__ ci, Ctr* ctr, const BucketArgs& ba) {
    PrepAcc acc;
    if (f.mk) {
        const u64 n = f.ni + f.nd;
        for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
            const u64 k = f.mk[i];
            prep_one<kBucket>(f, db, ib, ck, ci, ba, i, src_of(k) & 0x7FFFFFFFu, dst_of(k), !(k >> 63), acc);
        }
    } else {
        if (f.ni) prep_segment<kBucket>(f, db, ib, ck, ci, ba, f.is, f.id, f.ni, 0, true, acc);
        if (f.nd) prep_segment<kBucket>(f, db, ib, ck, ci, ba, f.ds, f.dd, f.nd, f.ni, false, acc);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        acc.guards += __shfl_xor_sync(FULL, acc.guards, d);
        acc.bad = max(acc.bad, __shfl_xor_sync(FULL, acc.bad, d));
        acc.oor |= __shfl_xor_sync(FULL, acc.oor, d);
        acc.bigrun |= __shfl_xor_sync(FULL, acc.bigrun, d);
    }
    if ((threadIdx.x & 31) == 0) {
        if (acc.guards) atomicAdd(&ctr->gdel, acc.guards);
        if (acc.bad) atomicMax(&ctr->bad_ins, acc.bad);
        if (acc.oor) atomicOr(&ctr->oor, 1ull);
        if (acc.bigrun) atomicOr(&ctr->bigrun, 1ull);
    }
}
template <bool kBucket>
__global__ void __launch_bounds__(256, kBucket ? 4 : 1) k_prep_graph(GraphFront f, int db, int ib, u64* __restrict__ ck,
                                                                     u32* __restrict__ ci, Ctr* ctr, BucketArgs ba) {
    stamp_first(&ctr->t_front);
    prep_graph_body<kBucket>(f, db, ib, ck, ci, ctr, ba);
}

// In-place ascending sort of buf[0, P) (P a power of two >= 32 E) by the
// A = P / E threads t < A (named barrier 1).  Each warp first sorts its
// contiguous run of 32 E words in registers — item e of a lane is run
// element 32 e + lane, so bitonic partners j < 32 are shuffles and j >= 32
// the lane's own items: no shared memory, no barrier — then runs are merged
// pairwise through shared memory (merge path: each thread finds the split
// of its E consecutive outputs by bisection and merges them), log2(P / 32E)
// rounds.  Words are distinct or identical, so stability is immaterial.
template <int E>
__device__ __forceinline__ void sort_block(u64* buf, u64* xb, u32 t, u32 A, u32 P) {
    constexpr u32 R0 = 32 * E;
    const u32 lane = t & 31, base = (t >> 5) * R0;
    u64 x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = buf[base + 32 * u32(e) + lane];
#pragma unroll
    for (u32 k = 2; k <= R0; k <<= 1) {
#pragma unroll
        for (u32 j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e)
#pragma unroll
                    for (int g = e + 1; g < E; ++g)
                        if (u32(e ^ g) == j / 32) {
                            const u64 lo = min(x[e], x[g]), hi = max(x[e], x[g]);
                            const bool asc = ((32 * u32(e) + lane) & k) == 0;
                            x[e] = asc ? lo : hi;
                            x[g] = asc ? hi : lo;
                        }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const u32 q = 32 * u32(e) + lane;
                    const u64 y = __shfl_xor_sync(FULL, x[e], j);
                    const bool keep_min = ((q & k) == 0) == ((q & j) == 0);
                    x[e] = keep_min ? min(x[e], y) : max(x[e], y);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) buf[base + 32 * u32(e) + lane] = x[e];
    auto bar = [A]() { asm volatile("bar.sync 1, %0;" ::"r"(A) : "memory"); };
    bar();
    u64* src = buf;
    u64* dst = xb;
    for (u32 R = R0; R < P; R <<= 1) {
        const u32 o0 = E * t;
        const u32 ps = o0 & ~(2 * R - 1), d = o0 - ps;
        const u64* Ar = src + ps;
        const u64* Br = Ar + R;
        u32 lo = d > R ? d - R : 0, hi = d < R ? d : R;
        while (lo < hi) {  // first a with A[a] > B[d - a - 1]
            const u32 mid = (lo + hi) >> 1;
            if (Ar[mid] <= Br[d - mid - 1]) lo = mid + 1;
            else hi = mid;
        }
        u32 ia = lo, ib = d - lo;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const bool take_a = ib >= R || (ia < R && Ar[ia] <= Br[ib]);
            dst[o0 + e] = take_a ? Ar[ia++] : Br[ib++];
        }
        bar();
        u64* tmp = src;
        src = dst;
        dst = tmp;
    }
    if (src != buf) {
#pragma unroll
        for (int e = 0; e < E; ++e) buf[E * t + e] = src[E * t + e];
        bar();
    }
}

constexpr int kSmallFrontThreads = 1024;
constexpr int kSmallFrontItems = 4;
constexpr u32 kSmallFrontMax = kSmallFrontThreads * kSmallFrontItems;
constexpr int kSmallFrontSmem = 2 * kSmallFrontMax * 8;  // double-buffered exchange

// Duplicate resolution of a small batch's sorted words ck[0, n) by one CTA of
// kSmallFrontThreads (segment_engine.hpp:346-363): the last word of each
// equal-key run survives; a delete there takes the run's last insert.  Warp
// w owns the words [32 w I, 32 (w + 1) I) (I = kItems per lane, n <= 1024 I),
// read 32 consecutive words at a time (no bank conflicts) and compacted in
// order by ballots; thread 0
// publishes the front end's counters (s_acc: guard deletes, first bad insert,
// out-of-layout delete).
template <int kItems>
__device__ __forceinline__ void small_resolve(const u64* ck, u32 n, const GraphFront& f, int db, int ib, Ctr* ctr,
                                              const ull* s_acc, u64 gt0, u32* s_wsum, u64* __restrict__ o_k,
                                              u64* __restrict__ o_v, u8* __restrict__ o_o) {
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const u64 pmask = (1ull << ib) - 1;
    const u64 skipkey = 1ull << (2 * db);
    const u32 base = warp * (32 * kItems);
    u32 fm[kItems];
    u32 wcnt = 0;
#pragma unroll
    for (int e = 0; e < kItems; ++e) {
        const u32 i = base + 32 * u32(e) + lane;
        bool keep = false;
        if (i < n) {
            const u64 c = ck[i] >> ib;
            keep = ((i + 1 == n) || (ck[i + 1] >> ib) != c) && c < skipkey;
        }
        fm[e] = __ballot_sync(FULL, keep);
        wcnt += __popc(fm[e]);
    }
    if (lane == 0) s_wsum[warp] = wcnt;
    __syncthreads();
    if (warp == 0) {
        u32 w = s_wsum[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(FULL, w, d);
            if (lane >= u32(d)) w += y;
        }
        s_wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    u32 x0 = warp ? s_wsum[warp - 1] : 0u;
    const u32 below = (1u << lane) - 1u;
    const double* gw = f.iw;
#pragma unroll
    for (int e = 0; e < kItems; ++e) {
        if ((fm[e] >> lane) & 1u) {
            const u32 i = base + 32 * u32(e) + lane;
            const u32 x = x0 + __popc(fm[e] & below);
            const u64 c = ck[i] >> ib;
            u64 a = ck[i] & pmask;
            bool ins = a != pmask;
            if (!ins) {  // delete at a run end: any earlier insert of the key wins
                for (long long q = (long long)i - 1; q >= 0 && (ck[q] >> ib) == c; --q) {
                    const u64 aq = ck[q] & pmask;
                    if (aq != pmask) {
                        a = aq;
                        ins = true;
                        break;
                    }
                }
            }
            o_k[x] = ((c >> db) << 32) | (c & ((1ull << db) - 1));
            o_v[x] = ins ? u64(__double_as_longlong(gw ? gw[a] : 1.0)) : 0;
            o_o[x] = ins ? kOpInsert : kOpDelete;
        }
        x0 += __popc(fm[e]);
    }
    if (t == 0) {
        const ull total = s_wsum[kSmallFrontThreads / 32 - 1];
        ctr->nsort = n;
        ctr->gt0 = gt0;
        ctr->seq = f.seq;
        ctr->gdel = s_acc[0];
        ctr->bad_ins = s_acc[1];
        ctr->oor = s_acc[2];
        ctr->n_unique = total;
        ctr->np[0] = (s_acc[1] || s_acc[2]) ? 0ull : total;
    }
}

// Whole front end of a captured small batch in ONE CTA (n <= kSmallFrontMax):
// zero the counters and the graph's look-back words, read the descriptor
// straight from page-locked host memory, pack + check every update
// (prep_code), sort the packed words (sort_block), then resolve duplicates
// and compact the unique updates with a CTA-wide scan — the same output as
// k_prep_graph, the radix sort and the duplicate-resolution compaction of the
// general path, without their launches and the look-back between CTAs.

__global__ void __launch_bounds__(kSmallFrontThreads, 1)
    k_small_front(const GraphFront* __restrict__ hf, int db, int ib, Ctr* ctr, ull* ws_tiles, u64 ws_words,
                  u64* __restrict__ o_k, u64* __restrict__ o_v, u8* __restrict__ o_o) {
    extern __shared__ u64 sbuf[];  // [2][kSmallFrontMax]
    __shared__ u64 s_desc[(sizeof(GraphFront) + 7) / 8];
    __shared__ u32 s_wsum[kSmallFrontThreads / 32];
    __shared__ ull s_acc[4];
    const u32 t = threadIdx.x, lane = t & 31;
    u64 gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    pdl_enter();  // (the chain's head: launched without the attribute, lets the leaf search be scheduled early)
    // descriptor: one word per thread over PCIe; counters + look-back words zeroed
    if (t < (sizeof(GraphFront) + 7) / 8) s_desc[t] = reinterpret_cast<const volatile u64*>(hf)[t];
    for (u32 i = t; i < sizeof(Ctr) / 8; i += kSmallFrontThreads) reinterpret_cast<ull*>(ctr)[i] = 0;
    for (u64 i = t; i < ws_words; i += kSmallFrontThreads) ws_tiles[i] = 0;
    if (t < 4) s_acc[t] = 0;
    __syncthreads();
    const GraphFront& f = *reinterpret_cast<const GraphFront*>(s_desc);
    const u32 n = u32(f.ni + f.nd);
    u32 P = 32;
    while (P < n) P <<= 1;
    // pack: item e of thread t is element t + e * 1024 (coalesced reads); the
    // words go to shared memory, ~0 pads up to P
    PrepAcc acc;
#pragma unroll
    for (int e = 0; e < kSmallFrontItems; ++e) {
        const u32 i = t + u32(e) * kSmallFrontThreads;
        if (i < n) {
            const bool ins = i < f.ni;
            const u32 s = ins ? f.is[i] : f.ds[i - f.ni];
            const u32 d = ins ? f.id[i] : f.dd[i - f.ni];
            int cls;
            sbuf[i] = pack_word(f, ib, prep_code(f, db, s, d, i, ins, acc, cls), i, ins);
        } else if (i < P) {
            sbuf[i] = ~0ull;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        acc.guards += __shfl_xor_sync(FULL, acc.guards, d);
        acc.bad = max(acc.bad, __shfl_xor_sync(FULL, acc.bad, d));
        acc.oor |= __shfl_xor_sync(FULL, acc.oor, d);
    }
    if (lane == 0) {
        if (acc.guards) atomicAdd(&s_acc[0], acc.guards);
        if (acc.bad) atomicMax(&s_acc[1], acc.bad);
        if (acc.oor) atomicOr(&s_acc[2], 1ull);
    }
    __syncthreads();
    // only P / E threads sort (idle warps would take issue slots every stage)
    if (P <= kSmallFrontThreads) {
        if (t < P) sort_block<1>(sbuf, sbuf + kSmallFrontMax, t, P, P);
    } else if (P == 2 * kSmallFrontThreads) {
        sort_block<2>(sbuf, sbuf + kSmallFrontMax, t, kSmallFrontThreads, P);
    } else {
        sort_block<4>(sbuf, sbuf + kSmallFrontMax, t, kSmallFrontThreads, P);
    }
    __syncthreads();
    small_resolve<kSmallFrontItems>(sbuf, n, f, db, ib, ctr, s_acc, gt0, s_wsum, o_k, o_v, o_o);
}

// The same front end over several SMs for small batches of more than
// small_onecta_ updates, where the one-CTA sort is issue-bound (a CTA's
// shuffles and shared-memory bisections at 1024 - 4096 words cost more than
// spreading the work):
//   1. a CTA per 256-update chunk: pack + checks, sort in shared memory;
//   2. merge by rank, in every chunk's CTA: each word's place in the merged
//      order = its index in its chunk + the words below it in every other
//      chunk (a bisection per chunk, equal words ordered by chunk; 4 threads
//      per word, a quarter of the other chunks each), scattered;
//   3. CTA 0: duplicate resolution of the merged words (small_resolve, as in
//      k_small_front); its spare threads clear the counters during 1.
// k_small_front_cluster runs the three stages in one 16-CTA cluster through
// distributed shared memory; k_small_front_grid (where such a cluster cannot
// be resident) in a cooperative grid through L2 scratch sb (u64 words):
// [0, 4096) sorted chunks, [4096, 8192) merged, then 4 words per chunk
// (guard deletes, first bad insert, out-of-layout), the descriptor, its ready
// flag and two grid-barrier counters.  Only chunk 0 reads the descriptor over
// PCIe (concurrent reads of the same host lines from 16 SMs serialise: ~14 µs
// for the last one); the other chunks wait for its device copy.
constexpr u32 kChunk = 256;
constexpr u32 kChunks = kSmallFrontMax / kChunk;
constexpr u32 kSbMerged = kSmallFrontMax;
constexpr u32 kSbPart = 2 * kSmallFrontMax;
constexpr u32 kSbDesc = kSbPart + 4 * kChunks;
constexpr u32 kDescWords = (sizeof(GraphFront) + 7) / 8;
constexpr u32 kSbFlag = kSbDesc + kDescWords;  // + two grid-barrier counters (k_small_front_grid)
constexpr u32 kSbWords = kSbFlag + 3;
static_assert(kDescWords <= 32, "descriptor copied by one warp");

// Cooperative grid: grid barrier after the chunk sort, CTA 0 waits for every
// chunk's scatter, then resets the flag and both counters.
__global__ void __launch_bounds__(kSmallFrontThreads, 1)
    k_small_front_grid(const GraphFront* __restrict__ hf, int db, int ib, u64* __restrict__ sb, Ctr* ctr,
                       ull* ws_tiles, u64 ws_words, u64* __restrict__ o_k, u64* __restrict__ o_v,
                       u8* __restrict__ o_o) {
    __shared__ u64 s[kSmallFrontMax];
    __shared__ u64 s_desc[kDescWords];
    __shared__ u32 s_wsum[kSmallFrontThreads / 32];
    __shared__ u32 s_rank[kChunk];
    __shared__ ull s_acc[3], s_tot[3];
    const u32 t = threadIdx.x, lane = t & 31, c = blockIdx.x;
    ull* flag = reinterpret_cast<ull*>(sb + kSbFlag);
    ull* cnt1 = flag + 1;
    ull* cnt2 = flag + 2;
    u64 gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    pdl_enter();
    if (t < 3) s_acc[t] = 0;
    if (t < kChunk) s_rank[t] = 0;
    if (c == 0) {
        if (t < kDescWords) sb[kSbDesc + t] = s_desc[t] = reinterpret_cast<const volatile u64*>(hf)[t];
        __syncthreads();
        if (t == 0) {
            __threadfence();
            st_volatile(flag, 1ull);
        }
    } else {
        if (t == 0)
            while (ld_volatile(flag) == 0) {
            }
        __syncthreads();
        if (t < kDescWords) s_desc[t] = ld_volatile(reinterpret_cast<const ull*>(sb + kSbDesc + t));
    }
    __syncthreads();
    const GraphFront& f = *reinterpret_cast<const GraphFront*>(s_desc);
    const u32 n = u32(f.ni + f.nd), nch = (n + kChunk - 1) / kChunk;
    if (c >= nch) return;  // (uniform over the CTA; never waited for)
    if (t < kChunk) {
        const u32 i = c * kChunk + t;
        PrepAcc acc;
        u64 w = ~0ull;  // pads sort last
        if (i < n) {
            const bool ins = i < f.ni;
            const u32 su = ins ? f.is[i] : f.ds[i - f.ni];
            const u32 dv = ins ? f.id[i] : f.dd[i - f.ni];
            int cls;
            w = pack_word(f, ib, prep_code(f, db, su, dv, i, ins, acc, cls), i, ins);
        }
        s[t] = w;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            acc.guards += __shfl_xor_sync(FULL, acc.guards, d);
            acc.bad = max(acc.bad, __shfl_xor_sync(FULL, acc.bad, d));
            acc.oor |= __shfl_xor_sync(FULL, acc.oor, d);
        }
        if (lane == 0) {
            if (acc.guards) atomicAdd(&s_acc[0], acc.guards);
            if (acc.bad) atomicMax(&s_acc[1], acc.bad);
            if (acc.oor) atomicOr(&s_acc[2], 1ull);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kChunk) : "memory");
        sort_block<1>(s, s + kChunk, t, kChunk, kChunk);
        sb[i] = s[t];
        if (t < 3) sb[kSbPart + 4 * c + t] = s_acc[t];
    } else if (c == 0) {  // CTA 0's other threads: counters and look-back words
        for (u32 i = t - kChunk; i < sizeof(Ctr) / 8; i += kSmallFrontThreads - kChunk)
            reinterpret_cast<ull*>(ctr)[i] = 0;
        for (u64 i = t - kChunk; i < ws_words; i += kSmallFrontThreads - kChunk) ws_tiles[i] = 0;
    }
    __syncthreads();
    if (t == 0) {  // grid barrier: every chunk sorted
        __threadfence();
        atomicAdd(cnt1, 1ull);
        while (ld_volatile(cnt1) < nch) {
        }
        __threadfence();
    }
    __syncthreads();
    for (u32 i = t; i < nch * kChunk; i += kSmallFrontThreads) s[i] = __ldcg(sb + i);
    __syncthreads();
    {
        const u32 e = t & (kChunk - 1), part = t / kChunk;
        const u64 x = s[c * kChunk + e];
        u32 cnt = 0;
        if (c * kChunk + e < n) {
#pragma unroll
            for (u32 k = 0; k < kChunks / 4; ++k) {
                const u32 q = part + 4 * k;
                if (q < nch && q != c) {
                    const u64* run = s + q * kChunk;
                    const bool le = q < c;  // equal words: earlier chunks first
                    u32 lo = 0;
#pragma unroll
                    for (u32 step = kChunk / 2; step > 0; step >>= 1) {
                        const u64 y = run[lo + step - 1];
                        if (le ? y <= x : y < x) lo += step;
                    }
                    const u64 y = run[lo];
                    if (le ? y <= x : y < x) ++lo;
                    cnt += lo;
                }
            }
            if (cnt) atomicAdd(&s_rank[e], cnt);
        }
        __syncthreads();
        if (t < kChunk && c * kChunk + t < n) sb[kSbMerged + t + s_rank[t]] = x;
    }
    __syncthreads();
    if (t == 0) {
        __threadfence();
        atomicAdd(cnt2, 1ull);
    }
    if (c != 0) return;
    if (t == 0) {  // every chunk's words scattered
        while (ld_volatile(cnt2) < nch) {
        }
        __threadfence();
        *flag = 0;
        *cnt1 = 0;
        *cnt2 = 0;
    }
    __syncthreads();
    for (u32 i = t; i < n; i += kSmallFrontThreads) s[i] = __ldcg(sb + kSbMerged + i);
    if (t < 32) {
        ull g = 0, b = 0, o = 0;
        if (t < nch) {
            g = __ldcg(sb + kSbPart + 4 * t);
            b = __ldcg(sb + kSbPart + 4 * t + 1);
            o = __ldcg(sb + kSbPart + 4 * t + 2);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            g += __shfl_xor_sync(FULL, g, d);
            b = max(b, __shfl_xor_sync(FULL, b, d));
            o |= __shfl_xor_sync(FULL, o, d);
        }
        if (t == 0) {
            s_tot[0] = g;
            s_tot[1] = b;
            s_tot[2] = o;
        }
    }
    __syncthreads();
    small_resolve<kSmallFrontItems>(s, n, f, db, ib, ctr, s_tot, gt0, s_wsum, o_k, o_v, o_o);
}

// The same stages in ONE thread-block cluster of 16 CTAs, exchanging through
// distributed shared memory instead of L2: chunks of kC = 256 words for up to
// kSmallFrontMax updates, 1024 words (the whole CTA) for up to 16384.  CTA 0
// reads the descriptor, the others copy it from CTA 0's shared memory; every
// chunk's sorted words are copied from its CTA's shared memory and the
// merged words stored straight into CTA 0's — for kC = 1024 into CTA 0's
// copy of the chunks (shared memory holds one 16K-word array, not two),
// after a fourth cluster barrier; hardware cluster barriers replace the
// flag and counters (no global round trip between stages).  Chunk size,
// bisections and run loops are compile-time: the runtime-chunk version of
// this kernel measured +2.4 µs at B = 1000.
constexpr u32 kClusterCtas = 16;
constexpr u32 kSmallMultiMax = kClusterCtas * kSmallFrontThreads;
template <u32 kC>
constexpr int cluster_smem() {  // own chunk (x2), all chunks, merged words (kC < 1024: separate)
    return int((2 * kC + (kC < kSmallFrontThreads ? 2 : 1) * kClusterCtas * kC) * 8);
}

template <u32 kC>
__global__ void __launch_bounds__(kSmallFrontThreads, 1)
    k_small_front_cluster(const GraphFront* __restrict__ hf, int db, int ib, Ctr* ctr, ull* ws_tiles, u64 ws_words,
                          u64* __restrict__ o_k, u64* __restrict__ o_v, u8* __restrict__ o_o) {
    namespace cg = cooperative_groups;
    constexpr bool kAlias = kC == kSmallFrontThreads;  // merged words over CTA 0's copy of the chunks
    constexpr u32 kParts = kSmallFrontThreads / kC;     // threads per word in the rank step
    extern __shared__ u64 dyn[];
    u64* s_own = dyn;                                               // [2 kC]: this chunk, sorted in place
    u64* s_all = dyn + 2 * kC;                                      // [16 kC]: every chunk
    u64* s_mrg = kAlias ? s_all : s_all + kClusterCtas * kC;        // [16 kC]: merged words (CTA 0)
    __shared__ u64 s_desc[kDescWords];
    __shared__ u32 s_wsum[kSmallFrontThreads / 32];
    __shared__ u32 s_rank[kC];
    __shared__ ull s_acc[3], s_tot[3];
    __shared__ ull s_part[kClusterCtas * 3];  // CTA 0: every chunk's check partials
    cg::cluster_group cl = cg::this_cluster();
    const u32 t = threadIdx.x, lane = t & 31, c = cl.block_rank();
    u64 gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    pdl_enter();
    if (t < 3) s_acc[t] = 0;
    if (t < kC) s_rank[t] = 0;
    if (c == 0 && t < kDescWords) s_desc[t] = reinterpret_cast<const volatile u64*>(hf)[t];
    cl.sync();  // the descriptor is in CTA 0
    if (c != 0 && t < kDescWords) s_desc[t] = cl.map_shared_rank(s_desc, 0)[t];
    __syncthreads();
    const GraphFront& f = *reinterpret_cast<const GraphFront*>(s_desc);
    const u32 n = u32(f.ni + f.nd), nch = (n + kC - 1) / kC;
    const bool live = c < nch;
    auto clear_counters = [&](u32 from, u32 stride) {  // CTA 0: counters and look-back words
        for (u32 i = from; i < sizeof(Ctr) / 8; i += stride) reinterpret_cast<ull*>(ctr)[i] = 0;
        for (u64 i = from; i < ws_words; i += stride) ws_tiles[i] = 0;
    };
    if (live && t < kC) {
        const u32 i = c * kC + t;
        PrepAcc acc;
        u64 w = ~0ull;  // pads sort last
        if (i < n) {
            const bool ins = i < f.ni;
            const u32 su = ins ? f.is[i] : f.ds[i - f.ni];
            const u32 dv = ins ? f.id[i] : f.dd[i - f.ni];
            int cls;
            w = pack_word(f, ib, prep_code(f, db, su, dv, i, ins, acc, cls), i, ins);
        }
        s_own[t] = w;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            acc.guards += __shfl_xor_sync(FULL, acc.guards, d);
            acc.bad = max(acc.bad, __shfl_xor_sync(FULL, acc.bad, d));
            acc.oor |= __shfl_xor_sync(FULL, acc.oor, d);
        }
        if (lane == 0) {
            if (acc.guards) atomicAdd(&s_acc[0], acc.guards);
            if (acc.bad) atomicMax(&s_acc[1], acc.bad);
            if (acc.oor) atomicOr(&s_acc[2], 1ull);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kC) : "memory");
        sort_block<1>(s_own, s_own + kC, t, kC, kC);
        if (t < 3) cl.map_shared_rank(s_part, 0)[3 * c + t] = s_acc[t];
    } else if (c == 0) {  // CTA 0's other threads clear the counters while the chunk sorts
        clear_counters(t - kC, kSmallFrontThreads - kC);
    }
    if constexpr (kC == kSmallFrontThreads) {  // (no other threads)
        if (c == 0) {
            __syncthreads();
            clear_counters(t, kSmallFrontThreads);
        }
    }
    cl.sync();  // every chunk sorted
    bool mine = false;
    u32 my_r = 0;
    u64 x = 0;
    if (live) {
        for (u32 i = t; i < nch * kC; i += kSmallFrontThreads) {
            const u32 q = i / kC;
            s_all[i] = q == c ? s_own[i - q * kC] : cl.map_shared_rank(s_own, q)[i - q * kC];
        }
        __syncthreads();
        // place in the merged order: index in the chunk + the words below it
        // in every other chunk (kParts threads per word, independent bisections)
        const u32 e = t % kC, part = t / kC;
        x = s_all[c * kC + e];
        if (c * kC + e < n) {
            u32 cnt = 0;
#pragma unroll
            for (u32 k = 0; k < kClusterCtas / kParts; ++k) {
                const u32 q = part + kParts * k;
                if (q < nch && q != c) {
                    const u64* run = s_all + q * kC;
                    const bool le = q < c;  // equal words: earlier chunks first
                    u32 lo = 0;
#pragma unroll
                    for (u32 step = kC / 2; step > 0; step >>= 1) {
                        const u64 y = run[lo + step - 1];
                        if (le ? y <= x : y < x) lo += step;
                    }
                    const u64 y = run[lo];
                    if (le ? y <= x : y < x) ++lo;
                    cnt += lo;
                }
            }
            if (cnt) atomicAdd(&s_rank[e], cnt);
        }
        __syncthreads();
        if (t < kC && c * kC + t < n) {
            mine = true;
            my_r = t + s_rank[t];
        }
        if (!kAlias && mine) cl.map_shared_rank(s_mrg, 0)[my_r] = x;
    }
    if constexpr (kAlias) {
        cl.sync();  // every CTA has read its copy of the chunks: CTA 0's becomes the merged array
        if (mine) cl.map_shared_rank(s_mrg, 0)[my_r] = x;
    }
    cl.sync();  // merged words in CTA 0 (and no CTA reads another's shared memory past here)
    if (c != 0) return;
    if (t < 32) {
        ull g = 0, b = 0, o = 0;
        if (t < nch) {
            g = s_part[3 * t];
            b = s_part[3 * t + 1];
            o = s_part[3 * t + 2];
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            g += __shfl_xor_sync(FULL, g, d);
            b = max(b, __shfl_xor_sync(FULL, b, d));
            o |= __shfl_xor_sync(FULL, o, d);
        }
        if (t == 0) {
            s_tot[0] = g;
            s_tot[1] = b;
            s_tot[2] = o;
        }
    }
    __syncthreads();
    small_resolve<kClusterCtas * kC / kSmallFrontThreads>(s_mrg, n, f, db, ib, ctr, s_tot, gt0, s_wsum, o_k, o_v,
                                                          o_o);
}

static cudaLaunchConfig_t cluster_front_config(cudaStream_t st, cudaLaunchAttribute* at, int smem) {  // 16 CTAs
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(kClusterCtas);
    lc.blockDim = dim3(kSmallFrontThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kClusterCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return lc;
}
template <u32 kC>
static bool cluster_variant_available() {
    static const bool ok = [] {
        if (cudaFuncSetAttribute(k_small_front_cluster<kC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 cluster_smem<kC>()) != cudaSuccess ||
            cudaFuncSetAttribute(k_small_front_cluster<kC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        cudaLaunchAttribute at[1];
        const cudaLaunchConfig_t lc = cluster_front_config(nullptr, at, cluster_smem<kC>());
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k_small_front_cluster<kC>, &lc) != cudaSuccess) {
            cudaGetLastError();
            nc = 0;
        }
        return nc > 0;
    }();
    return ok;
}
static bool cluster_front_available() {
    return cluster_variant_available<256>() && cluster_variant_available<kSmallFrontThreads>();
}

// Leaf of every unique update of a small batch (leaf_for_key), a warp per
// key: each step loads 32 evenly spaced headers of the row's leaf bracket and
// keeps the sub-range the ballot picks, so a bracket of 2^k leaves takes
// ceil(k / 5) dependent loads instead of k (the latency is the cost at this
// size).  Keys outside the row-offset range fall back to one lane's search.
__global__ void __launch_bounds__(256) k_leaf_search_warp(const u64* __restrict__ uk, const ull* n_dev,
                                                         const u64* __restrict__ hdr, u64 L, const u8* __restrict__ st,
                                                         u64 leaf, const u64* __restrict__ ro, u64 rlo, u64 rhi,
                                                         u32* __restrict__ ul) {
    pdl_enter();
    const u64 n = *n_dev;
    const u32 lane = threadIdx.x & 31;
    for (u64 w = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; w < n; w += (u64(gridDim.x) * blockDim.x) >> 5) {
        const u64 key = uk[w];
        const u64 u = key >> 32;
        if (!(ro && u >= rlo && u < rhi && !is_guard(key))) {
            if (lane == 0) ul[w] = u32(leaf_for_key(key, hdr, L, st, leaf, ro, rlo, rhi));
            continue;
        }
        const u64 a = __ldg(&ro[u]), b = __ldg(&ro[u + 1]);
        u64 lo = a ? (a - 1) / leaf : 0;
        u64 hi = (b - 1) / leaf + 1;
        if (hi > L) hi = L;
        while (hi - lo > 1) {  // largest index in [lo, hi) with hdr <= key (as the bisection)
            const u64 m = hi - lo - 1;  // candidates lo + 1 .. hi - 1
            const u64 q = lo + 1 + (m * lane) / 32;
            const unsigned bal = __ballot_sync(FULL, __ldg(&hdr[q]) <= key);
            const int c = __popc(bal);
            const u64 q_lo = lo + 1 + (m * u64(c - 1)) / 32, q_hi = lo + 1 + (m * u64(c)) / 32;
            if (c == 0) hi = lo + 1;
            else {
                lo = q_lo;
                if (c < 32) hi = q_hi;
            }
        }
        if (lane == 0) ul[w] = u32(lo);
    }
}

// bucket scatter: update i -> position off[bucket] + ordinal (bucket order,
// arbitrary order inside a bucket)
// (ci / oci: the arrival payloads when key and index do not fit one word)
__global__ void k_bucket_scatter(const u64* __restrict__ ck, const u32* __restrict__ ci, const u32* __restrict__ lf,
                                 const u32* __restrict__ od, const u32* __restrict__ off, u64 n, u64* __restrict__ out,
                                 u32* __restrict__ oci) {
    pdl_enter();
    // four updates per thread per step: four independent offset lookups in flight
    const u64 nt = u64(gridDim.x) * blockDim.x;
    for (u64 i0 = blockIdx.x * u64(blockDim.x) + threadIdx.x; i0 < n; i0 += 4 * nt) {
        u32 b[4], o[4];
        u64 w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const u64 i = i0 + j * nt;
            if (i < n) {
                b[j] = lf[i];
                o[j] = od[i];
                w[j] = ck[i];
            }
        }
        u64 p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i0 + j * nt < n) p[j] = off[b[j]] + o[j];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i0 + j * nt < n) {
                out[p[j]] = w[j];
                if (ci) oci[p[j]] = ci[i0 + j * nt];
            }
        }
    }
}

// (key word, payload) order of the in-bucket sort: the packed word alone, or
// the key then the arrival payload (index << 1 | is_insert: indices are unique)
__device__ __forceinline__ bool bucket_before(u64 x, u32 xc, u32 xt, u64 w, u32 wc, u32 wt, bool pairs) {
    if (x != w) return x < w;
    if (pairs) return xc < wc;
    return xt < wt;  // identical packed delete words: by position
}

// in-bucket sort by the whole packed word (key, then arrival index): a warp
// takes 32 consecutive buckets, i.e. the contiguous positions
// [off[b0], off[b0 + 32]), one lane per position; a lane finds its bucket
// among the warp's 33 offsets (shuffle binary search) and ranks its word
// among the bucket's (ties — identical delete words — by position).  Buckets
// are short (updates per leaf, ~1 on average); longer ones (> kSmallRun) are
// listed for k_bucket_sort_big.  Also writes each sorted position's leaf (the
// resolve pass emits it).  The guard-delete bucket L holds identical words:
// copied as is.  `out` is the front end's word array, so positions of an
// overflowed bucket (batch redone) keep valid words of this batch.
constexpr u32 kSmallRun = 16;
__global__ void k_bucket_sort_small(const u64* __restrict__ in, const u32* __restrict__ inc,
                                    const u32* __restrict__ off, u64 L, u64* __restrict__ out,
                                    u32* __restrict__ outc, u32* __restrict__ slf, u32* __restrict__ big, Ctr* ctr) {
    pdl_enter();
    const bool pairs = inc != nullptr;
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    const u64 nb = L + 1;  // buckets 0..L (L = guard deletes)
    for (u64 b0 = warp * 32; b0 < nb; b0 += nwarps * 32) {
        const u64 bl = b0 + lane < nb ? b0 + lane : nb;
        const u32 o = off[bl];            // start of bucket b0 + lane (or the end)
        const u32 P1 = __shfl_sync(FULL, off[b0 + 32 < nb ? b0 + 32 : nb], 0);
        const u32 P0 = __shfl_sync(FULL, o, 0);
        const u32 oe = __shfl_down_sync(FULL, o, 1);
        const u32 last_end = lane == 31 ? P1 : oe;  // end of bucket b0 + lane
        // long buckets: their first lane lists them
        if (b0 + lane < nb && last_end - o > kSmallRun && b0 + lane != L)
            big[atomicAdd(&ctr->nbig_buckets, 1ull)] = u32(b0 + lane);
        for (u32 base = P0; base < P1; base += 32) {  // warp-uniform
            const u32 p = base + lane;
            const bool act = p < P1;
            // bucket of p: the largest k with off[b0 + k] <= p
            int k = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const u32 ok = __shfl_sync(FULL, o, k + step);
                if (k + step < 32 && ok <= p) k += step;
            }
            const u32 a = __shfl_sync(FULL, o, k);
            const u32 e = __shfl_sync(FULL, last_end, k);
            if (!act) continue;
            const u64 b = b0 + k;
            slf[p] = u32(b);
            const u64 w = in[p];
            const u32 wc = pairs ? inc[p] : 0u;
            if (e - a == 1 || b == L) {
                out[p] = w;
                if (pairs) outc[p] = wc;
                continue;
            }
            if (e - a > kSmallRun) continue;
            u32 r = 0;
            for (u32 t = a; t < e; ++t) r += bucket_before(in[t], pairs ? inc[t] : 0u, t, w, wc, p, pairs);
            out[a + r] = w;
            if (pairs) outc[a + r] = wc;
        }
    }
}

// the long buckets, one CTA each: staged in shared memory, ranked there
__global__ void __launch_bounds__(256) k_bucket_sort_big(const u64* __restrict__ in, const u32* __restrict__ inc,
                                                         const u32* __restrict__ off, const u32* __restrict__ big,
                                                         const ull* nbig, u64* __restrict__ out,
                                                         u32* __restrict__ outc) {
    pdl_enter();
    __shared__ u64 sm[kRunMax];
    __shared__ u32 smc[kRunMax];
    const bool pairs = inc != nullptr;
    const u64 nb = *nbig;
    for (u64 k = blockIdx.x; k < nb; k += gridDim.x) {
        const u32 b = big[k];
        const u32 a = off[b], len = off[b + 1] - a;
        if (len > kRunMax) continue;  // flagged: the batch is redone
        __syncthreads();
        for (u32 q = threadIdx.x; q < len; q += blockDim.x) {
            sm[q] = in[a + q];
            smc[q] = pairs ? inc[a + q] : 0u;
        }
        __syncthreads();
        for (u32 q = threadIdx.x; q < len; q += blockDim.x) {
            const u64 w = sm[q];
            const u32 wc = smc[q];
            u32 r = 0;
            for (u32 t = 0; t < len; ++t) r += bucket_before(sm[t], smc[t], t, w, wc, q, pairs);
            out[a + r] = w;
            if (pairs) outc[a + r] = wc;
        }
    }
}


__global__ void k_iota(u32* p, const ull* n_dev) {
    const u64 n = *n_dev;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) p[i] = u32(i);
}

__global__ void k_leaf_search(const u64* __restrict__ uk, const ull* n_dev, const u64* __restrict__ hdr, u64 L,
                              const u8* __restrict__ st, u64 leaf, u32* __restrict__ ul) {
    const u64 n = *n_dev;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        ul[i] = u32(leaf_of_key(hdr, L, st, leaf, uk[i]));
}

// Leaf assignment of the sorted unique keys (assign_leaves_sorted,
// pma.hpp:258-289, through the backward-filled headers: last header <= key,
// else 0).  Graph PMAs bracket the answer with the row offsets first: edge
// (u, v) sorts between the guards of u - 1 (slot ro[u] - 1) and u (slot
// ro[u+1] - 1), so its leaf lies in [leaf(ro[u] - 1), leaf(ro[u+1] - 1)] —
// two adjacent loads plus a bisection over the row's few leaves instead of a
// log2(C/16)-level descent.  Other keys (plain PMAs, ids >= |V|) take the
// uniform descent; keys are in order across the warp either way.
__global__ void k_leaf_search_sorted(const u64* __restrict__ uk, const ull* n_dev, const u64* __restrict__ hdr, u64 L,
                                     const u8* __restrict__ st, u64 leaf, const u64* __restrict__ ro, u64 rlo,
                                     u64 rhi, u32* __restrict__ ul) {
    pdl_enter();
    const u64 n = *n_dev;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        ul[i] = u32(leaf_for_key(uk[i], hdr, L, st, leaf, ro, rlo, rhi));
}

// --------------------------------------------------------------- commit args

struct CommitArgs {
    u32* gridlist;  // non-null: merges of this level are handed to the grid tier (Pma::grid_merge)
    u64* t0;     // level 0: one touched word per group (its merge range, or ~0)
    u64* tlist;  // levels >= 1: touched words of merge commits, appended at ctr->ntouched_next
    int cb;      // touched word = (log2(size) << cb) | begin
    u64* keys;
    u64* vals;
    u8* st;
    const u64* uk;
    const u64* uv;
    const u8* uop;
    const u32* ul;
    const u32* pidx;
    const u32* gstart;
    const u32* gseg;
    u8* gflag;
    Ctr* ctr;
    u64* hdr;
    u64* ro;
    u64* rlist;
    u32* biglist;
    int level;
    u64 m;
    u64 leaf;
    u64 mn;
    u64 mx;
    int eager;
    int large;
    int cap_gt_min;
    // CTA-tier scratch (slot space / pending space)
    u64* ek;
    u64* ev;
    u32* es;
    u8* mflag;
    u64* ok;
    u64* ov;
    u64* ik;
    u64* iv;
    u32* ir;
};

struct Acc {
    ull committed = 0, missed = 0, tomb = 0, writes = 0, merge = 0;
    long long vd = 0, td = 0, ed = 0;
    ull bytes = 0;  // algorithmic HBM bytes of the commit (alg_bytes)
};

// Algorithmic bytes of one examined group of an m-slot segment with an
// s-update slice: descriptor (gstart, gseg, gflag) + slice
// (key, value, op) + the segment's states and keys (decision and matching),
// plus 1 B/slot of state writes for tombstone commits or, for merges, the
// values read and keys/values/states written back (25 B/slot).
__device__ __forceinline__ ull alg_bytes(ull m, ull s, int mode) {
    return 9ull + 17ull * s + 9ull * m + (mode == 1 ? m : (mode == 2 ? 25ull * m : 0ull));
}

__device__ __forceinline__ void flush_acc(const Acc& a, Ctr* ctr) {
    // called by one thread per CTA with CTA totals
    if (a.committed) atomicAdd(&ctr->committed, a.committed);
    if (a.missed) atomicAdd(&ctr->missed, a.missed);
    if (a.tomb) atomicAdd(&ctr->tomb_added, a.tomb);
    if (a.writes) atomicAdd(&ctr->slot_writes, a.writes);
    if (a.merge) atomicAdd(&ctr->merge_slots, a.merge);
    if (a.vd) atomicAdd(reinterpret_cast<ull*>(&ctr->valid_delta), ull(a.vd));
    if (a.td) atomicAdd(reinterpret_cast<ull*>(&ctr->tomb_delta), ull(a.td));
    if (a.ed) atomicAdd(reinterpret_cast<ull*>(&ctr->empty_delta), ull(a.ed));
    if (a.bytes) atomicAdd(&ctr->commit_bytes, a.bytes);
}

// level span stamps of the commit kernels (Ctr::lvl_tmin / lvl_tmax)
__device__ __forceinline__ void level_stamp(Ctr* c, int level, bool begin) {
    if (level < 16 && threadIdx.x == 0) {
        u64 g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        if (begin) atomicMax(&c->lvl_tmin[level], ~ull(g));
        else atomicMax(&c->lvl_tmax[level], ull(g));
    }
}

__device__ void block_flush(Acc acc, Ctr* ctr) {
    __shared__ ull s_acc[9];
    if (threadIdx.x < 9) s_acc[threadIdx.x] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        if (acc.committed) atomicAdd(&s_acc[0], acc.committed);
        if (acc.missed) atomicAdd(&s_acc[1], acc.missed);
        if (acc.tomb) atomicAdd(&s_acc[2], acc.tomb);
        if (acc.writes) atomicAdd(&s_acc[3], acc.writes);
        if (acc.merge) atomicAdd(&s_acc[4], acc.merge);
        if (acc.vd) atomicAdd(&s_acc[5], ull(acc.vd));
        if (acc.td) atomicAdd(&s_acc[6], ull(acc.td));
        if (acc.ed) atomicAdd(&s_acc[7], ull(acc.ed));
        if (acc.bytes) atomicAdd(&s_acc[8], acc.bytes);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Acc t;
        t.committed = s_acc[0];
        t.missed = s_acc[1];
        t.tomb = s_acc[2];
        t.writes = s_acc[3];
        t.merge = s_acc[4];
        t.vd = (long long)s_acc[5];
        t.td = (long long)s_acc[6];
        t.ed = (long long)s_acc[7];
        t.bytes = s_acc[8];
        flush_acc(t, ctr);
    }
}

// ------------------------------------------------------------- warp tier
// One warp per group, segment <= 32 slots (leaf and level-1 segments carry
// >= 99.5% of commits).  Slot t of the segment lives in lane t;
// the (typically 1-3) updates of the group are broadcast one by one and
// ranked against the segment with two ballots, so a group costs O(|slice|)
// warp instructions.  Inserts keep their merged position in lane p; survivors
// take the remaining positions in order (__fns over the free-position mask).
// Decision, merge, even re-dispatch and — when every leaf of the rewritten
// segment is non-empty — the leaf-header and row-offset refresh are fused, so
// each slot is read once and written once (128-B key/value lines per leaf).
constexpr int kWarpTierWarps = 8;

__device__ __forceinline__ void warp_reduce_acc(Acc& acc) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        acc.committed += __shfl_xor_sync(FULL, acc.committed, d);
        acc.missed += __shfl_xor_sync(FULL, acc.missed, d);
        acc.tomb += __shfl_xor_sync(FULL, acc.tomb, d);
        acc.writes += __shfl_xor_sync(FULL, acc.writes, d);
        acc.merge += __shfl_xor_sync(FULL, acc.merge, d);
        acc.vd += __shfl_xor_sync(FULL, acc.vd, d);
        acc.td += __shfl_xor_sync(FULL, acc.td, d);
        acc.ed += __shfl_xor_sync(FULL, acc.ed, d);
        acc.bytes += __shfl_xor_sync(FULL, acc.bytes, d);
    }
}

// Group descriptors for a tile of 32 groups, one per lane (one coalesced
// round trip instead of one dependent load chain per group).
__device__ __forceinline__ void load_group_tile(const CommitArgs& a, ull g0, ull ngroups, unsigned lane, u32& t_lo,
                                                u32& t_hi, u32& t_seg) {
    const ull gl = g0 + lane;
    t_lo = t_hi = t_seg = 0;
    if (gl < ngroups) {
        t_lo = a.gstart[gl];
        t_hi = a.gstart[gl + 1];
        t_seg = a.gseg[gl];
    }
}

// --- leaf tier: thread per group, 16-slot segments (>= 99.5% of commits).
// The warp stages the 32 leaves of its group tile in shared memory with
// coalesced 16-byte loads (8 lanes per 128-byte key/value line); each thread
// then commits its own leaf with branch-light bit arithmetic instead of a
// serial merge walk:
//   * every update of the slice is ranked against the 16 slot keys (held in
//     registers) by 16 unrolled 64-bit compares -> lt mask; the only possible
//     match is the first non-Empty slot not below it (non-Empty keys of a leaf
//     are strictly increasing);
//   * deletes hit -> del mask, inserts hit -> overwrite mask; an insert's
//     final rank is popc(kept & lt) + #inserts before it (updates are sorted,
//     so every earlier drop/overwrite below it is already known), and every
//     slot at or above it gets +1 in a nibble-packed "inserts below" counter;
//   * survivor i lands on floor(16 j_i / k) with j_i = popc(kept below i) +
//     nibble_i (commit_in_place / place_evenly give the same layout,
//     segment_engine.hpp:147-230, pma.hpp:440-467): the division is a
//     multiply by ceil(2^16 / k), exact for 16 j <= 240;
//   * the row is permuted in place: survivors moving right in decreasing
//     source order, then survivors moving left in increasing order (the
//     placement is monotone, so neither pass reads a clobbered slot), vacated
//     slots cleared, inserts written last.
// Leaf header, row offsets of moved guards and the state bytes are refreshed
// in the same pass and the warp stores the rewritten leaves back coalesced.
// Groups with more than kBigSlice updates (RMAT hub rows) are handed to the
// CTA kernel through `biglist`.
constexpr int kLeafWarps = 4;
#ifndef GPMA_LEAF_CTAS
#define GPMA_LEAF_CTAS 6  // resident CTAs per SM the register budget is sized for
#endif
constexpr u32 kBigSlice = 32;   // leaf kernel: larger slices go to the CTA kernel
constexpr u32 kLaneBig = 64;    // lane kernels: larger slices go to the CTA kernel
constexpr u32 kStage = 64;      // updates of a 32-group tile staged in smem (overflow read from HBM)

// bit i of m (i < 16) -> bit 4i
__device__ __forceinline__ u64 spread_nibbles(u32 m) {
    u64 x = m & 0xffffu;
    x = (x | (x << 24)) & 0x000000FF000000FFull;
    x = (x | (x << 12)) & 0x000F000F000F000Full;
    x = (x | (x << 6)) & 0x0303030303030303ull;
    x = (x | (x << 3)) & 0x1111111111111111ull;
    return x;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(unsigned(__cvta_generic_to_shared(smem))),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(unsigned(__cvta_generic_to_shared(smem))),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(unsigned(__cvta_generic_to_shared(smem))),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// touched range of a merge commit (update_stats.hpp touched_ranges), as one
// sortable word (log2(size) << cb) | begin.  Level 0 (>= 99.5% of them) writes
// one word per GROUP at the group's index — groups are in ascending segment
// order, so an ordered compaction yields them in the reference's order with
// no sort and no shared counter; higher levels append (see touched_ranges).
__device__ __forceinline__ u64 touched_word(const CommitArgs& a, u64 b, u64 m) {
    return (u64(63 - __clzll(m)) << a.cb) | b;
}
// level >= 1 (a few hundred groups at most): appended in any order, sorted
// at fetch time
__device__ __forceinline__ void touched_append(const CommitArgs& a, u64 b, u64 e) {
    const ull slot = atomicAdd(&a.ctr->ntouched_next, 1ull);
    a.tlist[slot] = touched_word(a, b, e - b);
}

// Only launched at level 0 (m == leaf == 16), where the pending list is the
// identity (a.pidx == nullptr): a tile's updates are one contiguous range.
// Staging is asynchronous (cp.async, no registers held): phase 1 brings the
// tile's states, keys and update slice in one round trip; the decision then
// issues phase 2 (values of the merge groups only), which overlaps the
// ranking of the slices.
// Staged rows are 16 slots (128 B) with their 16-byte chunks XOR-swizzled by
// the row (chunk c of row r lives at chunk c ^ (r & 7)): the same bank spread
// as a padded row, without the pad — 4 KB less shared memory per CTA, which
// with u32 segment ids and <= 80 registers fits 6 CTAs (24 warps) per SM.
// (for i < 16, flipping bits 1-3 of i by the row's low 3 bits is exactly the
// chunk XOR; bit 0 — the word inside a 16-byte chunk — stays)
__device__ __forceinline__ u32 swz(u32 row, u32 i) { return row * 16u + (i ^ ((row & 7u) << 1)); }

__global__ void __launch_bounds__(kLeafWarps * 32, GPMA_LEAF_CTAS) k_commit_leaf(CommitArgs a) {
    __shared__ __align__(16) u64 s_k[kLeafWarps][32 * 16];
    __shared__ __align__(16) u64 s_v[kLeafWarps][32 * 16];
    __shared__ u64 s_uk[kLeafWarps][kStage];
    __shared__ u64 s_uv[kLeafWarps][kStage];
    __shared__ u32 s_uo[kLeafWarps][kStage / 4 + 2];
    __shared__ u32 s_b[kLeafWarps][32];  // segment (= leaf) of each group of the tile
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    u64* const rowk = &s_k[w][lane * 16];
    u64* const rowv = &s_v[w][lane * 16];
    const u32 rx = (lane & 7u) << 1;
    auto RK = [=](u32 i) -> u64& { return rowk[i ^ rx]; };  // slot i of this lane's leaf
    auto RV = [=](u32 i) -> u64& { return rowv[i ^ rx]; };
    const u8* s_op = reinterpret_cast<const u8*>(&s_uo[w][0]);
    pdl_enter();
    level_stamp(a.ctr, a.level, true);
    const ull ngroups = a.ctr->ngroups;
    // tiles handed out dynamically (one counter per launch): tiles differ in
    // cost (merges vs tombstone flips vs deferrals), a static stride left
    // warps idle at the end of the launch
    auto grab = [&]() -> ull {
        ull t = 0;
        if (lane == 0) t = atomicAdd(&a.ctr->leaf_tiles, 1ull);
        return __shfl_sync(FULL, t, 0) * 32;
    };
    ull g0 = grab();
    ull gnext = 0;
    // descriptors of the first tile; each iteration prefetches the next tile's
    u32 n_lo = 0, n_hi = 0, n_seg = 0;
    if (g0 + lane < ngroups) {
        n_lo = a.gstart[g0 + lane];
        n_hi = a.gstart[g0 + lane + 1];
        n_seg = a.gseg[g0 + lane];
    }
    Acc acc;
    for (; g0 < ngroups; g0 = gnext) {
        const ull gl = g0 + lane;
        const bool act = gl < ngroups;
        const u32 lo = n_lo, hi = n_hi;
        const u64 b = u64(n_seg) * 16;
        const unsigned tile_n = (ngroups - g0) < 32 ? unsigned(ngroups - g0) : 32u;
        const u32 tlo = __shfl_sync(FULL, lo, 0);
        const u32 thi = __shfl_sync(FULL, hi, tile_n - 1);
        s_b[w][lane] = n_seg;
        __syncwarp();
        // ---- phase 1: states, keys, update slice of the tile
        uint4 sv = make_uint4(0, 0, 0, 0);
        if (act) sv = *reinterpret_cast<const uint4*>(a.st + b);  // in flight with the copies
        const u32 staged = (thi - tlo) < kStage ? (thi - tlo) : kStage;
        for (u32 i = lane; i < staged; i += 32) {
            cp_async8(&s_uk[w][i], a.uk + tlo + i);
            cp_async8(&s_uv[w][i], a.uv + tlo + i);
        }
        {
            const u32 w0 = tlo >> 2, w1 = (tlo + staged + 3) >> 2;
            for (u32 i = lane; i < w1 - w0; i += 32)
                cp_async4(&s_uo[w][i], reinterpret_cast<const u32*>(a.uop) + w0 + i);
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) {  // 8 lanes per 128-byte key line
            const unsigned row = it * 4 + (lane >> 3), part = lane & 7u;
            if (row < tile_n) cp_async16(&s_k[w][swz(row, 2 * part)], a.keys + u64(s_b[w][row]) * 16 + 2 * part);
        }
        // descriptors of the next tile while the copies fly
        gnext = grab();
        {
            const ull gn = gnext + lane;
            n_lo = n_hi = n_seg = 0;
            if (gn < ngroups) {
                n_lo = a.gstart[gn];
                n_hi = a.gstart[gn + 1];
                n_seg = a.gseg[gn];
            }
        }
        cp_async_wait_all();
        __syncwarp();
        const u32 s = hi - lo;
        const u32 soff = lo - tlo;
        const u32 obase = tlo & 3u;
        auto U = [&](u32 q, u64& key, u8& op) {
            const u32 i = soff + q;
            if (i < staged) {
                key = s_uk[w][i];
                op = s_op[obase + i];
            } else {
                key = a.uk[lo + q];
                op = a.uop[lo + q];
            }
        };
        auto UVAL = [&](u32 q) -> u64 {
            const u32 i = soff + q;
            return i < staged ? s_uv[w][i] : a.uv[lo + q];
        };
        // state masks (bit i = slot i)
        unsigned valid = 0, nonempty = 0;
        if (act) {
            const u32 words[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u32 x = words[q];
                const u32 v1 = x & 0x01010101u;             // state 1 = Valid
                const u32 ne = (x | (x >> 1)) & 0x01010101u; // non-zero byte
                valid |= ((v1 * 0x01020408u) >> 24 & 0xfu) << (4 * q);
                nonempty |= ((ne * 0x01020408u) >> 24 & 0xfu) << (4 * q);
            }
        }
        const unsigned nv = __popc(valid);
        int mode = 0;  // 0 defer, 1 tombstones, 2 merge, 3 big slice (CTA kernel)
        u32 ins = 0;
        if (act) {
            if (s > kBigSlice) {
                mode = 3;
            } else {
                // op bytes are 0 (insert) / 1 (delete): deletes = popc of the
                // slice's op words (masked at both ends)
                static_assert(kOpInsert == 0 && kOpDelete == 1, "op encoding");
                u32 dels = 0;
                if (soff + s <= staged) {
                    const u32 st0 = obase + soff, st1 = st0 + s;
                    for (u32 wd = st0 >> 2; wd < (st1 + 3) >> 2; ++wd) {
                        u32 x = s_uo[w][wd];
                        if (wd == (st0 >> 2)) x &= 0xffffffffu << (8 * (st0 & 3u));
                        if (wd == ((st1 - 1) >> 2) && (st1 & 3u)) x &= 0xffffffffu >> (8 * (4 - (st1 & 3u)));
                        dels += __popc(x);
                    }
                } else {
                    for (u32 q = 0; q < s; ++q) {
                        const u32 i = soff + q;
                        dels += (i < staged ? s_op[obase + i] : a.uop[lo + q]) == kOpDelete;
                    }
                }
                ins = s - dels;
                if (!a.eager && ins == 0) mode = 1;
                else if (!(nv + ins > a.mx || (a.eager && a.cap_gt_min && u64(nv) < u64(dels) + a.mn))) mode = 2;
            }
        }
        // ---- phase 2: values of the merge groups (overlaps the ranking)
        const unsigned mergemask = __ballot_sync(FULL, mode == 2);
        if (mergemask) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const unsigned row = it * 4 + (lane >> 3), part = lane & 7u;
                if ((mergemask >> row) & 1u)
                    cp_async16(&s_v[w][swz(row, 2 * part)], a.vals + u64(s_b[w][row]) * 16 + 2 * part);
            }
        }
        unsigned newvalid = valid, tombs = 0;
        u32 missed = 0, del_hit = 0, moves = 0, k = 0;
        u32 ovr = 0, nins = 0, guards = 0;
        u64 cnt = 0, insj = 0;
        if (mode == 1 || mode == 2) {
            // ---- rank the slice against the leaf (commit_tombstones /
            // merge_entries, segment_engine.hpp:119-137, 285-310)
            u64 K[16];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {  // 16-B row reads: conflict-free per quarter warp
                const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(&RK(i));
                K[i] = kk.x;
                K[i + 1] = kk.y;
            }
            if (mode == 2 && a.ro) {
#pragma unroll
                for (int i = 0; i < 16; ++i) guards |= (u32(K[i]) == u32(kGuardDst) ? 1u : 0u) << i;
            }
            for (u32 q = 0; q < s; ++q) {
                u64 u;
                u8 op;
                U(q, u, op);
                u32 lt = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) lt |= (K[i] < u ? 1u : 0u) << i;
                const u32 cm = nonempty & ~lt;
                const int c = __ffs(cm) - 1;  // the only slot that can hold u
                const bool hit = cm != 0 && ((valid >> c) & 1u) && RK(c) == u;
                if (op == kOpDelete) {
                    if (hit) del_hit |= 1u << c;
                    else ++missed;
                } else {
                    if (hit) ovr |= 1u << c;
                    const u32 j = __popc(valid & ~(del_hit | ovr) & lt) + nins;
                    insj |= u64(j) << (4 * nins);
                    cnt += spread_nibbles(~lt);
                    ++nins;
                }
            }
        }
        cp_async_wait_all();
        __syncwarp();
        if (mode == 1) {
            newvalid = valid & ~del_hit;
            tombs = nonempty & ~newvalid;
        } else if (mode == 2) {
            const u32 keepa = valid & ~del_hit;
            const u32 keepf = keepa & ~ovr;
            k = __popc(keepf) + nins;
            const int tz = __ffs(~keepa) - 1;  // <= 16
            moves = __popc(keepa & (0xffffffffu << tz));
            const u32 mk = k ? (65536u + k - 1) / k : 0u;
            // destinations of the survivors (nibble-packed)
            u64 dst = 0;
            u32 right = 0, out = 0;
            for (u32 m = keepf; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const u32 j = __popc(keepf & ((1u << i) - 1u)) + u32((cnt >> (4 * i)) & 0xfu);
                const u32 x = (j * 16u * mk) >> 16;
                dst |= u64(x) << (4 * i);
                out |= 1u << x;
                if (x > u32(i)) right |= 1u << i;
            }
            for (u32 m = right; m; m &= ~(1u << (31 - __clz(m)))) {
                const int i = 31 - __clz(m);
                const u32 x = u32(dst >> (4 * i)) & 0xfu;
                RK(x) = RK(i);
                RV(x) = RV(i);
            }
            for (u32 m = keepf & ~right; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const u32 x = u32(dst >> (4 * i)) & 0xfu;
                if (x != u32(i)) {
                    RK(x) = RK(i);
                    RV(x) = RV(i);
                }
            }
            for (u32 m = nonempty & ~out; m; m &= m - 1) {
                const int x = __ffs(m) - 1;
                RK(x) = 0;
                RV(x) = 0;
            }
            // inserts, in key order
            u32 nth = 0;
            for (u32 q = 0; nth < nins; ++q) {
                u64 u;
                u8 op;
                U(q, u, op);
                if (op == kOpDelete) continue;
                const u32 j = u32(insj >> (4 * nth)) & 0xfu;
                const u32 x = (j * 16u * mk) >> 16;
                RK(x) = u;
                RV(x) = UVAL(q);
                out |= 1u << x;
                ++nth;
            }
            newvalid = out;
            // row offsets: every guard of the rewritten leaf (graph.hpp:176)
            for (u32 m = keepf & guards; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                const u32 x = u32(dst >> (4 * i)) & 0xfu;
                a.ro[src_of(RK(x)) + 1] = b + x + 1;
            }
        }
        __syncwarp();
        // write back: states (own leaf), keys/values (merge groups, coalesced)
        if (mode == 1 || mode == 2) {
            // 4 mask bits -> 4 bytes (bit i -> bit 0 of byte i) by one multiply;
            // Valid = 1, Tombstone = 2 (newvalid and tombs are disjoint)
            static_assert(kValid == 1 && kTombstone == 2 && kEmpty == 0, "state encoding");
            auto bytes4 = [](u32 m) { return ((m & 0xfu) * 0x00204081u) & 0x01010101u; };
            uint4 ns;
            ns.x = bytes4(newvalid) | (bytes4(tombs) << 1);
            ns.y = bytes4(newvalid >> 4) | (bytes4(tombs >> 4) << 1);
            ns.z = bytes4(newvalid >> 8) | (bytes4(tombs >> 8) << 1);
            ns.w = bytes4(newvalid >> 12) | (bytes4(tombs >> 12) << 1);
            *reinterpret_cast<uint4*>(a.st + b) = ns;
        }
        if (mergemask) {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const unsigned grp = it * 4 + (lane >> 3), part = lane & 7u;
                if ((mergemask >> grp) & 1u) {
                    const u64 gb = u64(s_b[w][grp]) * 16;
                    *reinterpret_cast<ulonglong2*>(a.keys + gb + 2 * part) =
                        *reinterpret_cast<const ulonglong2*>(&s_k[w][swz(grp, 2 * part)]);
                    *reinterpret_cast<ulonglong2*>(a.vals + gb + 2 * part) =
                        *reinterpret_cast<const ulonglong2*>(&s_v[w][swz(grp, 2 * part)]);
                }
            }
        }
        if (mode == 2) {
            if (k > 0) a.hdr[b / 16] = RK(0);  // entry 0 always lands on slot 0
            else {
                const ull slot = atomicAdd(&a.ctr->nrefresh, 1ull);
                a.rlist[2 * slot] = b;
                a.rlist[2 * slot + 1] = b + 16;
            }
        }
        // touched word of the group (level 0: dense by group index; a hub
        // group's word is written again by the CTA kernel)
        if (act) a.t0[gl] = mode == 2 ? touched_word(a, b, 16) : ~0ull;
        if (act) {
            a.gflag[gl] = u8(mode == 3 ? 0 : mode);
            if (mode != 3) acc.bytes += alg_bytes(16, s, mode);
            if (mode == 3) {
                const ull slot = atomicAdd(&a.ctr->nbig, 1ull);
                a.biglist[slot] = u32(gl);
            } else if (mode == 1) {
                const u32 added = __popc(del_hit);
                acc.committed++;
                acc.tomb += added;
                acc.missed += missed;
                acc.writes += added;
                acc.vd -= added;
                acc.td += added;
            } else if (mode == 2) {
                acc.committed++;
                acc.missed += missed;
                acc.writes += 16 + (a.large ? moves : 0u);
                acc.merge += 16;
                acc.vd += (long long)k - (long long)nv;
                acc.td -= __popc(nonempty & ~valid);
                acc.ed += (k == 0 ? 1 : 0) - (nonempty == 0 ? 1 : 0);
            }
        }
        __syncwarp();  // smem of this tile is reused by the next
    }
    warp_reduce_acc(acc);
    if ((threadIdx.x & 31u) != 0) acc = Acc{};
    block_flush(acc, a.ctr);
    level_stamp(a.ctr, a.level, false);
}

// --- warp tiers.  G = 16 (half-warp per group: leaf-level segments, two
// groups per warp) or G = 32 (full warp: level-1 segments).  Lane hl of a
// group owns slot hl of its segment (keys, values, state in registers).
// Updates are ranked lane-parallel, G at a time: each lane binary-searches its
// update among the segment's Valid keys (the r-th Valid key sits in lane
// __fns(valid, 0, r+1)), so a group costs O(|slice| / G) warp iterations even
// for hub rows with thousands of updates.  Every ballot / shuffle runs on all
// 32 lanes and is split per group, so the two half-warp groups never diverge
// around a warp collective.  Outcomes: tombstone flips, merge + even
// re-dispatch with fused leaf-header / row-offset refresh, or deferral.
template <int G>
__global__ void __launch_bounds__(kWarpTierWarps * 32, 4) k_commit_lanes(CommitArgs a) {
    static_assert(G == 16 || G == 32, "group width");
    constexpr unsigned GM = G == 32 ? 0xffffffffu : 0xffffu;
    constexpr int kSearch = G == 32 ? 6 : 5;
    __shared__ u64 s_ok[kWarpTierWarps][32], s_ov[kWarpTierWarps][32];
    __shared__ u64 s_ik[kWarpTierWarps][32], s_iv[kWarpTierWarps][32];
    __shared__ u64 s_vk[kWarpTierWarps][32];             // Valid keys of the segment, compacted
    __shared__ unsigned char s_vl[kWarpTierWarps][32];   // their lanes
    __shared__ unsigned char s_ir[kWarpTierWarps][32];   // insert p: # Valid keys below it
    pdl_enter();
    level_stamp(a.ctr, a.level, true);
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const unsigned hb = G == 32 ? 0u : (lane & 16u), hl = lane & unsigned(G - 1);
    const ull ngroups = a.ctr->ngroups;
    const unsigned m = unsigned(a.m);
    const unsigned leaf = unsigned(a.leaf);
    const unsigned nleaves = m / leaf;
    const unsigned leafmask = (leaf >= 32) ? 0xffffffffu : ((1u << leaf) - 1u);
    const unsigned below = (1u << hl) - 1u;  // lanes of my group below me (hl < 32)
    Acc acc;
    // groups per warp tile (<= 32), from the device-side group count: small
    // rounds spread over many warps (one group each), big ones pack 32
    unsigned T = unsigned((ngroups + 148 * 32 - 1) / (148 * 32));
    T = T < 1 ? 1 : (T > 32 ? 32 : T);
    if (G == 16) T = (T + 1) & ~1u;  // half-warp tier handles pairs
    for (ull g0 = (ull(blockIdx.x) * kWarpTierWarps + w) * T; g0 < ngroups; g0 += ull(gridDim.x) * kWarpTierWarps * T) {
        u32 t_lo = 0, t_hi = 0, t_seg = 0;
        if (lane < T) load_group_tile(a, g0, ngroups, lane, t_lo, t_hi, t_seg);
        const u32 t_gid = u32(g0 + lane);
        const unsigned tile_n = (ngroups - g0) < T ? unsigned(ngroups - g0) : T;
        for (unsigned j = 0; j < tile_n; j += 32 / G) {
            const unsigned gi = j + (hb >> 4);
            const bool act = gi < tile_n;
            const u32 lo = __shfl_sync(FULL, t_lo, gi & 31u);
            const u32 hi = __shfl_sync(FULL, t_hi, gi & 31u);
            const u32 sv = __shfl_sync(FULL, t_seg, gi & 31u);
            const u32 sfull = act ? hi - lo : 0u;
            const bool big = sfull > kLaneBig;  // hub group: CTA kernel takes it
            const u32 s = big ? 0u : sfull;
            const u64 b = u64(sv) * m;
            u8 stt = kEmpty;
            u64 key = 0, val = 0;
            if (act && !big && hl < m) {
                stt = a.st[b + hl];
                key = a.keys[b + hl];
                val = a.vals[b + hl];
            }
            u64 ck = 0, cv = 0;
            u8 co = kOpDelete;
            if (hl < s) {
                const u32 pi = a.pidx ? a.pidx[lo + hl] : lo + hl;
                ck = a.uk[pi];
                co = a.uop[pi];
                cv = a.uv[pi];
            }
            const unsigned valid = (__ballot_sync(FULL, stt == kValid) >> hb) & GM;
            const unsigned nonempty = (__ballot_sync(FULL, stt != kEmpty) >> hb) & GM;
            const unsigned nv = __popc(valid);
            unsigned ins = __popc((__ballot_sync(FULL, hl < s && co == kOpInsert) >> hb) & GM);
            const u32 smax = __reduce_max_sync(FULL, s);
            for (u32 c = G; c < smax; c += G) {
                bool isins = false;
                if (c + hl < s) isins = a.uop[a.pidx ? a.pidx[lo + c + hl] : lo + c + hl] == kOpInsert;
                ins += __popc((__ballot_sync(FULL, isins) >> hb) & GM);
            }
            const u32 dels = s - ins;
            int mode = 0;  // 0 defer, 1 tombstones, 2 merge
            if (act && !big) {
                if (!a.eager && ins == 0) mode = 1;
                else if (!(nv + ins > a.mx || (a.eager && a.cap_gt_min && u64(nv) < u64(dels) + a.mn))) mode = 2;
            }
            unsigned hits = 0, mdel = 0, missed = 0, nins = 0;
            const unsigned vrank = __popc(valid & below);
            if ((valid >> hl) & 1u) {
                s_vk[w][hb + vrank] = key;
                s_vl[w][hb + vrank] = (unsigned char)hl;
            }
            __syncwarp();
            if (__any_sync(FULL, mode != 0)) {
                for (u32 c = 0; c < smax; c += G) {
                    if (c > 0) {
                        ck = cv = 0;
                        co = kOpDelete;
                        if (mode != 0 && c + hl < s) {
                            const u32 pi = a.pidx ? a.pidx[lo + c + hl] : lo + c + hl;
                            ck = a.uk[pi];
                            co = a.uop[pi];
                            cv = a.uv[pi];
                        }
                    }
                    const bool in = mode != 0 && c + hl < s;
                    // rank of my update among the Valid keys (binary search in smem)
                    unsigned rlo = 0, rhi = nv;
#pragma unroll
                    for (int it = 0; it < kSearch; ++it) {
                        if (rlo < rhi) {
                            const unsigned mid = (rlo + rhi) >> 1;
                            if (s_vk[w][hb + mid] < ck) rlo = mid + 1;
                            else rhi = mid;
                        }
                    }
                    const bool hit = in && rlo < nv && s_vk[w][hb + rlo] == ck;
                    const bool isins = in && co == kOpInsert;
                    const unsigned hitbit = hit ? (1u << (unsigned(s_vl[w][hb + rlo]) + hb)) : 0u;
                    hits |= (__reduce_or_sync(FULL, hitbit) >> hb) & GM;
                    mdel |= (__reduce_or_sync(FULL, (hit && !isins) ? hitbit : 0u) >> hb) & GM;
                    missed += __popc((__ballot_sync(FULL, in && !isins && !hit) >> hb) & GM);
                    const unsigned im = (__ballot_sync(FULL, isins) >> hb) & GM;
                    if (isins && mode == 2) {
                        const unsigned p = nins + __popc(im & below);
                        s_ik[w][hb + p] = ck;
                        s_iv[w][hb + p] = cv;
                        s_ir[w][hb + p] = (unsigned char)rlo;
                    }
                    nins += __popc(im);
                }
            }
            __syncwarp();
            if (mode == 1 && ((hits >> hl) & 1u)) a.st[b + hl] = kTombstone;
            // merge output (merge_entries order): insert p lands at p + survivors
            // below it; survivor t lands at its survivor rank + inserts below it
            const unsigned surv = valid & ~hits;
            const unsigned k = __popc(surv) + nins;
            const bool is_ins = mode == 2 && hl < nins;
            unsigned ipos = 0;
            u64 ik = 0, iv = 0;
            if (is_ins) {
                ik = s_ik[w][hb + hl];
                iv = s_iv[w][hb + hl];
                const unsigned r = s_ir[w][hb + hl];
                const unsigned vbelow = r < nv ? ((1u << s_vl[w][hb + r]) - 1u) : GM;
                ipos = hl + __popc(surv & vbelow);
            }
            unsigned spos = 0;
            const bool is_surv = mode == 2 && ((surv >> hl) & 1u);
            if (is_surv) {
                unsigned ib = 0;
                for (unsigned p = 0; p < nins; ++p) ib += s_ir[w][hb + p] <= vrank;
                spos = __popc(surv & below) + ib;
            }
            const unsigned pa = valid & ~mdel;  // commit_in_place pass-A survivors
            const unsigned moved =
                (__ballot_sync(FULL, mode == 2 && ((pa >> hl) & 1u) && unsigned(__popc(pa & below)) != hl) >> hb) & GM;
            if (is_ins) {
                s_ok[w][hb + ipos] = ik;
                s_ov[w][hb + ipos] = iv;
            }
            if (is_surv) {
                s_ok[w][hb + spos] = key;
                s_ov[w][hb + spos] = val;
            }
            __syncwarp();
            if (mode == 2) {
                if (hl < m) {
                    u64 jj = 0;
                    const bool tgt = placement_target(hl, k, m, &jj);
                    const u64 nk = tgt ? s_ok[w][hb + jj] : 0;
                    a.keys[b + hl] = nk;
                    a.vals[b + hl] = tgt ? s_ov[w][hb + jj] : 0;
                    a.st[b + hl] = tgt ? kValid : kEmpty;
                    if (a.ro && tgt && is_guard(nk)) a.ro[src_of(nk) + 1] = b + hl + 1;  // graph.hpp:176
                }
                if (k >= nleaves) {
                    if (hl < nleaves) a.hdr[b / leaf + hl] = s_ok[w][hb + (u64(hl) * leaf * k + m - 1) / m];
                } else if (hl == 0) {
                    const ull slot = atomicAdd(&a.ctr->nrefresh, 1ull);
                    a.rlist[2 * slot] = b;
                    a.rlist[2 * slot + 1] = b + m;
                }
            }
            const u32 gid_ = __shfl_sync(FULL, t_gid, gi & 31u);
            if (hl == 0 && act && big) {
                a.gflag[gid_] = 0;
                if (a.level == 0) a.t0[gid_] = ~0ull;  // the CTA kernel writes it
                const ull slot = atomicAdd(&a.ctr->nbig, 1ull);
                a.biglist[slot] = gid_;
            }
            if (hl == 0 && act && !big) {
                a.gflag[gid_] = u8(mode);
                if (a.level == 0) a.t0[gid_] = mode == 2 ? touched_word(a, b, m) : ~0ull;
                else if (mode == 2) touched_append(a, b, b + m);
                acc.bytes += alg_bytes(m, s, mode);
                if (mode == 1) {
                    const unsigned added = __popc(hits);
                    acc.committed++;
                    acc.tomb += added;
                    acc.missed += missed;
                    acc.writes += added;
                    acc.vd -= added;
                    acc.td += added;
                } else if (mode == 2) {
                    int old_empty = 0;
                    for (unsigned l = 0; l < nleaves; ++l) old_empty += ((nonempty >> (l * leaf)) & leafmask) == 0;
                    acc.committed++;
                    acc.missed += missed;
                    acc.writes += m + (a.large ? __popc(moved) : 0u);
                    acc.merge += m;
                    acc.vd += (long long)k - (long long)nv;
                    acc.td -= __popc(nonempty & ~valid);
                    acc.ed += (k >= nleaves ? 0 : int(nleaves - k)) - old_empty;
                }
            }
            __syncwarp();
        }
    }
    warp_reduce_acc(acc);
    if (lane != 0) acc = Acc{};
    block_flush(acc, a.ctr);
    level_stamp(a.ctr, a.level, false);
}

// ------------------------------------------------------------- CTA tier
// Any segment size.  One CTA per group; the segment's Valid entries are
// compacted to slot-space scratch E, update ranks come from binary searches
// in E, survivors/inserts scatter to O by rank, and the segment is rewritten
// by destination-driven placement.  Also the engine of the sequential ops.
__global__ void __launch_bounds__(kCtaThreads) k_commit_cta(CommitArgs a) {
    __shared__ ull s_w64[kCtaThreads / 32];
    pdl_enter();
    level_stamp(a.ctr, a.level, true);
    // biglist mode: only the hub groups the warp tiers handed over
    const ull ngroups = a.biglist ? a.ctr->nbig : a.ctr->ngroups;
    Acc acc;
    for (ull gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        const ull g = a.biglist ? a.biglist[gi] : gi;
        const u32 lo = a.gstart[g], hi = a.gstart[g + 1];
        const u64 s = hi - lo;
        if (threadIdx.x == 0) atomicMax(&a.ctr->max_slice, ull(s));
        const u64 seg = a.gseg[g];
        const u64 m = a.m;
        const u64 b = seg * m;
        SlicePending sl{a.uk, a.uv, a.uop, a.pidx, lo};
        ull ins = 0;
        for (u64 q = threadIdx.x; q < s; q += kCtaThreads) ins += sl.op(q) == kOpInsert;
        ins = block_sum(ins, s_w64);
        ull nv = 0, nt = 0;
        for (u64 t = threadIdx.x; t < m; t += kCtaThreads) {
            const u8 x = a.st[b + t];
            nv += x == kValid;
            nt += x == kTombstone;
        }
        nv = block_sum(nv, s_w64);
        nt = block_sum(nt, s_w64);
        const u64 dels = s - ins;
        u8 flag = 0;
        if (!a.eager && ins == 0) {
            // tombstones: a pending key, if present, still sits in its batch-start
            // leaf (no commit has rewritten that leaf yet), so probe the leaf.
            ull added = 0, missed = 0;
            for (u64 q = threadIdx.x; q < s; q += kCtaThreads) {
                const u64 u = sl.key(q);
                const u64 lb = u64(a.ul[sl.pid(q)]) * a.leaf;
                bool hit = false;
                for (u64 t = lb; t < lb + a.leaf; ++t) {
                    if (a.st[t] != kEmpty && a.keys[t] == u) {
                        if (a.st[t] == kValid) {
                            a.st[t] = kTombstone;
                            hit = true;
                        }
                        break;
                    }
                }
                added += hit;
                missed += !hit;
            }
            added = block_sum(added, s_w64);
            missed = block_sum(missed, s_w64);
            if (threadIdx.x == 0) {
                acc.tomb += added;
                acc.missed += missed;
                acc.writes += added;
                acc.vd -= (long long)added;
                acc.td += (long long)added;
            }
            flag = 1;
        } else if (nv + ins > a.mx || (a.eager && a.cap_gt_min && nv < dels + a.mn)) {
            flag = 0;
        } else if (a.gridlist) {
            // grid tier (large segments, commit_in_place segment_engine.hpp:
            // 147-230): decided here, merged by device-wide kernels afterwards
            // (Pma::grid_merge); headers and touched range queued as usual
            if (threadIdx.x == 0) {
                a.gridlist[atomicAdd(&a.ctr->ngrid, 1ull)] = u32(g);
                const ull slot = atomicAdd(&a.ctr->nrefresh, 1ull);
                a.rlist[2 * slot] = b;
                a.rlist[2 * slot + 1] = b + m;
            }
            flag = 4;
        } else {
            const u64 nleaves = m / a.leaf;
            ull old_empty = 0;
            for (u64 l = threadIdx.x; l < nleaves; l += kCtaThreads) {
                bool e = true;
                for (u64 t = b + l * a.leaf; t < b + (l + 1) * a.leaf; ++t) e &= a.st[t] == kEmpty;
                old_empty += e;
            }
            old_empty = block_sum(old_empty, s_w64);
            const MergeOut r = block_merge_segment(a.keys, a.vals, a.st, b, m, nv, sl, s, a.large != 0, a.ek, a.ev,
                                                   a.es, a.mflag, a.ok, a.ov, a.ik + lo, a.iv + lo, a.ir + lo);
            if (threadIdx.x == 0) {
                acc.missed += r.missed;
                acc.writes += m + r.moves;
                acc.merge += m;
                acc.vd += (long long)r.k - (long long)nv;
                acc.td -= (long long)nt;
                const long long new_empty = r.k >= nleaves ? 0 : (long long)(nleaves - r.k);
                acc.ed += new_empty - (long long)old_empty;
                const ull slot = atomicAdd(&a.ctr->nrefresh, 1ull);  // headers/row offsets: post-pass
                a.rlist[2 * slot] = b;
                a.rlist[2 * slot + 1] = b + m;
            }
            flag = 2;
        }
        if (threadIdx.x == 0) {
            a.gflag[g] = flag;
            if (a.level == 0) a.t0[g] = flag == 2 ? touched_word(a, b, m) : ~0ull;
            else if (flag == 2 || flag == 4) touched_append(a, b, b + m);
            acc.bytes += alg_bytes(m, s, flag == 4 ? 2 : flag);
            if (flag) acc.committed++;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) acc = Acc{};
    block_flush(acc, a.ctr);
    level_stamp(a.ctr, a.level, false);
}

// ------------------------------------------------------------- grid tier
// A large segment (>= grid_seg_ slots) is merged by device-wide kernels, the
// root path's algorithm on the range [b, b + m): Valid entries compacted to
// E (tombstones purged), the slice ranked in E, survivors and inserts
// scattered to O by rank, destination-driven even placement back.  The
// slice is the group's pending indices; counts live in the Ctr.
__global__ void k_grid_ranks(const u64* __restrict__ uk, const u8* __restrict__ uop, const u32* __restrict__ plist,
                             u64 s, const u64* __restrict__ ek, const ull* nv_dev, u8* __restrict__ mflag, Ctr* ctr) {
    const u64 nv = *nv_dev;
    ull missed = 0;
    for (u64 q = blockIdx.x * u64(blockDim.x) + threadIdx.x; q < s; q += u64(gridDim.x) * blockDim.x) {
        const u32 pi = plist[q];
        const u64 u = uk[pi];
        const u64 r = lower_bound_dev(ek, nv, u);
        const bool isins = uop[pi] == kOpInsert;
        if (r < nv && ek[r] == u) mflag[r] = isins ? 2 : 1;
        else if (!isins) ++missed;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) missed += __shfl_xor_sync(FULL, missed, d);
    if ((threadIdx.x & 31) == 0 && missed) atomicAdd(&ctr->missed, missed);
}

// tombstones and empty leaves of [b, b + m) before the merge
__global__ void k_grid_seg_counts(const u8* __restrict__ st, u64 b, u64 m, u64 leaf, Ctr* ctr) {
    ull nt = 0, ne = 0;
    for (u64 l = blockIdx.x * u64(blockDim.x) + threadIdx.x; l < m / leaf; l += u64(gridDim.x) * blockDim.x) {
        bool empty = true;
        for (u64 t = b + l * leaf; t < b + (l + 1) * leaf; ++t) {
            const u8 x = st[t];
            nt += x == kTombstone;
            empty &= x == kEmpty;
        }
        ne += empty;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        nt += __shfl_xor_sync(FULL, nt, d);
        ne += __shfl_xor_sync(FULL, ne, d);
    }
    if ((threadIdx.x & 31) == 0) {
        if (nt) atomicAdd(&ctr->seg_tomb, nt);
        if (ne) atomicAdd(&ctr->seg_empty, ne);
    }
}

// the merge's counters, as k_commit_cta's accumulator would add them
__global__ void k_grid_account(Ctr* ctr, u64 m, u64 leaf, int large) {
    const ull k = ctr->k, nv = ctr->nv, moves = large ? ctr->moves : 0;
    const u64 nleaves = m / leaf;
    const long long new_empty = k >= nleaves ? 0 : (long long)(nleaves - k);
    ctr->slot_writes += m + moves;
    ctr->merge_slots += m;
    ctr->valid_delta += (long long)k - (long long)nv;
    ctr->tomb_delta -= (long long)ctr->seg_tomb;
    ctr->empty_delta += new_empty - (long long)ctr->seg_empty;
}

// ------------------------------------------------------------- refresh

// Leaf headers (and graph row offsets, graph.hpp:167-180) over the ranges
// the commit kernels could not refresh in place (sparse or CTA-tier
// segments), one warp per range: hdr[i] = first non-Empty key at or after
// leaf i (the scan may run past the range end into untouched leaves).
__global__ void k_refresh_ranges(const u64* __restrict__ ranges, const ull* n_dev, u64 n_host,
                                 const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap, u64 leaf,
                                 u64* __restrict__ hdr, u64* __restrict__ ro, Ctr* cctr = nullptr,
                                 Ctr* hctr = nullptr) {
    pdl_enter();
    const u64 nranges = n_dev ? *n_dev : n_host;
    const unsigned lane = threadIdx.x & 31u;
    const u64 warp = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 r = warp; r < nranges; r += nwarps) {
        const u64 b = ranges[2 * r], e = ranges[2 * r + 1];
        for (u64 i = b / leaf + lane; i < (e + leaf - 1) / leaf; i += 32) {
            u64 v = ~0ull;
            for (u64 t = i * leaf; t < cap; ++t) {
                if (st[t] != kEmpty) {
                    v = keys[t];
                    break;
                }
            }
            hdr[i] = v;
        }
        if (ro) {
            for (u64 t = b + lane; t < e; t += 32) {
                if (st[t] == kValid) {
                    const u64 k = keys[t];
                    if (is_guard(k)) ro[src_of(k) + 1] = t + 1;
                }
            }
        }
    }
    if (hctr) {
        // captured small batches: the last CTA to finish stamps the end of
        // the device span and returns the counters to page-locked host memory
        // (no copy node, no event nodes)
        __shared__ bool s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&cctr->refresh_done, 1ull) == gridDim.x - 1;
            if (s_last) {
                __threadfence();
                u64 g;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                cctr->gt1 = g;
            }
        }
        __syncthreads();
        if (s_last) {
            const ull* src = reinterpret_cast<const ull*>(cctr);
            ull* dst = reinterpret_cast<ull*>(hctr);
            for (u32 i = threadIdx.x; i < sizeof(Ctr) / 8; i += blockDim.x) dst[i] = ld_volatile(src + i);
            __syncthreads();
            if (threadIdx.x == 0) {  // the counters landed first: the host may read them once it sees this
                __threadfence_system();
                st_volatile(&hctr->done_seq, ld_volatile(&cctr->seq));
            }
        }
    }
}

// Empty leaves left of a touched range inherit its first header.
// (over the batch's touched words: level 0's dense words t0 — ~0 = none —
// then the appended rest)
__global__ void k_left_walk(const u64* __restrict__ t0, u64 n0, const u64* __restrict__ trest, u64 nrest, int cb,
                            const u8* __restrict__ st, u64 leaf, u64* __restrict__ hdr, const ull* n0_dev = nullptr,
                            const ull* nrest_dev = nullptr) {
    pdl_enter();
    if (n0_dev) n0 = *n0_dev;
    if (nrest_dev) nrest = *nrest_dev;
    for (u64 r = blockIdx.x * u64(blockDim.x) + threadIdx.x; r < n0 + nrest; r += u64(gridDim.x) * blockDim.x) {
        const u64 w = r < n0 ? t0[r] : trest[r - n0];
        if (w == ~0ull) continue;
        const u64 la = (w & ((1ull << cb) - 1)) / leaf;
        const u64 v = hdr[la];
        for (u64 i = la; i-- > 0;) {
            bool empty = true;
            for (u64 t = i * leaf; t < (i + 1) * leaf; ++t)
                if (st[t] != kEmpty) {
                    empty = false;
                    break;
                }
            if (!empty) break;
            hdr[i] = v;
        }
    }
}

__global__ void k_row_offsets_full(const u64* __restrict__ keys, const u8* __restrict__ st, u64 cap,
                                   u64* __restrict__ ro) {
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < cap; t += u64(gridDim.x) * blockDim.x) {
        if (st[t] == kValid) {
            const u64 k = keys[t];
            if (is_guard(k)) ro[src_of(k) + 1] = t + 1;
        }
    }
}

// ------------------------------------------------------------- root path
// Device-wide merge of the single root group (segment_engine.hpp:435-463).

__global__ void k_root_ranks(const u64* __restrict__ uk, const u8* __restrict__ uop, const u32* __restrict__ pidx,
                             const ull* npend_dev, const u64* __restrict__ ek, const ull* nv_dev, u8* mflag,
                             Ctr* ctr) {
    const u64 n = *npend_dev, nv = *nv_dev;
    ull missed = 0;
    for (u64 p = blockIdx.x * u64(blockDim.x) + threadIdx.x; p < n; p += u64(gridDim.x) * blockDim.x) {
        const u32 pi = pidx[p];
        const u64 u = uk[pi];
        const u64 r = lower_bound_dev(ek, nv, u);
        const bool isins = uop[pi] == kOpInsert;
        if (r < nv && ek[r] == u) mflag[r] = isins ? 2 : 1;
        else if (!isins) ++missed;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) missed += __shfl_xor_sync(FULL, missed, d);
    if ((threadIdx.x & 31) == 0 && missed) atomicAdd(&ctr->missed, missed);
}

__global__ void k_root_scatter_surv(const u64* __restrict__ ek, const u64* __restrict__ ev, const ull* nv_dev,
                                    const u8* __restrict__ mflag, const u32* __restrict__ mbv,
                                    const u32* __restrict__ irr, const ull* nins_dev, u64* __restrict__ okk,
                                    u64* __restrict__ ovv) {
    const u64 nv = *nv_dev, nins = *nins_dev;
    for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < nv; j += u64(gridDim.x) * blockDim.x) {
        if (mflag[j] != 0) continue;
        const u64 pos = (j - mbv[j]) + upper_bound_u32(irr, nins, j);
        okk[pos] = ek[j];
        ovv[pos] = ev[j];
    }
}

__global__ void k_root_scatter_ins(const u64* __restrict__ ikk, const u64* __restrict__ ivv,
                                   const u32* __restrict__ irr, const ull* nins_dev, const u32* __restrict__ mbv,
                                   u64* __restrict__ okk, u64* __restrict__ ovv, Ctr* ctr) {
    const u64 nins = *nins_dev;
    for (u64 p = blockIdx.x * u64(blockDim.x) + threadIdx.x; p < nins; p += u64(gridDim.x) * blockDim.x) {
        const u64 r = irr[p];
        const u64 pos = (r - mbv[r]) + p;
        okk[pos] = ikk[p];
        ovv[pos] = ivv[p];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->k = (ctr->nv - ctr->nmatched) + nins;
}

// ------------------------------------------------------------- point queries

__global__ void k_search(const u64* __restrict__ q, u64 n, const u64* __restrict__ hdr, u64 L,
                         const u64* __restrict__ keys, const u64* __restrict__ vals, const u8* __restrict__ st,
                         u64 leaf, u64* out_vals, u8* found, u64* leaves) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        const u64 key = q[i];
        const u64 lf = leaf_of_key(hdr, L, st, leaf, key);
        if (leaves) leaves[i] = lf;
        if (found) {
            u8 f = 0;
            u64 v = 0;
            for (u64 t = lf * leaf; t < (lf + 1) * leaf; ++t) {
                if (st[t] != kEmpty && keys[t] == key) {
                    if (st[t] == kValid) {
                        f = 1;
                        v = vals[t];
                    }
                    break;
                }
            }
            found[i] = f;
            out_vals[i] = v;
        }
    }
}

__global__ void k_count_valid(const u8* __restrict__ st, u64 b, u64 e, Ctr* ctr) {
    ull c = 0;
    for (u64 t = b + blockIdx.x * u64(blockDim.x) + threadIdx.x; t < e; t += u64(gridDim.x) * blockDim.x)
        c += st[t] == kValid;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(FULL, c, d);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&ctr->nv, c);
}

// Parity digest of the slot array (tests/golden/hashing.py restates it in
// numpy): slot i contributes mix(key + mix(value ^ (i * phi + state))) and a
// chunk's hash is the wrapping sum over its slots, so keys, values, states
// and gap positions are all pinned without downloading the array.
__device__ __forceinline__ u64 mix64(u64 x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void k_slot_hash(const u64* __restrict__ keys, const u64* __restrict__ vals, const u8* __restrict__ st,
                            u64 cap, int chunk_log2, ull* out) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < cap; i += u64(gridDim.x) * blockDim.x) {
        const u64 a = i * 0x9E3779B97F4A7C15ull + st[i];
        ull h = mix64(keys[i] + mix64(vals[i] ^ a));
        if (chunk_log2 >= 5) {  // a warp's 32 consecutive slots share one chunk
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) h += __shfl_xor_sync(FULL, h, d);
            if ((threadIdx.x & 31) == 0) atomicAdd(&out[i >> chunk_log2], h);
        } else {
            atomicAdd(&out[i >> chunk_log2], h);
        }
    }
}

// ========================================================== host pipeline

void Pma::headers_closed_form(const u64* d_ek, u64 k) {
    const u64 L = num_leaves();
    k_headers_closed<<<grid_for(L, 256), 256, 0, stream_>>>(d_hdr, L, leaf_, cap_, d_ek, nullptr, k);
    GPMA_LAUNCH_CHECK();
}

void Pma::place_root_from(const u64* d_ek, const u64* d_ev, u64 k) {
    if (k > 0) {
        k_place_evenly<<<grid_for(cap_, 256, 148 * 32), 256, 0, stream_>>>(d_keys, d_vals, d_st, 0, cap_, d_ek, d_ev,
                                                                           nullptr, k);
        GPMA_LAUNCH_CHECK();
        slot_writes += cap_;
    }
    valid_count = k;
    tombstone_count = 0;
    empty_leaves = k >= num_leaves() ? 0 : (long long)(num_leaves() - k);  // spacing >= leaf: one entry per leaf
    headers_closed_form(d_ek, k);
}

// from_sorted (pma.hpp:160-187): capacity rule on the host, placement on
// the device.  d_keys/d_vals are device arrays of n strictly increasing keys.
void Pma::from_sorted_device(const u64* dk, const u64* dv, u64 n, double fill_target) {
    if (!(fill_target > 0.0 && fill_target <= prof_.leaf_upper + 1e-12))
        throw ApiError(PMA_EINVAL, "from_sorted: fill_target must be in (0, leaf_upper]");
    if (n > 1) {
        GPMA_CUDA(cudaMemsetAsync(d_ctr, 0xFF, sizeof(ull) * 0, stream_));
        ull init = ~0ull;
        GPMA_CUDA(cudaMemcpyAsync(&d_ctr->bad_index, &init, sizeof(ull), cudaMemcpyHostToDevice, stream_));
        k_validate_sorted<<<grid_for(n, 256), 256, 0, stream_>>>(dk, n, d_ctr);
        GPMA_LAUNCH_CHECK();
        sync_ctr();
        if (h_ctr->bad_index != ~0ull)
            throw ApiError(PMA_EINVAL,
                           "from_sorted: keys must be strictly increasing (duplicate or unsorted input at index " +
                               std::to_string(h_ctr->bad_index) + ")");
    }
    slot_writes = 0;  // a fresh array (from_sorted returns a new PMA)
    u64 cap = 16;
    while (double(n) > fill_target * double(cap)) cap <<= 1;
    u64 c = cap;
    // capacity search on the host before allocating
    auto mx_root = [&](u64 cc) { return max_at_capacity(cc); };
    auto mn_root = [&](u64 cc) {
        const u64 lf = leaf_size_for(cc);
        const u64 mn0 = u64(std::ceil(prof_.leaf_lower * double(lf) - 1e-9));
        return mn0 << height_for(cc, lf);
    };
    while (n > mx_root(c)) c <<= 1;
    while (c > 16 && n < mn_root(c) && n <= mx_root(c >> 1)) c >>= 1;
    reset_layout(c);
    place_root_from(dk, dv, n);
    if (d_row_offsets) rebuild_row_offsets_full();
}

void Pma::load_slots(size_t capacity, const u64* keys, const u64* values, const u8* states) {
    if (capacity < 16 || (capacity & (capacity - 1)))
        throw ApiError(PMA_EINVAL, "load_slots: capacity must be a power of two >= 16");
    reset_layout(capacity);
    GPMA_CUDA(cudaMemcpyAsync(d_st, states, capacity, cudaMemcpyHostToDevice, stream_));
    // Empty slots must be zero: sanitize on the host copy path
    std::vector<u64> k(keys, keys + capacity), v(values, values + capacity);
    u64 nv = 0, nt = 0;
    for (size_t i = 0; i < capacity; ++i) {
        if (states[i] == kEmpty) k[i] = v[i] = 0;
        nv += states[i] == kValid;
        nt += states[i] == kTombstone;
    }
    GPMA_CUDA(cudaMemcpyAsync(d_keys, k.data(), capacity * 8, cudaMemcpyHostToDevice, stream_));
    GPMA_CUDA(cudaMemcpyAsync(d_vals, v.data(), capacity * 8, cudaMemcpyHostToDevice, stream_));
    // full header rebuild over 4096-slot chunks (forward scans cross chunks)
    const u64 chunk = capacity < 4096 ? capacity : 4096;
    std::vector<u64> ranges;
    for (u64 b = 0; b < capacity; b += chunk) {
        ranges.push_back(b);
        ranges.push_back(b + chunk);
    }
    u64 empties = 0;
    for (u64 l = 0; l < capacity / leaf_; ++l) {
        bool e = true;
        for (u64 t = l * leaf_; t < (l + 1) * leaf_; ++t) e &= states[t] == kEmpty;
        empties += e;
    }
    stage_k.reserve(ranges.size());
    GPMA_CUDA(cudaMemcpyAsync(stage_k.ptr, ranges.data(), ranges.size() * 8, cudaMemcpyHostToDevice, stream_));
    k_refresh_ranges<<<grid_for(ranges.size() / 2 * 32, 256), 256, 0, stream_>>>(
        stage_k.ptr, nullptr, ranges.size() / 2, d_keys, d_st, cap_, leaf_, d_hdr, nullptr);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaStreamSynchronize(stream_));
    valid_count = nv;
    tombstone_count = nt;
    slot_writes = 0;
    empty_leaves = (long long)empties;
}

void Pma::download(u64* keys, u64* values, u8* states) {
    if (keys) GPMA_CUDA(cudaMemcpyAsync(keys, d_keys, cap_ * 8, cudaMemcpyDeviceToHost, stream_));
    if (values) GPMA_CUDA(cudaMemcpyAsync(values, d_vals, cap_ * 8, cudaMemcpyDeviceToHost, stream_));
    if (states) GPMA_CUDA(cudaMemcpyAsync(states, d_st, cap_, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

void Pma::rebuild_row_offsets_full() {
    if (!d_row_offsets) return;
    GPMA_CUDA(cudaMemsetAsync(d_row_offsets, 0, (num_vertices + 1) * 8, stream_));
    k_row_offsets_full<<<grid_for(cap_, 256, 148 * 16), 256, 0, stream_>>>(d_keys, d_st, cap_, ro_base());
    GPMA_LAUNCH_CHECK();
}

// rebuild_at_capacity (pma.hpp:597-601): compact Valid entries, re-place at
// the root of a fresh array of `cap` slots.
void Pma::rebuild_at_capacity(u64 cap) {
    ensure_slot_scratch();
    u64* dek = ek.ptr;
    u64* dev = ev.ptr;
    const u64* kk = d_keys;
    const u64* vv = d_vals;
    const u8* ss = d_st;
    run_compact(
        stream_, ws, nullptr, cap_, cap_, [=] __device__(ull i) { return ss[i] == kValid; },
        [=] __device__(ull i, unsigned f, ull x) {
            if (f) {
                dek[x] = kk[i];
                dev[x] = vv[i];
            }
        },
        NoFin{});
    const u64 n = valid_count;
    reset_layout(cap);
    place_root_from(dek, dev, n);
}

// Grid tier: merge segment [b, b + m) with the group's slice (pending
// indices plist[0, s)) by device-wide kernels (see k_grid_ranks).  The
// counters land in the Ctr as a CTA-tier merge's would (k_grid_account);
// headers / row offsets and the touched range were queued by k_commit_cta.
void Pma::grid_merge(u64 b, u64 m, const u32* plist, u64 s, bool large) {
    ensure_slot_scratch();
    GPMA_CUDA(cudaMemsetAsync(&d_ctr->seg_tomb, 0, 2 * sizeof(ull), stream_));
    k_grid_seg_counts<<<grid_for(m / leaf_, 256, 148 * 8), 256, 0, stream_>>>(d_st, b, m, leaf_, d_ctr);
    GPMA_LAUNCH_CHECK();
    u64* dek = ek.ptr + b;
    u64* dev = ev.ptr + b;
    u32* des = es.ptr + b;
    u8* mf = mflag.ptr + b;
    u32* mbv = mb.ptr + b;
    const u64* kk = d_keys + b;
    const u64* vv = d_vals + b;
    const u8* ss = d_st + b;
    Ctr* ctr = d_ctr;
    run_compact(
        stream_, ws, nullptr, m, m, [=] __device__(ull i) { return ss[i] == kValid; },
        [=] __device__(ull i, unsigned f, ull x) {
            if (f) {
                dek[x] = kk[i];
                dev[x] = vv[i];
                des[x] = u32(i);
                mf[x] = 0;
            }
        },
        [=] __device__(ull total) { ctr->nv = total; });
    k_grid_ranks<<<grid_for(s, 256, 148 * 8), 256, 0, stream_>>>(uk.ptr, uop.ptr, plist, s, dek, &d_ctr->nv, mf,
                                                               d_ctr);
    GPMA_LAUNCH_CHECK();
    {
        const u64* uuk = uk.ptr;
        const u64* uuv = uv.ptr;
        const u8* uuo = uop.ptr;
        u64* ikk = ik.ptr;
        u64* ivv = iv.ptr;
        u32* irr = ir.ptr;
        const ull* nvp = &d_ctr->nv;
        run_compact(
            stream_, ws, nullptr, s, s, [=] __device__(ull q) { return uuo[plist[q]] == kOpInsert; },
            [=] __device__(ull q, unsigned f, ull x) {
                if (!f) return;
                const u64 u = uuk[plist[q]];
                ikk[x] = u;
                ivv[x] = uuv[plist[q]];
                irr[x] = u32(lower_bound_dev(dek, *nvp, u));
            },
            [=] __device__(ull total) { ctr->nins = total; });
    }
    run_compact(
        stream_, ws, &d_ctr->nv, 0, m + 1, [=] __device__(ull j) { return mf[j] != 0; },
        [=] __device__(ull j, unsigned, ull x) { mbv[j] = u32(x); },
        [=] __device__(ull total) {
            ctr->nmatched = total;
            mbv[ctr->nv] = u32(total);
        });
    k_root_scatter_surv<<<grid_for(m, 256, 148 * 16), 256, 0, stream_>>>(dek, dev, &d_ctr->nv, mf, mbv, ir.ptr,
                                                                        &d_ctr->nins, ok.ptr + b, ov.ptr + b);
    GPMA_LAUNCH_CHECK();
    k_root_scatter_ins<<<grid_for(s, 256, 148 * 8), 256, 0, stream_>>>(ik.ptr, iv.ptr, ir.ptr, &d_ctr->nins, mbv,
                                                                      ok.ptr + b, ov.ptr + b, d_ctr);
    GPMA_LAUNCH_CHECK();
    if (large) {  // commit_in_place counts the compaction moves (segment_engine.hpp:147-230)
        GPMA_CUDA(cudaMemsetAsync(&d_ctr->moves, 0, sizeof(ull), stream_));
        run_compact(
            stream_, ws, &d_ctr->nv, 0, m + 1, [=] __device__(ull j) { return mf[j] != 1; },
            [=] __device__(ull j, unsigned f, ull x) {
                if (f && u64(des[j]) != x) atomicAdd(&ctr->moves, 1ull);
            },
            NoFin{});
    }
    k_place_evenly<<<grid_for(m, 256, 148 * 32), 256, 0, stream_>>>(d_keys, d_vals, d_st, b, m, ok.ptr + b, ov.ptr + b,
                                                                   &d_ctr->k, 0);
    GPMA_LAUNCH_CHECK();
    k_grid_account<<<1, 1, 0, stream_>>>(d_ctr, m, leaf_, large ? 1 : 0);
    GPMA_LAUNCH_CHECK();
}

// One round (level) of the engine (segment_engine.hpp:78-105, 320-341):
// group the pending list by segment (unique_segments), decide + commit every
// group, keep the deferred groups' updates (advance_round).  Every kernel
// reads its counts on the device; npend is a host-known upper bound of the
// pending count.  (The commit kernels stamp the level's span into the
// counters: lvl_tmin / lvl_tmax.)
// Round-disjointness check (the reference's assert, segment_engine.hpp:400-405,
// live in its release builds): a level's groups name strictly
// increasing segments, each with a non-empty slice of the pending updates,
// so no two commits of a round touch the same slots.  Debug switch
// GPMA_CHECK_ROUNDS=1; a violation fails the batch with PMA_ELOGIC.
__global__ void k_check_rounds(const u32* __restrict__ gseg, const u32* __restrict__ gstart, Ctr* ctr) {
    pdl_enter();
    const ull ng = ctr->ngroups;
    ull bad = 0;
    for (ull g = blockIdx.x * u64(blockDim.x) + threadIdx.x; g < ng; g += u64(gridDim.x) * blockDim.x) {
        if (gstart[g] >= gstart[g + 1]) ++bad;
        if (g && gseg[g] <= gseg[g - 1]) ++bad;
    }
    if (bad) atomicAdd(&ctr->round_overlap, bad);
}

void Pma::enqueue_level(int level, u64 npend, u32* pcur, u32* pnext, u64* touched_ptr, u64 n, const EngineCfg& cfg,
                        ScanWorkspace& ws, bool events, u64& launches) {
    const u64 m = leaf_ << level;
    ull* np_cur = &d_ctr->np[level & 1];
    ull* np_next = &d_ctr->np[(level + 1) & 1];
    // group = segment heads (unique_segments)
    {
        const u32* ulp = ul.ptr;
        const u32* pp = pcur;
        u32* gs = gstart.ptr;
        u32* gg = gseg.ptr;
        u32* gi = gid.ptr;
        Ctr* ctr = d_ctr;
        const int lv = level;
        run_compact(
            stream_, ws, np_cur, 0, npend,
            [=] __device__(ull p) {
                return p == 0 || (ulp[pp ? pp[p] : p] >> lv) != (ulp[pp ? pp[p - 1] : p - 1] >> lv);
            },
            [=] __device__(ull p, unsigned f, ull x) {
                if (f) {
                    gs[x] = u32(p);
                    gg[x] = ulp[pp ? pp[p] : p] >> lv;
                }
                gi[p] = u32(x + f - 1);
            },
            [=] __device__(ull total) {
                ctr->ngroups = total;
                gs[total] = u32(*np_cur);
                ctr->lvl_npend[lv] = *np_cur;
            },
            level == 0 ? &d_ctr->t_rounds : nullptr);
        ++launches;
    }
    if (check_rounds_) {
        launch_k(k_check_rounds, dim3(grid_for(npend, 256, 148 * 4)), dim3(256), 0, stream_,
                 static_cast<const u32*>(gseg.ptr), static_cast<const u32*>(gstart.ptr), d_ctr);
        ++launches;
    }
    // commit (decide + merge + scatter)
    CommitArgs a{};
    a.t0 = touched_ptr;
    a.tlist = touched_ptr + touched_split_;
    a.cb = touched_cb_;
    a.keys = d_keys;
    a.vals = d_vals;
    a.st = d_st;
    a.uk = uk.ptr;
    a.uv = uv.ptr;
    a.uop = uop.ptr;
    a.ul = ul.ptr;
    a.pidx = pcur;
    a.gstart = gstart.ptr;
    a.gseg = gseg.ptr;
    a.gflag = gflag.ptr;
    a.ctr = d_ctr;
    a.hdr = d_hdr;
    a.ro = ro_base();
    a.rlist = rlist.ptr;
    a.level = level;
    a.m = m;
    a.leaf = leaf_;
    a.mn = mn_[level];
    a.mx = mx_[level];
    a.eager = cfg.eager;
    a.large = cfg.large_for(m);
    a.cap_gt_min = cap_ > 16;
    if (level_events_ && events && level < 16) GPMA_CUDA(cudaEventRecord(lev_ev_[2 * level], stream_));
    ensure_slot_scratch();
    ik.reserve(n);
    iv.reserve(n);
    ir.reserve(n);
    biglist.reserve(npend + 1);
    a.ek = ek.ptr;
    a.ev = ev.ptr;
    a.es = es.ptr;
    a.mflag = mflag.ptr;
    a.ok = ok.ptr;
    a.ov = ov.ptr;
    a.ik = ik.ptr;
    a.iv = iv.ptr;
    a.ir = ir.ptr;
    a.biglist = biglist.ptr;
    if (m <= 32) {
        // warp tiers; hub groups (large slices) are appended to biglist
        if (m == 16 && leaf_ == 16 && pcur == nullptr) {  // level 0: identity pending list
            // exactly the resident CTAs (persistent: the grid-stride tile
            // loop balances; a partial last wave costs ~10%, measured)
            static const unsigned resident = [] {
                int per_sm = 0, dev = 0, sms = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_commit_leaf, kLeafWarps * 32, 0);
                return unsigned((per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148));
            }();
            const unsigned grid = grid_for((npend + 31) / 32, kLeafWarps, resident);
            launch_k(k_commit_leaf, dim3(grid), dim3(kLeafWarps * 32), 0, stream_, a);
        } else {
            // grid for the host bound; the kernel sizes its tiles from the
            // device-side group count (<= npend)
            const unsigned grid = grid_for(npend, kWarpTierWarps, 148 * 8);
            if (m <= 16) launch_k(k_commit_lanes<16>, dim3(grid), dim3(kWarpTierWarps * 32), 0, stream_, a);
            else launch_k(k_commit_lanes<32>, dim3(grid), dim3(kWarpTierWarps * 32), 0, stream_, a);
        }
        GPMA_LAUNCH_CHECK();
        // CTA kernel over the hub groups only (grid bounded by npend / kBigSlice)
        launch_k(k_commit_cta, dim3(grid_for(npend / kBigSlice + 1, 1, 148 * 2)), dim3(kCtaThreads), 0, stream_, a);
    } else {
        a.biglist = nullptr;
        const bool grid_tier = m >= grid_seg_;
        if (grid_tier) {
            a.gridlist = biglist.ptr;
            GPMA_CUDA(cudaMemsetAsync(&d_ctr->ngrid, 0, sizeof(ull), stream_));
        }
        const unsigned grid = grid_for(npend, 1, 148 * 4);
        k_commit_cta<<<grid, kCtaThreads, 0, stream_>>>(a);
        GPMA_LAUNCH_CHECK();
        if (grid_tier) {
            // large segments: the CTAs decided; the merges run device-wide,
            // one group at a time (a handful per level at most)
            sync_ctr();
            const u64 ng = h_ctr->ngrid;
            if (ng) {
                std::vector<u32> gl(ng), gsv, gst;
                GPMA_CUDA(cudaMemcpyAsync(gl.data(), biglist.ptr, ng * 4, cudaMemcpyDeviceToHost, stream_));
                const u64 ngr = h_ctr->ngroups;
                gst.resize(ngr + 1);
                gsv.resize(ngr);
                GPMA_CUDA(cudaMemcpyAsync(gst.data(), gstart.ptr, (ngr + 1) * 4, cudaMemcpyDeviceToHost, stream_));
                GPMA_CUDA(cudaMemcpyAsync(gsv.data(), gseg.ptr, ngr * 4, cudaMemcpyDeviceToHost, stream_));
                GPMA_CUDA(cudaStreamSynchronize(stream_));
                std::sort(gl.begin(), gl.end());
                for (const u32 g : gl) {
                    grid_merge(u64(gsv[g]) * m, m, pcur + gst[g], u64(gst[g + 1] - gst[g]), cfg.large_for(m));
                    launches += 9;
                    timing.grid_merges++;
                }
            }
        }
    }
    GPMA_LAUNCH_CHECK();
    if (level_events_ && events && level < 16) GPMA_CUDA(cudaEventRecord(lev_ev_[2 * level + 1], stream_));
    ++launches;
    // advance_round: keep deferred groups' updates
    {
        const u8* gf = gflag.ptr;
        const u32* gi = gid.ptr;
        const u32* pp = pcur;
        u32* pn = pnext;
        Ctr* ctr = d_ctr;
        const int lv = level;
        run_compact(
            stream_, ws, np_cur, 0, npend, [=] __device__(ull p) { return gf[gi[p]] == 0; },
            [=] __device__(ull p, unsigned f, ull x) {
                if (f) pn[x] = pp ? pp[p] : u32(p);
            },
            [=] __device__(ull total) {
                *np_next = total;
                // the level's stats (read at the next host sync)
                ctr->lvl_committed[lv] = ctr->committed;
                ctr->lvl_bytes[lv] = ctr->commit_bytes;  // cumulative up to this level
                ctr->lvl_groups[lv] = ctr->ngroups;
                ctr->lvl_big[lv] = ctr->nbig;
                ctr->lvl_maxslice[lv] = ctr->max_slice;
                ctr->lvl_merge[lv] = ctr->merge_slots;
                ctr->committed = 0;
                ctr->nbig = 0;
                ctr->max_slice = 0;
            });
        ++launches;
    }
}

// ---- small graph batches ----------------------------------------------
// A batch of up to kSmallGraphMax graph updates is latency-bound: a dozen
// tiny kernels whose cost is their launches and the host round trips between
// rounds.  Its whole front end (k_small_front: pack + checks, one-CTA sort,
// duplicate resolution; k_leaf_search_warp) and round 0 are captured ONCE as
// a CUDA graph with programmatic edges, whose nodes read the batch descriptor
// (in place, page-locked) and every count from device memory; each batch then
// costs one descriptor write, one graph launch and a poll of the sequence
// word the last node writes.  The graph embeds array and scratch pointers,
// the layout and the engine config; any change re-captures it.
bool Pma::small_graph_ok(u64 n, const GraphFront& gf) const {
    if (!small_graphs_ || gf.mk || n == 0 || n > kSmallGraphMax || height_ < 1 || !ro_base() || !stream_) return false;
    // (beyond one CTA's sort and the cooperative grid's chunks: the cluster only)
    if (n > kSmallFrontMax && !(small_cluster_ && cluster_front_available())) return false;
    int db = 1;
    while (db < 32 && (1ull << db) < gf.nv) ++db;
    return 2 * db + kSmallIb <= 64;
}

std::vector<uintptr_t> Pma::small_graph_key(int db, const EngineCfg& cfg, int levels) const {
    const void* ptrs[] = {d_keys, d_vals, d_st, d_hdr, ro_base(), d_ctr, d_desc_, h_desc_, h_ctr, sk_in.ptr,
                          sk_out.ptr, uk.ptr, uv.ptr, uop.ptr, ul.ptr, pidx0.ptr, pidx1.ptr, gid.ptr, gstart.ptr,
                          gseg.ptr, gflag.ptr, touched.ptr, rlist.ptr, ik.ptr, iv.ptr, ir.ptr, biglist.ptr, ek.ptr,
                          ev.ptr, es.ptr, mflag.ptr, ok.ptr, ov.ptr, small_ws_.tiles.ptr, small_sb_.ptr, stream_};
    std::vector<uintptr_t> k;
    for (const void* p : ptrs) k.push_back(reinterpret_cast<uintptr_t>(p));
    const u64 vals[] = {cap_, leaf_, u64(height_), ro_lo, num_vertices, u64(db), u64(cfg.eager), cfg.small_max,
                        cfg.medium_max, u64(cfg.force), u64(levels), u64(empty_leaves != 0), u64(small_cluster_), u64(check_rounds_)};
    for (const u64 v : vals) k.push_back(uintptr_t(v));
    return k;
}

void Pma::capture_small_graph(int db, const EngineCfg& cfg, int levels, int multi) {
    cudaGraphExec_t& exec = small_exec_[multi];
    if (exec) {
        GPMA_CUDA(cudaGraphExecDestroy(exec));
        exec = nullptr;
    }
    const int ib = kSmallIb;
    static const bool attr = [] {
        GPMA_CUDA(cudaFuncSetAttribute(k_small_front, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallFrontSmem));
        return true;
    }();
    (void)attr;
    if (!h_desc_dev_) GPMA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_desc_dev_), h_desc_, 0));
    if (!h_ctr_dev_) GPMA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_ctr_dev_), h_ctr, 0));
    u64 dummy = 0;
    cudaGraph_t graph = nullptr;
    GPMA_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    try {
        // front end in one CTA (counters and look-back words zeroed there,
        // descriptor read in place from page-locked memory), then the leaf of
        // every unique update (pma.hpp:234-289), a warp per key
        static_assert(kSmallGraphMax <= kSmallMultiMax, "small graph batches fit the cluster front end");
        if (multi && small_cluster_ && cluster_front_available()) {  // (one cluster: distributed shared memory)
            cudaLaunchAttribute at[1];
            const GraphFront* hd = h_desc_dev_;
            if (multi == 2) {
                const cudaLaunchConfig_t lc = cluster_front_config(stream_, at, cluster_smem<kSmallFrontThreads>());
                GPMA_CUDA(cudaLaunchKernelEx(&lc, k_small_front_cluster<kSmallFrontThreads>, hd, db, ib, d_ctr,
                                             small_ws_.tiles.ptr, u64(small_ws_.tiles.cap), uk.ptr, uv.ptr, uop.ptr));
            } else {
                const cudaLaunchConfig_t lc = cluster_front_config(stream_, at, cluster_smem<256>());
                GPMA_CUDA(cudaLaunchKernelEx(&lc, k_small_front_cluster<256>, hd, db, ib, d_ctr, small_ws_.tiles.ptr,
                                             u64(small_ws_.tiles.cap), uk.ptr, uv.ptr, uop.ptr));
            }
        } else if (multi) {  // (one cooperative grid: its CTAs wait on each other)
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(kChunks);
            lc.blockDim = dim3(kSmallFrontThreads);
            lc.stream = stream_;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            GPMA_CUDA(cudaLaunchKernelEx(&lc, k_small_front_grid, static_cast<const GraphFront*>(h_desc_dev_), db, ib,
                                         small_sb_.ptr, d_ctr, small_ws_.tiles.ptr, u64(small_ws_.tiles.cap), uk.ptr,
                                         uv.ptr, uop.ptr));
        } else {
            k_small_front<<<1, kSmallFrontThreads, kSmallFrontSmem, stream_>>>(
                h_desc_dev_, db, ib, d_ctr, small_ws_.tiles.ptr, small_ws_.tiles.cap, uk.ptr, uv.ptr, uop.ptr);
            GPMA_LAUNCH_CHECK();
        }
        // the rest of the chain: programmatic edges (GPMA_NO_PDL=1: ordinary ones)
        pdl_chain() = pdl_;
        launch_k(k_leaf_search_warp, dim3(kSmallGraphMax / 8), dim3(256), 0, stream_, uk.ptr, &d_ctr->n_unique, d_hdr,
                 num_leaves(), d_st, leaf_, ro_base(), ro_lo, ro_lo + num_vertices, ul.ptr);
        u32* pcur = nullptr;
        u32* pnext = pidx0.ptr;
        for (int level = 0; level < levels; ++level) {
            enqueue_level(level, kSmallGraphMax, pcur, pnext, touched.ptr, kSmallGraphMax, cfg, small_ws_, false, dummy);
            pcur = pnext;
            pnext = (pcur == pidx0.ptr) ? pidx1.ptr : pidx0.ptr;
        }
        // headers / row offsets of the rewritten ranges, left walks
        static_assert(sizeof(Ctr) % 8 == 0, "counters copied as words");
        // (left walks first: the refresh's last CTA closes the device span)
        if (empty_leaves != 0)  // headers of empty leaves inherit the next leaf's first key
            launch_k(k_left_walk, dim3(16), dim3(128), 0, stream_, touched.ptr, u64(0), static_cast<const u64*>(nullptr),
                     u64(0), touched_cb_, d_st, leaf_, d_hdr, &d_ctr->ngroups, static_cast<const ull*>(nullptr));
        launch_k(k_refresh_ranges, dim3(64), dim3(256), 0, stream_, rlist.ptr, &d_ctr->nrefresh, u64(0), d_keys, d_st,
                 cap_, leaf_, d_hdr, ro_base(), d_ctr, h_ctr_dev_);
        pdl_chain() = false;
    } catch (...) {
        pdl_chain() = false;
        cudaStreamEndCapture(stream_, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    GPMA_CUDA(cudaStreamEndCapture(stream_, &graph));
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    GPMA_CUDA(e);
}

int Pma::run_small_graph(const GraphFront& gf, const EngineCfg& cfg) {
    int db = 1;
    while (db < 32 && (1ull << db) < gf.nv) ++db;
    const int levels = std::min(kSmallGraphLevels, height_);
    const u64 n = gf.ni + gf.nd;
    const int multi = n > kSmallFrontMax ? 2 : n > std::min<u64>(small_onecta_, kSmallFrontMax) ? 1 : 0;
    small_sb_.reserve(kSbWords);  // (both variants' keys name it)
    auto key = small_graph_key(db, cfg, levels);
    if (!small_exec_[multi] || key != small_key_[multi]) {
        // every buffer the nodes touch, at its final size, before capture
        reserve_batch(kSmallGraphMax);
        small_ws_.tiles.reserve(64);
        small_ws_.epoch = 0;
        key = small_graph_key(db, cfg, levels);
        GPMA_CUDA(cudaMemsetAsync(small_sb_.ptr + kSbFlag, 0, 24, stream_));
        capture_small_graph(db, cfg, levels, multi);
        small_key_[multi] = key;
    }
    // read by the graph's first node (the previous replay is past it: its
    // done_seq is written at the very end of the graph)
    *h_desc_ = gf;
    h_desc_->seq = ++small_seq_;
    GPMA_CUDA(cudaGraphLaunch(small_exec_[multi], stream_));
    if (small_poll_) {
        // the last refresh CTA writes the counters, then done_seq, to
        // page-locked memory after every other kernel of the batch finished:
        // poll it (the stream's completion would arrive a few µs later); a
        // failed replay never writes it, so fall back to the stream sync,
        // which reports the error
        const volatile ull* done = &h_ctr->done_seq;
        const auto t0 = std::chrono::steady_clock::now();
        for (u32 spin = 0; *done != small_seq_; ++spin) {
            if ((spin & 1023u) == 1023u && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(200)) {
                GPMA_CUDA(cudaStreamSynchronize(stream_));
                if (*done != small_seq_) throw ApiError(PMA_ECUDA, "small-batch graph did not complete");
                break;
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    } else {
        GPMA_CUDA(cudaStreamSynchronize(stream_));
    }
    return levels;
}

void Pma::batch_update_device(const u64* dk, const u64* dv, const u8* dop, u64 n, const EngineCfg& cfg,
                              pma_stats* out, GraphFront* gf) {
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    NvtxScope nv_batch("gpma.apply_batch");
    NvtxStages nv_stage;
    pma_stats st;
    std::memset(&st, 0, sizeof(st));
    st.batch_size = n;
    st.num_levels = height_ + 1;
    last_ntouched = 0;
    last_ngroups0_ = last_nrest_ = 0;
    last_resized = false;
    timing = pma_timing{};
    touched_cb_ = 1;
    while ((1ull << touched_cb_) <= cap_) ++touched_cb_;  // begin < 2^cb
    touched_split_ = n;  // level-0 groups <= n
    const u64 leaf0 = leaf_;  // (a root grow may re-derive the leaf size)
    u64 launches = 0;
    const u64 writes_base = slot_writes;
    if (n == 0) {
        st.wall_ns = u64(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
        if (out) *out = st;
        return;
    }
    bool bucket = false;
    // this batch's stage events: the other set (a deferred record two
    // batches old is resolved first — its tail finished long ago)
    latest_pending_ = false;  // (`timing` now belongs to this batch)
    ev_set_ ^= 1;
    if (pend_[ev_set_]) resolve_set(ev_set_);
    const bool small_graph = gf && small_graph_ok(n, *gf);
    if (!small_graph) event(0);  // (a graph batch is timed by the graph's own %globaltimer stamps)
    // ---- small graph batches: the front end and the first rounds replayed
    // as one captured CUDA graph (no per-kernel launch cost, no host round
    // trip); the host loop below continues only if updates are still pending
    if (small_graph) nv_stage.next("gpma.small_graph");
    const int graph_levels = small_graph ? run_small_graph(*gf, cfg) : 0;
    const u64 graph_ns = graph_levels && h_ctr->gt1 > h_ctr->gt0 ? h_ctr->gt1 - h_ctr->gt0 : 0;
    if (graph_levels) {
        // (stage events skipped: a small batch's whole device span is the
        // graph, E(0) -> E(4); every host API call counts at this size)
    } else {
    // ---- 1. sort (stable, varying bits only) ----
    nv_stage.next("gpma.sort");
    GPMA_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(Ctr), stream_));
    sk_in.reserve(n);
    sk_out.reserve(n);
    si_in.reserve(n);
    si_out.reserve(n);
    int nbits = 0;
    int packed_ib = 0;
    if (gf) {
        // graph front end: pack + id check + compression in one pass; the
        // key layout is fixed by |V| (src, dst < 2^db), so no host round trip
        int db = 1;
        while (db < 32 && (1ull << db) < gf->nv) ++db;
        nbits = 2 * db;  // key = src << db | dst (guard deletes take the redo path)
        int ib = 1;
        while ((1ull << ib) < n) ++ib;
        while ((1ull << ib) <= n) ++ib;  // the all-ones index is reserved for deletes
        gf->opbit = 0;
        if (nbits + ib > 64) {
            // no room for the index: unweighted batches carry the op alone
            // (inserts precede deletes in arrival order, so the stable key
            // sort still yields arrival order; the weight is 1.0) — keys-only
            // passes of 8 B instead of (key, payload) pairs of 12 B
            if (!gf->iw && nbits + 1 <= 64) {
                ib = 1;
                gf->opbit = 1;
            } else {
                ib = 0;  // key + payload pairs
            }
        }
        packed_ib = ib;
        // leaf-bucket front end for large batches: the leaf of every update is
        // found up front and the batch counting-sorted by leaf (one scatter)
        // then ranked inside each leaf's short bucket — the same order as the
        // radix sort over all 2db + 1 key bits, in ~4 light passes instead of
        // one per 8 bits.  Skipped after a batch whose buckets overflowed.
        BucketArgs ba{};
        const u64 L = num_leaves();
        // Taken while the leaf headers stay L2-resident (the unsorted leaf
        // searches then hit L2; past that they are HBM-latency bound) and the
        // passes over the L leaf counters stay small next to the radix passes
        // over the n updates (measured: C2 and C3 gain, C4's 33.5M and C5's
        // 16.7M leaves lose).
        bucket = ro_base() && n >= kBucketMinBatch && n < (1ull << 31) && L <= kBucketMaxLeaves &&
                 L <= 8 * n && bucket_skip_ == 0 && buckets_;
        if (bucket_skip_) --bucket_skip_;
        if (bucket) {
            const u32* bc0 = bcnt.ptr;
            bcnt.reserve(L + 2);
            if (bcnt.ptr != bc0) bcnt_zero_ = 0;  // reallocated
            boff.reserve(L + 2);
            blf.reserve(n);
            bod.reserve(n);
            bslf.reserve(n);
            // the counters are left zeroed by the previous batch's scan
            if (bcnt_zero_ < L + 2) GPMA_CUDA(cudaMemsetAsync(bcnt.ptr, 0, bcnt.cap * sizeof(u32), stream_));
            bcnt_zero_ = 0;  // counted into below; zero again once the scan is enqueued
            ba = BucketArgs{d_hdr, L, d_st, leaf_, ro_base(), ro_lo, ro_lo + num_vertices, bcnt.ptr, blf.ptr, bod.ptr};
            k_prep_graph<true><<<grid_for(n, 256, 148 * 8), 256, 0, stream_>>>(*gf, db, ib, sk_in.ptr, si_in.ptr,
                                                                               d_ctr, ba);
        } else {
            k_prep_graph<false><<<grid_for(n, 256, 148 * 8), 256, 0, stream_>>>(*gf, db, ib, sk_in.ptr, si_in.ptr,
                                                                                d_ctr, ba);
        }
        GPMA_LAUNCH_CHECK();
        ++launches;
    } else {
        k_or_mask<<<grid_for(n, 256, 148 * 8), 256, 0, stream_>>>(dk, n, d_ctr);
        GPMA_LAUNCH_CHECK();
        ++launches;
        sync_ctr();
        const u64 mask = h_ctr->mask_or;
        BitRuns runs{};
        for (int bit = 0; bit < 64;) {
            if (!((mask >> bit) & 1)) {
                ++bit;
                continue;
            }
            int e = bit;
            while (e < 64 && ((mask >> e) & 1)) ++e;
            if (runs.n == 16) {  // too fragmented: fall back to the full key
                runs.n = 1;
                runs.lo[0] = 0;
                runs.len[0] = 64;
                runs.out[0] = 0;
                nbits = 64;
                break;
            }
            runs.lo[runs.n] = bit;
            runs.len[runs.n] = e - bit;
            runs.out[runs.n] = nbits;
            nbits += e - bit;
            runs.n++;
            bit = e;
        }
        k_compress<<<grid_for(n, 256, 148 * 8), 256, 0, stream_>>>(dk, dop, n, runs, sk_in.ptr, si_in.ptr);
        GPMA_LAUNCH_CHECK();
        ++launches;
    }
    const u64* sorted_ck = sk_in.ptr;
    const u32* sorted_ci = si_in.ptr;
    if (bucket) {
        const u64 L = num_leaves();
        // (the bucket kernels chained by programmatic edges, as the rounds)
        bbig.reserve(n / (kSmallRun + 1) + 1);
        const bool pairs = packed_ib == 0;
        static const unsigned scat_res = resident_grid(k_bucket_scatter, 256);
        static const unsigned sort_res = resident_grid(k_bucket_sort_small, 256);
        pdl_chain() = pdl_;
        try {
            exclusive_sum(stream_, ws, bcnt.ptr, boff.ptr, L + 2, bcnt.ptr);  // (leaves bcnt[0, L + 2) zeroed)
            bcnt_zero_ = bcnt.cap;  // (entries past L + 2 were never counted into)
            launch_k(k_bucket_scatter, dim3(grid_for(n, 256, scat_res)), dim3(256), 0, stream_,
                     static_cast<const u64*>(sk_in.ptr), static_cast<const u32*>(pairs ? si_in.ptr : nullptr),
                     static_cast<const u32*>(blf.ptr), static_cast<const u32*>(bod.ptr),
                     static_cast<const u32*>(boff.ptr), n, sk_out.ptr, si_out.ptr);
            launch_k(k_bucket_sort_small, dim3(grid_for((L + 1 + 31) / 32 * 32, 256, sort_res)), dim3(256), 0,
                     stream_, static_cast<const u64*>(sk_out.ptr), static_cast<const u32*>(pairs ? si_out.ptr : nullptr),
                     static_cast<const u32*>(boff.ptr), L, sk_in.ptr, si_in.ptr, bslf.ptr, bbig.ptr, d_ctr);
            launch_k(k_bucket_sort_big, dim3(148 * 2), dim3(256), 0, stream_, static_cast<const u64*>(sk_out.ptr),
                     static_cast<const u32*>(pairs ? si_out.ptr : nullptr), static_cast<const u32*>(boff.ptr),
                     static_cast<const u32*>(bbig.ptr), static_cast<const ull*>(&d_ctr->nbig_buckets), sk_in.ptr,
                     si_in.ptr);
        } catch (...) {
            pdl_chain() = false;
            throw;
        }
        pdl_chain() = false;
        launches += 5;
    } else if (packed_ib && n > 1) {
        // keys-only: the arrival index rides in the low bits below the key
        // (histogram and digit passes chained by PDL edges)
        pdl_chain() = pdl_;
        int alt = 0;
        try {
            alt = radix_sort(stream_, rws, sk_in.ptr, sk_out.ptr, nullptr, nullptr, n, packed_ib, packed_ib + nbits,
                             &launches);
        } catch (...) {
            pdl_chain() = false;
            throw;
        }
        pdl_chain() = false;
        sorted_ck = alt ? sk_out.ptr : sk_in.ptr;
    } else if (nbits > 0 && n > 1) {
        pdl_chain() = pdl_;
        int alt = 0;
        try {
            alt = radix_sort(stream_, rws, sk_in.ptr, sk_out.ptr, si_in.ptr, si_out.ptr, n, 0, nbits, &launches);
        } catch (...) {
            pdl_chain() = false;
            throw;
        }
        pdl_chain() = false;
        sorted_ck = alt ? sk_out.ptr : sk_in.ptr;
        sorted_ci = alt ? si_out.ptr : si_in.ptr;
    }
    nv_stage.next("gpma.resolve_search");
    // ---- 2+3. resolve duplicates (run ends -> unique updates) fused with the
    // leaf assignment of each unique key (computed once per batch) ----
    uk.reserve(n + 4);
    uv.reserve(n + 4);
    uop.reserve(n + 32);  // k_commit_leaf stages 16-byte aligned runs of uk / uv / uop
    ul.reserve(n);
    // (no event record here: the compaction stays on a programmatic edge
    // from the sort and stamps the stage boundary itself, Ctr::t_dedup)
    pdl_chain() = pdl_;
    {
        const u64* ck = sorted_ck;
        const u32* ci = sorted_ci;
        const u64* kk = dk;
        const u64* vv = dv;
        const double* gw = gf ? gf->iw : nullptr;
        const int gdb = gf ? nbits / 2 : 0;  // graph layout: key = src << gdb | dst
        const u64 skipkey = gf ? (1ull << nbits) : ~0ull;
        const int pib = packed_ib;
        const u64 pmask = (1ull << pib) - 1;

        // sorted element i -> compressed key / payload (arrival index << 1 | is_insert)
        auto KEY = [=] __device__(ull i) -> u64 { return pib ? (ck[i] >> pib) : ck[i]; };
        auto PAY = [=] __device__(ull i) -> u32 {
            if (!pib) return ci[i];
            const u32 a = u32(ck[i] & pmask);
            return (a << 1) | (a != u32(pmask) ? 1u : 0u);  // all-ones index = a delete
        };
        u64* o_k = uk.ptr;
        u64* o_v = uv.ptr;
        u8* o_o = uop.ptr;
        u32* o_l = ul.ptr;
        const u32* slf = bucket ? bslf.ptr : nullptr;  // leaf-bucket front end: leaves already known
        Ctr* ctr = d_ctr;
        run_compact_tile(
            stream_, ws, nullptr, n, n,
            [=] __device__(ull i) {
                const u64 c = KEY(i);
                return ((i + 1 == n) || KEY(i + 1) != c) && c < skipkey;
            },
            [=] __device__(ull i0, ull nn, unsigned fm, const ull* xs) {
                // last insert of each equal-key run wins (segment_engine.hpp:346-363);
                // the op rides in the sort payload and, for graphs, the key is the
                // decompressed sort key — only insert values are gathered
#pragma unroll
                for (int j = 0; j < kScanItems; ++j) {
                    if (!((fm >> j) & 1u)) continue;
                    const ull i = i0 + ull(j) * kScanThreads;
                    const u64 c = KEY(i);
                    const u32 p0 = PAY(i);
                    u32 p = p0;
                    if (!(p & 1u) && i > 0 && KEY(i - 1) == c) {  // delete at a run end: any earlier insert?
                        for (long long t = (long long)i - 1; t >= 0 && KEY(t) == c; --t) {
                            const u32 q = PAY(t);
                            if (q & 1u) {
                                p = q;
                                break;
                            }
                        }
                    }
                    const u32 a = p >> 1;
                    const bool ins = p & 1u;
                    u64 key, val = 0;
                    if (gdb) {
                        key = ((c >> gdb) << 32) | (c & ((1ull << gdb) - 1));
                        if (ins) val = u64(__double_as_longlong(gw ? gw[a] : 1.0));
                    } else {
                        key = kk[p0 >> 1];
                        if (ins && vv) val = vv[a];
                    }
                    o_k[xs[j]] = key;
                    o_v[xs[j]] = val;
                    o_o[xs[j]] = ins ? kOpInsert : kOpDelete;
                    if (slf) o_l[xs[j]] = slf[i];
                }
            },
            [=] __device__(ull total) {
                ctr->n_unique = total;
                // pending count of round 0 = the unique updates, or 0 when the
                // graph front end flagged a bad insert id, an out-of-layout
                // delete or an overflowed leaf bucket: every round is then a
                // no-op (nothing is mutated) and the batch is rejected or redone
                // after the first host sync — no round trip before the rounds
                ctr->np[0] = (ctr->bad_ins || ctr->oor || ctr->bigrun) ? 0ull : total;
            },
            &d_ctr->t_dedup);
        pdl_chain() = false;
        ++launches;
        if (!bucket) {
            // leaf assignment (pma.hpp:234-289), once per batch
            // (a programmatic edge from the compaction: it overlaps the launch)
            pdl_chain() = pdl_;
            try {
                launch_k(k_leaf_search_sorted, dim3(grid_for(n, 256, 148 * 8)), dim3(256), 0, stream_,
                         static_cast<const u64*>(uk.ptr), static_cast<const ull*>(&d_ctr->n_unique),
                         static_cast<const u64*>(d_hdr), num_leaves(), static_cast<const u8*>(d_st), leaf_,
                         static_cast<const u64*>(ro_base()), ro_lo, ro_lo + num_vertices, ul.ptr);
            } catch (...) {
                pdl_chain() = false;
                throw;
            }
            pdl_chain() = false;
            ++launches;
        }
    }
    }  // front end
    pidx0.reserve(n);
    pidx1.reserve(n);
    gid.reserve(n);
    gstart.reserve(n + 1);
    gseg.reserve(n + 1);
    gflag.reserve(n);
    touched.reserve(2 * n + 2);
    rlist.reserve(2 * n + 4);
    // ---- 4. rounds ----
    nv_stage.next("gpma.rounds");
    // Rounds are device-driven: every kernel reads its counts from d_ctr, the
    // per-level stats land in d_ctr->lvl_*, so while the pending list is large
    // (more rounds are near certain) the next round is launched without a host
    // round trip; the host syncs after odd levels, before the root, and
    // whenever the pending list is small.
    u64 npend = n;  // host-known upper bound of the pending count
    u64* touched_ptr = touched.ptr;
    u64 ntouched = 0;
    u32* pcur = nullptr;  // round 0: pending = all unique updates in order (identity)
    u32* pnext = pidx0.ptr;
    float seg_ms = 0.f;
    bool root_done = false;
    int synced_upto = -1;  // per-level stats collected for levels <= synced_upto
    int level0 = 0;
    if (graph_levels) {
        // the graph ran levels [0, graph_levels) and brought the counters back
        for (int l = 0; l < graph_levels; ++l) {
            if (l < 16) {
                timing.level_bytes[l] += h_ctr->lvl_bytes[l] - (l > 0 ? h_ctr->lvl_bytes[l - 1] : 0);
                timing.level_groups[l] += h_ctr->lvl_groups[l];
                timing.level_big[l] += h_ctr->lvl_big[l];
                timing.level_max_slice[l] = std::max<u64>(timing.level_max_slice[l], h_ctr->lvl_maxslice[l]);
            }
            if (h_ctr->lvl_npend[l] > 0) st.rounds++;
            st.segments_per_level[l] += h_ctr->lvl_committed[l];
        }
        synced_upto = graph_levels - 1;
        ntouched = h_ctr->ntouched_next;
        npend = h_ctr->np[graph_levels & 1];
        pcur = ((graph_levels - 1) & 1) == 0 ? pidx0.ptr : pidx1.ptr;  // the last advance's output
        pnext = (pcur == pidx0.ptr) ? pidx1.ptr : pidx0.ptr;
        level0 = graph_levels;
        launches += 1;
    }
    const bool host_levels = npend > 0;
    if (graph_levels && host_levels) event(0);  // the host-loop levels' span (added to the graph's)
    // speculative tail before each sync of the host loop (not after the root
    // path, which rebuilds headers in closed form; GPMA_NO_SPEC_TAIL=1 turns it off)
    static const bool no_spec_tail = [] {
        const char* e = std::getenv("GPMA_NO_SPEC_TAIL");
        return e && *e && *e != '0';
    }();
    const bool spec_tail_ok = !no_spec_tail;
    bool spec_tail = false, spec_walk = false;
    if (npend > 0) {
        for (int level = level0;; ++level) {
            // the level's kernels chained by programmatic edges (each waits
            // for its predecessor in pdl_enter; the launch overlaps its tail)
            pdl_chain() = pdl_;
            try {
                enqueue_level(level, npend, pcur, pnext, touched_ptr, n, cfg, ws, true, launches);
            } catch (...) {
                pdl_chain() = false;
                throw;
            }
            pdl_chain() = false;
            pcur = pnext;
            pnext = (pcur == pidx0.ptr) ? pidx1.ptr : pidx0.ptr;
            const bool speculate = npend >= (1u << 16) && (level & 1) == 0 && level < height_;
            if (speculate) continue;  // next round straight away; stats at the next sync
            if (spec_tail_ok) {
                // the counters first (the host waits for them only), then
                // this may be the last level: the tail (header / row-offset
                // refresh, left walks, end event) goes in before the sync,
                // gated by the device counts, so the GPU does not idle while
                // the host learns that nothing is left.  Both passes recompute
                // from the current slots, so when more levels follow they are
                // simply redone at the end.
                GPMA_CUDA(cudaMemcpyAsync(h_ctr, d_ctr, sizeof(Ctr), cudaMemcpyDeviceToHost, stream_));
                event(5);
                if (!graph_levels) event(3);
                k_refresh_ranges<<<148 * 4, 256, 0, stream_>>>(rlist.ptr, &d_ctr->nrefresh, 0, d_keys, d_st, cap_,
                                                              leaf_, d_hdr, ro_base());
                GPMA_LAUNCH_CHECK();
                spec_walk = empty_leaves != 0;
                if (spec_walk) {
                    k_left_walk<<<148 * 8, 128, 0, stream_>>>(touched_ptr, 0, touched_ptr + touched_split_, 0,
                                                              touched_cb_, d_st, leaf_, d_hdr, &d_ctr->lvl_groups[0],
                                                              &d_ctr->ntouched_next);
                    GPMA_LAUNCH_CHECK();
                }
                event(4);
                launches += spec_walk ? 2 : 1;
                spec_tail = true;
                GPMA_CUDA(cudaEventSynchronize(E(5)));
            } else {
                sync_ctr();
            }
            for (int l = synced_upto + 1; l <= level; ++l) {
                float ms = 0.f;
                if (l < 16 && level_events_)  // (cross-check mode: CUDA events around the commit kernels)
                    cudaEventElapsedTime(&ms, lev_ev_[2 * l], lev_ev_[2 * l + 1]);
                else if (l < 16 && h_ctr->lvl_tmin[l] && h_ctr->lvl_tmax[l])
                    ms = float(double(h_ctr->lvl_tmax[l] - ~h_ctr->lvl_tmin[l]) * 1e-6);
                seg_ms += ms;
                if (l < 16) {
                    timing.level_ms[l] += ms;
                    timing.level_bytes[l] += h_ctr->lvl_bytes[l] - (l > 0 ? h_ctr->lvl_bytes[l - 1] : 0);
                    timing.level_groups[l] += h_ctr->lvl_groups[l];
                    timing.level_big[l] += h_ctr->lvl_big[l];
                    timing.level_max_slice[l] = std::max<u64>(timing.level_max_slice[l], h_ctr->lvl_maxslice[l]);
                }
                if (h_ctr->lvl_npend[l] > 0) st.rounds++;
                st.segments_per_level[l] += h_ctr->lvl_committed[l];
            }
            synced_upto = level;
            ntouched = h_ctr->ntouched_next;
            const u64 left = h_ctr->np[(level + 1) & 1];
            if (left == 0) break;
            spec_tail = false;  // more levels: the tail is redone after them
            npend = left;
            if (level == height_) {
                // root path: everything left is the single root group
                GPMA_CUDA(cudaMemcpyAsync(&d_ctr->npend, &d_ctr->np[(level + 1) & 1], sizeof(ull),
                                          cudaMemcpyDeviceToDevice, stream_));
                // apply the counters of the finished rounds first
                valid_count = u64((long long)valid_count + h_ctr->valid_delta);
                tombstone_count = u64((long long)tombstone_count + h_ctr->tomb_delta);
                slot_writes += h_ctr->slot_writes;
                st.deletes_missed += h_ctr->missed;
                st.tombstones_added += h_ctr->tomb_added;
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->valid_delta, 0, sizeof(long long) * 2, stream_));
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->missed, 0, sizeof(ull) * 5, stream_));
                // inserts in the root slice
                {
                    const u8* uo = uop.ptr;
                    const u32* pp = pcur;
                    Ctr* ctr = d_ctr;
                    GPMA_CUDA(cudaMemsetAsync(&d_ctr->root_ins, 0, sizeof(ull), stream_));
                    run_compact(
                        stream_, ws, &d_ctr->npend, 0, npend, [=] __device__(ull p) { return uo[pp[p]] == kOpInsert; },
                        [=] __device__(ull, unsigned, ull) {}, [=] __device__(ull total) { ctr->root_ins = total; });
                }
                sync_ctr();
                const u64 ins = h_ctr->root_ins;
                while (valid_count + ins > mx_[height_]) {
                    rebuild_at_capacity(cap_ << 1);
                    st.grow_events++;
                }
                // forced merge at the (possibly grown) root
                ensure_slot_scratch();
                ik.reserve(n);
                iv.reserve(n);
                ir.reserve(n);
                {
                    u64* dek = ek.ptr;
                    u64* dev = ev.ptr;
                    u32* des = es.ptr;
                    u8* mf = mflag.ptr;
                    const u64* kk = d_keys;
                    const u64* vv = d_vals;
                    const u8* ss = d_st;
                    Ctr* ctr = d_ctr;
                    run_compact(
                        stream_, ws, nullptr, cap_, cap_, [=] __device__(ull i) { return ss[i] == kValid; },
                        [=] __device__(ull i, unsigned f, ull x) {
                            if (f) {
                                dek[x] = kk[i];
                                dev[x] = vv[i];
                                des[x] = u32(i);
                                mf[x] = 0;
                            }
                        },
                        [=] __device__(ull total) { ctr->nv = total; });
                    k_root_ranks<<<grid_for(npend, 256, 148 * 8), 256, 0, stream_>>>(
                        uk.ptr, uop.ptr, pcur, &d_ctr->npend, dek, &d_ctr->nv, mf, d_ctr);
                    GPMA_LAUNCH_CHECK();
                    // ordered insert list with ranks
                    const u64* uuk = uk.ptr;
                    const u64* uuv = uv.ptr;
                    const u8* uuo = uop.ptr;
                    const u32* pp = pcur;
                    u64* ikk = ik.ptr;
                    u64* ivv = iv.ptr;
                    u32* irr = ir.ptr;
                    const ull* nvp = &d_ctr->nv;
                    run_compact(
                        stream_, ws, &d_ctr->npend, 0, npend, [=] __device__(ull p) { return uuo[pp[p]] == kOpInsert; },
                        [=] __device__(ull p, unsigned f, ull x) {
                            if (!f) return;
                            const u64 u = uuk[pp[p]];
                            ikk[x] = u;
                            ivv[x] = uuv[pp[p]];
                            irr[x] = u32(lower_bound_dev(dek, *nvp, u));
                        },
                        [=] __device__(ull total) { ctr->nins = total; });
                    // matched-before prefix over E
                    u32* mbv = mb.ptr;
                    run_compact(
                        stream_, ws, &d_ctr->nv, 0, cap_ + 1, [=] __device__(ull j) { return mf[j] != 0; },
                        [=] __device__(ull j, unsigned, ull x) { mbv[j] = u32(x); },
                        [=] __device__(ull total) {
                            ctr->nmatched = total;
                            mbv[ctr->nv] = u32(total);
                        });
                    // (nv == 0: mb[0] is seeded after the sync below, before the
                    // insert scatter reads mb[r] for r <= nv)
                    k_root_scatter_surv<<<grid_for(cap_, 256, 148 * 16), 256, 0, stream_>>>(
                        dek, dev, &d_ctr->nv, mf, mbv, irr, &d_ctr->nins, ok.ptr, ov.ptr);
                    GPMA_LAUNCH_CHECK();
                    sync_ctr();
                    if (h_ctr->nv == 0) {
                        const u32 zero = 0;
                        GPMA_CUDA(cudaMemcpyAsync(mbv, &zero, 4, cudaMemcpyHostToDevice, stream_));
                        h_ctr->nmatched = 0;
                        GPMA_CUDA(cudaMemsetAsync(&d_ctr->nmatched, 0, sizeof(ull), stream_));
                    }
                    k_root_scatter_ins<<<grid_for(npend, 256, 148 * 8), 256, 0, stream_>>>(
                        ikk, ivv, irr, &d_ctr->nins, mbv, ok.ptr, ov.ptr, d_ctr);
                    GPMA_LAUNCH_CHECK();
                    if (cfg.large_for(cap_)) {
                        GPMA_CUDA(cudaMemsetAsync(&d_ctr->moves, 0, sizeof(ull), stream_));
                        run_compact(
                            stream_, ws, &d_ctr->nv, 0, cap_ + 1, [=] __device__(ull j) { return mf[j] != 1; },
                            [=] __device__(ull j, unsigned f, ull x) {
                                if (f && u64(des[j]) != x) atomicAdd(&ctr->moves, 1ull);
                            },
                            NoFin{});
                    }
                    sync_ctr();
                }
                const u64 k = h_ctr->k;
                const u64 moves = cfg.large_for(cap_) ? h_ctr->moves : 0;
                st.deletes_missed += h_ctr->missed;
                // write the root: every slot rewritten (place_evenly / commit_in_place)
                k_place_evenly<<<grid_for(cap_, 256, 148 * 32), 256, 0, stream_>>>(d_keys, d_vals, d_st, 0, cap_,
                                                                                   ok.ptr, ov.ptr, nullptr, k);
                GPMA_LAUNCH_CHECK();
                slot_writes += cap_ + moves;
                valid_count = k;
                tombstone_count = 0;
                empty_leaves = k >= num_leaves() ? 0 : (long long)(num_leaves() - k);
                headers_closed_form(ok.ptr, k);
                root_done = true;
                st.num_levels = height_ + 1;
                st.segments_per_level[height_]++;
                st.rounds++;
                if (cfg.eager && prof_.allow_shrink) {
                    bool shrunk = false;
                    while (cap_ > 16 && valid_count < mn_[height_]) {
                        rebuild_at_capacity(cap_ >> 1);
                        shrunk = true;
                    }
                    if (shrunk) st.shrink_events++;
                }
                st.resized = st.grow_events > 0 || st.shrink_events > 0;
                if (!st.resized) {
                    const u64 pair[2] = {0, cap_};
                    int lg = 0;
                    while ((1ull << lg) < pair[1]) ++lg;
                    const u64 word = (u64(lg) << touched_cb_) | pair[0];
                    GPMA_CUDA(cudaMemcpyAsync(touched_ptr + touched_split_ + ntouched, &word, 8, cudaMemcpyHostToDevice,
                                              stream_));
                    GPMA_CUDA(cudaStreamSynchronize(stream_));  // (word lives on the host stack)
                    ntouched++;
                }
                // counters already applied; clear device deltas
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->valid_delta, 0, sizeof(long long) * 2, stream_));
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->empty_delta, 0, sizeof(long long), stream_));
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->nrefresh, 0, sizeof(ull), stream_));
                GPMA_CUDA(cudaMemsetAsync(&d_ctr->missed, 0, sizeof(ull) * 5, stream_));
                sync_ctr();
                break;
            }
        }
    }
    // apply device counters
    valid_count = u64((long long)valid_count + h_ctr->valid_delta);
    tombstone_count = u64((long long)tombstone_count + h_ctr->tomb_delta);
    slot_writes += h_ctr->slot_writes;
    st.deletes_missed += h_ctr->missed;
    st.tombstones_added += h_ctr->tomb_added;
    timing.merge_slots = h_ctr->merge_slots;
    timing.commit_bytes = h_ctr->commit_bytes;
    timing.tombstone_flips = st.tombstones_added;
    if (!graph_levels && !spec_tail) event(3);
    // ---- 5. refresh leaf headers / row offsets ----
    nv_stage.next("gpma.refresh");
    // The warp tier refreshed dense segments in place; sparse and CTA-tier
    // segments were queued on rlist; left walks are needed only while empty
    // leaves exist (their headers inherit the next leaf's first key).
    last_resized = st.resized;
    // touched ranges: level 0's merges (dense words) + the appended rest
    const u64 ntouched0 = h_ctr->lvl_groups[0] ? h_ctr->lvl_merge[0] / leaf0 : 0;
    last_ngroups0_ = h_ctr->lvl_groups[0];
    last_nrest_ = ntouched;
    last_ntouched = ntouched0 + ntouched;
    if (root_done) {
        // whole array re-placed: headers rebuilt in closed form already
        if (d_row_offsets) rebuild_row_offsets_full();
        ++launches;
    } else if (graph_levels && !host_levels) {
        // the graph refreshed the headers / row offsets and walked left
        if (empty_leaves >= 0) empty_leaves += h_ctr->empty_delta;
    } else if (spec_tail) {
        // refreshed (and walked, if empty leaves were known) before the last
        // sync; a walk is still due if this batch created the first empty leaves
        if (empty_leaves >= 0) empty_leaves += h_ctr->empty_delta;
        if (!spec_walk && last_ntouched > 0 && empty_leaves != 0) {
            k_left_walk<<<grid_for(last_ngroups0_ + ntouched, 128, 148 * 8), 128, 0, stream_>>>(
                touched_ptr, last_ngroups0_, touched_ptr + touched_split_, ntouched, touched_cb_, d_st, leaf_, d_hdr);
            GPMA_LAUNCH_CHECK();
            ++launches;
            spec_tail = false;  // (synchronise below)
        }
    } else {
        if (empty_leaves >= 0) empty_leaves += h_ctr->empty_delta;
        const u64 nref = h_ctr->nrefresh;
        if (nref > 0) {
            k_refresh_ranges<<<grid_for(nref * 32, 256, 148 * 16), 256, 0, stream_>>>(
                rlist.ptr, nullptr, nref, d_keys, d_st, cap_, leaf_, d_hdr, ro_base());
            GPMA_LAUNCH_CHECK();
            ++launches;
        }
        if (last_ntouched > 0 && empty_leaves != 0) {
            k_left_walk<<<grid_for(last_ngroups0_ + ntouched, 128, 148 * 8), 128, 0, stream_>>>(
                touched_ptr, last_ngroups0_, touched_ptr + touched_split_, ntouched, touched_cb_, d_st, leaf_,
                                                                               d_hdr);
            GPMA_LAUNCH_CHECK();
            ++launches;
        }
    }
    // a host-loop batch whose tail was enqueued before the last sync returns
    // now: the counters are on the host, the refresh finishes on the stream
    // (every later call on this Pma is ordered behind it) — the host's return
    // and the next batch's set-up overlap it
    const bool async_tail = spec_tail && !graph_levels;
    if ((!graph_levels || host_levels) && !async_tail) {  // (a graph-only batch: synchronised already)
        if (!spec_tail) event(4);  // (a speculative tail recorded it)
        GPMA_CUDA(cudaStreamSynchronize(stream_));
    }
    st.slot_writes = slot_writes - writes_base;
    st.num_touched_ranges = last_ntouched;
    st.segment_phase_ns = u64(double(seg_ms) * 1e6);
    float a = 0, b = 0, c = 0, d = 0;
    if (graph_levels) {
        // the graph (its %globaltimer span) + any host-loop levels: reported as one stage
        a = float(double(graph_ns) * 1e-6);
        float hl = 0;
        if (host_levels) cudaEventElapsedTime(&hl, E(0), E(4));
        a += hl;
    } else {
        // front end and resolve from the kernels' stage stamps, the rest from
        // the events ev0 -> ev3 -> ev4 (a deferred batch: when resolved)
        auto t = [](ull x) { return x ? ~x : 0ull; };
        const ull tf = t(h_ctr->t_front), td = t(h_ctr->t_dedup), tr = t(h_ctr->t_rounds);
        a = (tf && td >= tf) ? float(double(td - tf) * 1e-6) : 0.f;
        b = (td && tr >= td) ? float(double(tr - td) * 1e-6) : 0.f;
        if (!async_tail) {
            float dev03 = 0;
            cudaEventElapsedTime(&dev03, E(0), E(3));
            cudaEventElapsedTime(&d, E(3), E(4));
            c = std::max(0.f, dev03 - a - b);
        }
    }
    timing.sort_ms = a;
    timing.search_ms = b;
    timing.rounds_ms = c;
    timing.refresh_ms = d;
    timing.device_ms = a + b + c + d;
    timing.kernel_launches = launches;
    timing.front_end = bucket ? 1 : 0;
    if (async_tail) {
        pend_t_[ev_set_] = timing;
        pend_[ev_set_] = true;
        latest_pending_ = true;
    } else {
        accumulate_timing(timing);
    }
    if (gf) {
        gf->guard_deletes = h_ctr->gdel;
        gf->bad_insert = h_ctr->bad_ins ? (long long)(~h_ctr->bad_ins) : -1;
        if (gf->bad_insert >= 0) return;  // caller throws; the gated rounds mutated nothing
        if (h_ctr->oor) {
            // a delete key outside the |V|-derived layout: pack the batch
            // without its guard deletes (the reference drops them before the
            // engine) and redo it on the generic key-reduction path
            const GraphFront f = *gf;
            u64* bk = f.bk;
            u64* bv = f.bv;
            u8* bo = f.bo;
            Ctr* ctr = d_ctr;
            run_compact(
                stream_, ws, nullptr, n, n,
                [=] __device__(ull i) {
                    if (f.mk) return !(f.mk[i] >> 63) || dst_of(f.mk[i]) != u32(kGuardDst);
                    return i < f.ni || f.dd[i - f.ni] != u32(kGuardDst);
                },
                [=] __device__(ull i, unsigned fl, ull x) {
                    if (!fl) return;
                    const bool ins = f.mk ? !(f.mk[i] >> 63) : i < f.ni;
                    if (f.mk) bk[x] = f.mk[i] & ~(1ull << 63);
                    else bk[x] = ins ? pack_edge(f.is[i], f.id[i]) : pack_edge(f.ds[i - f.ni], f.dd[i - f.ni]);
                    bv[x] = ins ? u64(__double_as_longlong(f.iw ? f.iw[i] : 1.0)) : 0;
                    bo[x] = ins ? kOpInsert : kOpDelete;
                },
                [=] __device__(ull total) { ctr->nt = total; });
            sync_ctr();
            const u64 m = h_ctr->nt;
            batch_update_device(bk, bv, bo, m, cfg, out, nullptr);
            if (out) out->batch_size = n;  // the caller subtracts the guard deletes
            return;
        }
        if (h_ctr->bigrun) {
            // a leaf bucket too long to rank in place (many updates between two
            // neighbouring keys, e.g. a burst into an empty vertex): the gated
            // rounds mutated nothing; redo through the radix sort and keep it
            // for the next batches
            bucket_skip_ = kBucketCooldown;
            batch_update_device(dk, dv, dop, n, cfg, out, gf);
            timing.front_end = 2;
            return;
        }
    }
    if (check_rounds_) {
        sync_ctr();
        if (h_ctr->round_overlap)
            throw ApiError(PMA_ELOGIC, "segment engine: overlapping segments in one round (" +
                                           std::to_string(h_ctr->round_overlap) + " groups)");
    }
    st.wall_ns = u64(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
    if (out) *out = st;
}

// Every per-batch buffer sized for batches of up to n updates (and the
// slot-space scratch of the CTA/grid tiers), so no allocation lands inside
// a later batch.  Buffers only grow; batch_update sizes them anyway.
void Pma::reserve_batch(u64 n) {
    if (n == 0) return;
    sk_in.reserve(n);
    sk_out.reserve(n);
    si_in.reserve(n);
    si_out.reserve(n);
    const u64 L = num_leaves();
    if (ro_base() && n >= kBucketMinBatch && L <= kBucketMaxLeaves) {
        bcnt.reserve(L + 2);
        boff.reserve(L + 2);
        blf.reserve(n);
        bod.reserve(n);
        bslf.reserve(n);
        bbig.reserve(n / (kSmallRun + 1) + 1);
    }
    uk.reserve(n + 4);
    uv.reserve(n + 4);
    uop.reserve(n + 32);
    ul.reserve(n);
    pidx0.reserve(n);
    pidx1.reserve(n);
    gid.reserve(n);
    gstart.reserve(n + 1);
    gseg.reserve(n + 1);
    gflag.reserve(n);
    touched.reserve(2 * n + 2);
    tw0.reserve(n + 1);
    tw1.reserve(2 * n + 2);
    rlist.reserve(2 * n + 4);
    ik.reserve(n);
    iv.reserve(n);
    ir.reserve(n);
    biglist.reserve(n + 1);
    ensure_slot_scratch();
    // look-back words of the compactions / exclusive sums and the radix
    // sort's per-tile digit words (the first batch would allocate them)
    const u64 tiles = std::max<u64>(n, L + 2) / kScanTile + 2;
    if (tiles > ws.tiles.cap) {
        ws.tiles.reserve(tiles);
        GPMA_CUDA(cudaMemsetAsync(ws.tiles.ptr, 0, ws.tiles.cap * sizeof(ull), stream_));
    }
    const u64 rt = (n / kRadixTile + 2) * kRadixBins;
    if (rt > rws.status.cap) {
        rws.status.reserve(rt);
        GPMA_CUDA(cudaMemsetAsync(rws.status.ptr, 0, rws.status.cap * sizeof(ull), stream_));
    }
    rws.hist.reserve(kRadixMaxPasses * kRadixBins);
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

// touched word (log2(size) << cb) | begin -> (begin, end): every range is a
// whole aligned segment of power-of-two size, so the word orders ranges by
// size then begin and decodes back exactly.
__global__ void k_touched_pairs(const u64* __restrict__ words, u64 n, int cb, u64* __restrict__ pairs) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        const u64 x = words[i];
        const u64 b = x & ((1ull << cb) - 1);
        reinterpret_cast<ulonglong2*>(pairs)[i] = make_ulonglong2(b, b + (1ull << (x >> cb)));
    }
}

void Pma::touched_ranges(u64* pairs, size_t capn, size_t* count) {
    *count = last_ntouched;
    const size_t n = std::min<size_t>(capn, last_ntouched);
    if (!n || !pairs) return;
    // the reference's order (rounds in level order = by size, segments
    // ascending inside a round): level 0's dense words by one ordered
    // compaction (groups are in segment order), then the few words of the
    // higher levels sorted (they are larger ranges, so they follow)
    const u64 m = last_ntouched;
    tw0.reserve(m + 1);
    tw1.reserve(2 * m + 2);  // sort alternate, then the decoded pairs
    const u64* t0 = touched.ptr;
    u64* o = tw0.ptr;
    if (last_ngroups0_)
        run_compact(
            stream_, ws, nullptr, last_ngroups0_, last_ngroups0_, [=] __device__(ull i) { return t0[i] != ~0ull; },
            [=] __device__(ull i, unsigned f, ull x) {
                if (f) o[x] = t0[i];
            },
            NoFin{});
    const u64 n0 = m - last_nrest_;
    const u64* words = tw0.ptr;
    if (last_nrest_) {
        GPMA_CUDA(cudaMemcpyAsync(tw0.ptr + n0, touched.ptr + touched_split_, last_nrest_ * 8,
                                  cudaMemcpyDeviceToDevice, stream_));
        const int alt = radix_sort(stream_, rws, tw0.ptr + n0, tw1.ptr + n0, nullptr, nullptr, last_nrest_, 0,
                                   touched_cb_ + 6);
        if (alt)
            GPMA_CUDA(cudaMemcpyAsync(tw0.ptr + n0, tw1.ptr + n0, last_nrest_ * 8, cudaMemcpyDeviceToDevice,
                                      stream_));
    }
    // decoded into (b, e) pairs on the device: a page-locked caller array is
    // written in place by the decoding kernel (PCIe writes from the SMs run
    // at ~2x the copy engine's D2H rate measured here), anything else gets
    // one DMA from a device staging buffer
    u64* dst = tw1.ptr;
    bool direct = false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, pairs) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer &&
        (reinterpret_cast<uintptr_t>(at.devicePointer) & 15) == 0 && direct_touched_) {
        dst = static_cast<u64*>(at.devicePointer);
        direct = true;
    } else {
        (void)cudaGetLastError();  // (pageable memory: the query's error is not the caller's)
    }
    k_touched_pairs<<<grid_for(n, 256, 148 * 8), 256, 0, stream_>>>(words, n, touched_cb_, dst);
    GPMA_LAUNCH_CHECK();
    if (!direct) GPMA_CUDA(cudaMemcpyAsync(pairs, tw1.ptr, n * 16, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

// try_insert_plus (segment_engine.hpp:320-341) for ONE group on the device:
// the group is set up exactly as a round of the batch engine would hand it to
// the CTA tier (slice = sorted, duplicate-resolved updates of segment `seg`
// at `level`), decided and committed by k_commit_cta, then the counters and
// the leaf headers / row offsets are brought up to date as after a round.
__global__ void k_group_leaves(const u64* __restrict__ uk, u64 n, const u64* __restrict__ hdr, u64 L,
                               const u8* __restrict__ st, u64 leaf, const u64* __restrict__ ro, u64 rlo, u64 rhi,
                               u64 first, u64 last, u32* __restrict__ ul) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        // a key whose leaf lies outside the segment cannot be in it: the
        // clamped leaf never holds it (the reference scans [b, e) only)
        u64 l = leaf_for_key(uk[i], hdr, L, st, leaf, ro, rlo, rhi);
        ul[i] = u32(l < first ? first : (l > last ? last : l));
    }
}

int Pma::try_group(int level, u64 seg, const u64* keys, const u64* vals, const u8* ops, u64 n, const EngineCfg& cfg,
                   u64* missed, u64* tombs) {
    if (level < 0 || level > height_) throw ApiError(PMA_ERANGE, "try_insert_plus: level out of range");
    const u64 m = leaf_ << level;
    if (seg >= cap_ / m) throw ApiError(PMA_ERANGE, "try_insert_plus: segment index out of range");
    uk.reserve(n + 4);
    uv.reserve(n + 4);
    uop.reserve(n + 32);
    ul.reserve(n + 1);
    gstart.reserve(2);
    gseg.reserve(2);
    gflag.reserve(1);
    touched.reserve(2 * n + 2);
    rlist.reserve(4);
    ik.reserve(n + 1);
    iv.reserve(n + 1);
    ir.reserve(n + 1);
    ensure_slot_scratch();
    if (n) {
        GPMA_CUDA(cudaMemcpyAsync(uk.ptr, keys, n * 8, cudaMemcpyHostToDevice, stream_));
        GPMA_CUDA(cudaMemcpyAsync(uv.ptr, vals, n * 8, cudaMemcpyHostToDevice, stream_));
        GPMA_CUDA(cudaMemcpyAsync(uop.ptr, ops, n, cudaMemcpyHostToDevice, stream_));
        const u64 first = seg * (m / leaf_), last = first + m / leaf_ - 1;
        k_group_leaves<<<grid_for(n, 256), 256, 0, stream_>>>(uk.ptr, n, d_hdr, num_leaves(), d_st, leaf_,
                                                              ro_base(), ro_lo, ro_lo + num_vertices, first, last,
                                                              ul.ptr);
        GPMA_LAUNCH_CHECK();
    }
    const u32 gs[2] = {0, u32(n)};
    const u32 gg[1] = {u32(seg)};
    GPMA_CUDA(cudaMemcpyAsync(gstart.ptr, gs, sizeof(gs), cudaMemcpyHostToDevice, stream_));
    GPMA_CUDA(cudaMemcpyAsync(gseg.ptr, gg, sizeof(gg), cudaMemcpyHostToDevice, stream_));
    GPMA_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(Ctr), stream_));
    const ull one = 1;
    GPMA_CUDA(cudaMemcpyAsync(&d_ctr->ngroups, &one, sizeof(ull), cudaMemcpyHostToDevice, stream_));
    CommitArgs a{};
    touched_cb_ = 1;
    while ((1ull << touched_cb_) <= cap_) ++touched_cb_;
    a.t0 = touched.ptr;  // (one group: g = 0)
    a.tlist = touched.ptr + 1;
    a.cb = touched_cb_;
    a.keys = d_keys;
    a.vals = d_vals;
    a.st = d_st;
    a.uk = uk.ptr;
    a.uv = uv.ptr;
    a.uop = uop.ptr;
    a.ul = ul.ptr;
    a.pidx = nullptr;
    a.gstart = gstart.ptr;
    a.gseg = gseg.ptr;
    a.gflag = gflag.ptr;
    a.ctr = d_ctr;
    a.hdr = d_hdr;
    a.ro = ro_base();
    a.rlist = rlist.ptr;
    a.biglist = nullptr;
    a.level = level;
    a.m = m;
    a.leaf = leaf_;
    a.mn = mn_[level];
    a.mx = mx_[level];
    a.eager = cfg.eager;
    a.large = cfg.large_for(m);
    a.cap_gt_min = cap_ > 16;
    a.ek = ek.ptr;
    a.ev = ev.ptr;
    a.es = es.ptr;
    a.mflag = mflag.ptr;
    a.ok = ok.ptr;
    a.ov = ov.ptr;
    a.ik = ik.ptr;
    a.iv = iv.ptr;
    a.ir = ir.ptr;
    k_commit_cta<<<1, kCtaThreads, 0, stream_>>>(a);
    GPMA_LAUNCH_CHECK();
    u8 flag = 0;
    GPMA_CUDA(cudaMemcpyAsync(&flag, gflag.ptr, 1, cudaMemcpyDeviceToHost, stream_));
    sync_ctr();
    valid_count = u64((long long)valid_count + h_ctr->valid_delta);
    tombstone_count = u64((long long)tombstone_count + h_ctr->tomb_delta);
    slot_writes += h_ctr->slot_writes;
    if (empty_leaves >= 0) empty_leaves += h_ctr->empty_delta;
    if (h_ctr->nrefresh > 0) {
        k_refresh_ranges<<<grid_for(h_ctr->nrefresh * 32, 256, 148 * 16), 256, 0, stream_>>>(
            rlist.ptr, nullptr, h_ctr->nrefresh, d_keys, d_st, cap_, leaf_, d_hdr, ro_base());
        GPMA_LAUNCH_CHECK();
    }
    if (empty_leaves != 0) {
        k_left_walk<<<1, 32, 0, stream_>>>(touched.ptr, 1, touched.ptr + 1, h_ctr->ntouched_next, touched_cb_, d_st,
                                          leaf_, d_hdr);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaStreamSynchronize(stream_));
    last_ntouched = 0;
    if (missed) *missed = h_ctr->missed;
    if (tombs) *tombs = h_ctr->tomb_added;
    return flag;  // 0 deferred, 1 tombstones committed, 2 merged
}

void Pma::binary_search_leaf(const u64* keys, size_t n, u64* leaves) {
    if (n == 0) return;
    const u64* dq = stage(stage_k, keys, n);
    stage_v.reserve(n);
    k_search<<<grid_for(n, 256), 256, 0, stream_>>>(dq, n, d_hdr, num_leaves(), d_keys, d_vals, d_st, leaf_, nullptr,
                                                     nullptr, stage_v.ptr);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaMemcpyAsync(leaves, stage_v.ptr, n * 8, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

void Pma::search(const u64* keys, size_t n, u64* values, u8* found) {
    if (n == 0) return;
    const u64* dq = stage(stage_k, keys, n);
    stage_v.reserve(n);
    stage_o.reserve(n);
    k_search<<<grid_for(n, 256), 256, 0, stream_>>>(dq, n, d_hdr, num_leaves(), d_keys, d_vals, d_st, leaf_,
                                                     stage_v.ptr, stage_o.ptr, nullptr);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaMemcpyAsync(values, stage_v.ptr, n * 8, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaMemcpyAsync(found, stage_o.ptr, n, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

void Pma::slot_hash(int level, u64* hashes) {
    if (level < 0 || level > height_) throw ApiError(PMA_ERANGE, "slot_hash: level out of range");
    int lg = 0;
    while ((u64(1) << lg) < (leaf_ << level)) ++lg;
    const u64 nh = cap_ >> lg;
    DevBuf<ull> out;
    out.reserve(nh);
    GPMA_CUDA(cudaMemsetAsync(out.ptr, 0, nh * sizeof(ull), stream_));
    // cap_ is a power of two >= 16: whole warps stay inside the array
    k_slot_hash<<<grid_for(cap_, 256, 148 * 8), 256, 0, stream_>>>(d_keys, d_vals, d_st, cap_, lg, out.ptr);
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaMemcpyAsync(hashes, out.ptr, nh * 8, cudaMemcpyDeviceToHost, stream_));
    GPMA_CUDA(cudaStreamSynchronize(stream_));
}

u64 Pma::count_valid_in(u64 b, u64 e) {
    if (e > cap_ || b > e) throw ApiError(PMA_ERANGE, "count_valid_in: range outside the slot array");
    GPMA_CUDA(cudaMemsetAsync(&d_ctr->nv, 0, sizeof(ull), stream_));
    if (e > b) {
        k_count_valid<<<grid_for(e - b, 256), 256, 0, stream_>>>(d_st, b, e, d_ctr);
        GPMA_LAUNCH_CHECK();
    }
    sync_ctr();
    return h_ctr->nv;
}

}  // namespace gpma
