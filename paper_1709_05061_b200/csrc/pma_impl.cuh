// pma_impl.cuh — device-resident Packed Memory Array and the GPMA+ batch
// pipeline (host orchestration of the sm_100a kernels in pma.cu).
//
// HBM layout (SoA, 17 B/slot):
//   keys   u64[C]   values u64[C]   states u8[C]     (Empty slot = all zero)
//   hdr    u64[C/leaf]  backward-filled leaf headers: first non-Empty key at
//                       or after the leaf's first slot, UINT64_MAX if none.
//                       upper_bound(hdr, key) - 1 == binary_search_leaf(key)
//                       (pma.hpp:234-245); maintained incrementally.
// Per-batch scratch is grow-only and sized by the batch; the slot-space
// merge scratch (E/O arrays) is allocated on first use of the CTA/grid tiers.
#pragma once

#include <chrono>
#include <string>
#include <vector>

#include "common.cuh"
#include "radix.cuh"

namespace gpma {

// Device-side per-batch counters (one D2H per round).
constexpr int kMaxLevels = 64;

struct Ctr {
    ull n_unique;
    ull npend;
    ull ngroups;
    ull npend_next;
    ull missed;
    ull tomb_added;
    ull slot_writes;
    ull merge_slots;
    ull committed;
    long long valid_delta;
    long long tomb_delta;
    ull ntouched_next;
    ull guard_deletes;
    ull bad_index;
    ull root_ins;
    ull moves;
    ull mask_or;
    ull nv;
    ull nmatched;
    ull nins;
    ull nsurv;
    ull k;
    ull nt;
    ull key0;
    ull nrefresh;
    long long empty_delta;
    ull nbig;
    ull max_slice;
    ull commit_bytes;
    ull bad_ins;    // graph front end: ~(first insert index with an id >= |V|), 0 = none
    ull oor;        // graph front end: a delete key outside the compressed key range
    ull gdel;       // graph front end: guard deletes (dropped, counted missed)
    ull bigrun;     // leaf-bucket front end: a bucket reached kRunMax updates
    ull nbig_buckets;  // leaf-bucket front end: buckets sorted by the CTA kernel
    ull nsort;      // graph-captured small batches: the batch size, written by the front end
    ull leaf_tiles; // k_commit_leaf's dynamic tile counter (level 0 runs once per batch)
    ull ngrid;      // grid tier: groups handed over by k_commit_cta at this level
    ull gt0, gt1;   // captured small batches: %globaltimer at the first kernel's entry / the last refresh CTA's exit
    ull refresh_done;  // captured small batches: refresh CTAs finished (the last returns the counters)
    // commit-kernel span of each level (%globaltimer, levels < 16): the
    // complement of the earliest CTA start (atomicMax of ~t) and the latest
    // CTA end — no event records between a level's kernels, so their
    // programmatic edges stay intact
    ull lvl_tmin[16];
    ull lvl_tmax[16];
    // stage starts of a host-loop batch (complements of %globaltimer, the
    // earliest CTA): front end, duplicate resolution, round 0 — no event
    // records between the front end's kernels, whose PDL edges stay intact
    ull t_front, t_dedup, t_rounds;
    ull seq;           // captured small batches: the replay's sequence number (from the descriptor)
    ull done_seq;      // ... written to the host copy LAST, after the counters (the host polls it)
    ull seg_tomb, seg_empty;  // grid tier: tombstones / empty leaves of the segment before its merge
    ull round_overlap;  // GPMA_CHECK_ROUNDS=1: groups of a round that overlap (k_check_rounds)
    // device-driven rounds: pending counts alternate between np[level & 1] and
    // np[(level + 1) & 1]; per-level stats are kept here and read at the next
    // host sync (rounds may run back to back without one)
    ull np[2];
    ull ntouched_base;
    ull lvl_merge[kMaxLevels];  // cumulative merged slots after each level (level-0 touched count)
    ull lvl_npend[kMaxLevels];
    ull lvl_committed[kMaxLevels];
    ull lvl_groups[kMaxLevels];
    ull lvl_big[kMaxLevels];
    ull lvl_maxslice[kMaxLevels];
    ull lvl_bytes[kMaxLevels];  // commit_bytes after each level (cumulative)
    ull pad[4];
};

struct EngineCfg {
    bool eager = false;
    u64 small_max = 32;
    u64 medium_max = 1024;
    int force = PMA_STRATEGY_AUTO;
    bool large_for(u64 m) const {
        if (force >= 0) return force == PMA_STRATEGY_LARGE;
        return m > medium_max && m > small_max;
    }
};

struct SeqArgs;

// Graph-mode batch front end (DynamicGraph::apply_batch, graph.hpp:130-162):
// raw insert / delete arrays, packed on the device by the same kernel that
// builds the sort input, with |V| fixing the compressed key layout (no key
// reduction + host round trip).  Packed (key, value, op) land in bk/bv/bo.
struct GraphFront {
    const u32* is;
    const u32* id;
    const double* iw;
    u64 ni;
    const u32* ds;
    const u32* dd;
    u64 nd;
    u64 nv;
    u64 lo, hi;  // owned source range (a shard; [0, nv) for a whole graph)
    const u64* mk = nullptr;  // routed EdgeKeys (bit 63 = delete), ni of them, instead of the arrays
    u64* bk;
    u64* bv;
    u8* bo;
    // unweighted batch whose key + arrival index overflow one word: the packed
    // word carries just the op (key << 1 | is_delete) — the stable sort keeps
    // arrival order, and no weight is gathered by index
    int opbit = 0;
    // results
    u64 guard_deletes = 0;
    long long bad_insert = -1;  // first insert index with an id >= nv
    u64 seq = 0;                // captured small batches: the replay's sequence number (echoed back when done)
};

class Pma {
public:
    explicit Pma(const pma_profile* profile, int device);
    ~Pma();

    // --- geometry (PmaLayout, pma.hpp:82-123; bounds pma.hpp:577-588) ---
    static u64 leaf_size_for(u64 cap);
    static int height_for(u64 cap, u64 leaf);
    u64 capacity() const { return cap_; }
    u64 leaf() const { return leaf_; }
    int height() const { return height_; }
    u64 num_leaves() const { return cap_ / leaf_; }
    u64 min_entries(int l) const { return mn_[l]; }
    u64 max_entries(int l) const { return mx_[l]; }
    u64 max_at_capacity(u64 cap) const;
    const pma_profile& profile() const { return prof_; }

    // --- API ---
    void from_sorted_device(const u64* d_keys, const u64* d_vals, u64 n, double fill_target);
    void load_slots(size_t capacity, const u64* keys, const u64* values, const u8* states);
    void download(u64* keys, u64* values, u8* states);
    void batch_update_device(const u64* d_keys, const u64* d_vals, const u8* d_ops, u64 n, const EngineCfg& cfg,
                             pma_stats* out, GraphFront* gf = nullptr);
    void binary_search_leaf(const u64* keys, size_t n, u64* leaves);
    void search(const u64* keys, size_t n, u64* values, u8* found);
    u64 count_valid_in(u64 b, u64 e);
    void slot_hash(int level, u64* hashes);
    void reserve_batch(u64 n);
    // grid tier: segments of at least grid_seg_ slots are merged device-wide
    u64 grid_seg_ = u64(1) << 16;
    void grid_merge(u64 b, u64 m, const u32* plist, u64 s, bool large);
    // small graph batches (pma.cu): captured front end + first rounds
    static constexpr u64 kSmallGraphMax = 16384;
    static constexpr int kSmallIb = 15;  // index bits of the packed sort word ((1 << 15) - 1 > 16384: delete marker)
    static constexpr int kSmallGraphLevels = 1;  // most small batches finish in round 0; more rounds: host loop
    bool small_graph_ok(u64 n, const GraphFront& gf) const;
    std::vector<uintptr_t> small_graph_key(int db, const EngineCfg& cfg, int levels) const;
    void capture_small_graph(int db, const EngineCfg& cfg, int levels, int multi);
    int run_small_graph(const GraphFront& gf, const EngineCfg& cfg);
    void enqueue_level(int level, u64 npend, u32* pcur, u32* pnext, u64* touched_ptr, u64 n, const EngineCfg& cfg,
                       ScanWorkspace& ws, bool events, u64& launches);
    int try_group(int level, u64 seg, const u64* keys, const u64* vals, const u8* ops, u64 n, const EngineCfg& cfg,
                  u64* missed, u64* tombs);
    void touched_ranges(u64* pairs, size_t cap, size_t* count);

    // sequential single-key ops (pma.hpp:294-386, 471-479)
    void insert(u64 key, u64 value);
    bool erase(u64 key);
    bool mark_tombstone(u64 key);
    void redispatch(int level, u64 seg, const u64* keys, const u64* values, size_t n);

    // row-offset maintenance hook used by the graph (graph.hpp:167-190):
    // when non-null, every refresh also rewrites ro[src+1] for guards.
    u64* d_row_offsets = nullptr;  // rows [ro_lo, ro_lo + num_vertices) of a graph (shard)
    u64 num_vertices = 0;
    u64 ro_lo = 0;
    // row-offset array indexed by GLOBAL source id (ro_base()[src + 1]): a
    // shard's array starts at its first owned vertex
    u64* ro_base() const { return d_row_offsets ? d_row_offsets - ro_lo : nullptr; }
    void rebuild_row_offsets_full();
    SeqArgs seq_args(int op);

    // staging for host-facing APIs
    template <typename T>
    T* stage(DevBuf<T>& buf, const T* host, size_t n) {
        buf.reserve(n ? n : 1);
        if (n) GPMA_CUDA(cudaMemcpyAsync(buf.ptr, host, n * sizeof(T), cudaMemcpyHostToDevice, stream_));
        return buf.ptr;
    }

    // a page-locked host array the device can read in place (UVA: the device
    // pointer of a cudaHostAlloc / cudaHostRegister block), else a staged copy
    template <class T>
    const T* stage_or_map(DevBuf<T>& buf, const T* host, size_t n) {
        if (!n) return stage(buf, host, n);
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer != nullptr)
            return static_cast<const T*>(at.devicePointer);
        cudaGetLastError();  // pageable memory: not an error worth keeping
        return stage(buf, host, n);
    }

    cudaStream_t stream() const { return stream_; }
    // run every call on a caller-provided stream (own: back to the handle's own;
    // a null caller stream is the legacy default stream)
    void set_stream(cudaStream_t s, bool own) { stream_ = own ? own_stream_ : s; }
    int device() const { return device_; }
    std::string err;
    pma_timing timing{};
    // A host-loop batch returns once its counters are on the host; its tail
    // (header / row-offset refresh) may still be running on the stream, so
    // the event-based stage times are resolved later (resolve_set): when its
    // event set comes round again, or when the timing is read (timing_now()).
    // Stage events alternate between two sets per batch, so a batch's set is
    // only re-recorded two batches later (its tail long finished): resolving
    // a deferred record never waits inside the next batch.
    int ev_set_ = 0;
    bool pend_[2] = {false, false};
    bool latest_pending_ = false;  // `timing` (the last batch's record) still lacks its stage times
    pma_timing pend_t_[2]{};
    cudaEvent_t E(int idx) const { return ev_[ev_set_ * 6 + idx]; }
    void resolve_set(int set);
    void resolve_all() {
        for (int k = 0; k < 2; ++k)
            if (pend_[k]) resolve_set(k);
    }
    // sum of the batches' records since the last reset (gpma_timing_sum)
    pma_timing tsum_{};
    u64 tsum_n_ = 0;
    void accumulate_timing(const pma_timing& t);
    const pma_timing& timing_now() {
        resolve_all();
        return timing;
    }

    u64 valid_count = 0;
    u64 tombstone_count = 0;
    u64 slot_writes = 0;
    bool last_resized = false;
    // number of all-Empty leaves (-1 = unknown after sequential ops): the
    // left-walk header pass only runs when empty leaves can exist
    long long empty_leaves = 0;
    u64 last_ntouched = 0;

    // device slot arrays
    u64* d_keys = nullptr;
    u64* d_vals = nullptr;
    u8* d_st = nullptr;
    u64* d_hdr = nullptr;

    // staging buffers for host APIs
    DevBuf<u64> stage_k, stage_v;
    DevBuf<u8> stage_o;
    DevBuf<u32> stage_a, stage_b, stage_c, stage_d;
    DevBuf<double> stage_w;

    ScanWorkspace ws;

public:  // (extended __device__ lambdas need public enclosing functions)
    void reset_layout(u64 cap);  // allocate zeroed arrays, bounds
    void free_arrays();
    void rebuild_at_capacity(u64 cap);
    void place_root_from(const u64* d_ek, const u64* d_ev, u64 k);  // even placement at root + headers
    void headers_closed_form(const u64* d_ek, u64 k);
    void refresh_after_batch();
    void root_path(const EngineCfg& cfg, pma_stats& st, u64 level_committed_base);
    void ensure_slot_scratch();
    void sync_ctr();
    void event(int idx);

    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t own_stream_ = nullptr;  // created with the handle; stream_ may be a caller's stream
    pma_profile prof_{};
    u64 cap_ = 0, leaf_ = 4;
    int height_ = 0;
    u64 mn_[PMA_MAX_LEVELS]{}, mx_[PMA_MAX_LEVELS]{};

    // counters
    Ctr* d_ctr = nullptr;
    Ctr* h_ctr = nullptr;  // pinned

    // batch scratch
    DevBuf<u64> sk_in, sk_out;   // compressed keys
    DevBuf<u32> si_in, si_out;   // arrival index payload
    RadixWorkspace rws;           // onesweep radix sort (radix.cuh)
    // small graph batches
    bool small_graphs_ = true;          // GPMA_NO_GRAPHS=1 disables (A/B measurements)
    cudaGraphExec_t small_exec_[3] = {nullptr, nullptr, nullptr};  // front end: one CTA, multi-CTA, multi-CTA > 4096
    std::vector<uintptr_t> small_key_[3];  // what each captured graph embeds
    u64 small_onecta_ = 512;            // larger small batches: the multi-CTA front end (GPMA_SMALL_ONECTA=n)
    DevBuf<u64> small_sb_;              // its scratch (k_small_front_grid)
    bool check_rounds_ = false;         // GPMA_CHECK_ROUNDS=1: the round-disjointness check after every grouping
    bool small_cluster_ = true;         // ... in one 16-CTA cluster (GPMA_SMALL_CLUSTER=0: a cooperative grid)
    GraphFront* h_desc_ = nullptr;      // page-locked batch descriptor (copied by the graph's first node)
    GraphFront* d_desc_ = nullptr;
    GraphFront* h_desc_dev_ = nullptr;  // device view of h_desc_ (read in place by the small graph)
    Ctr* h_ctr_dev_ = nullptr;          // device view of h_ctr (written by the small graph's last node)
    bool pdl_ = true;                   // small graph: programmatic edges between its kernels
    bool small_poll_ = true;            // small graph: the host polls done_seq instead of synchronising the stream
    bool direct_touched_ = true;        // touched ranges written in place into a page-locked caller array
    bool level_events_ = false;         // GPMA_LEVEL_EVENTS=1: level spans from CUDA events (cross-check of the stamps)
    cudaEvent_t lev_ev_[32]{};          // (only with level_events_: before / after the commit kernels of levels < 16)
    u64 small_seq_ = 0;
    ScanWorkspace small_ws_;            // the graph's own look-back words (cleared by every replay)
    // leaf-bucket front end (graph batches): per-leaf counters / offsets, per
    // update bucket + ordinal, per sorted position bucket
    DevBuf<u32> bcnt, boff, blf, bod, bslf, bbig;
    u64 bcnt_zero_ = 0;  // bcnt[0, bcnt_zero_) is known zero (the bucket scan clears what it reads)
    int bucket_skip_ = 0;  // batches left on the radix sort after a bucket overflow
    bool buckets_ = true;  // GPMA_NO_BUCKETS=1: always the radix front end (A/B measurements)
    static constexpr u64 kBucketMinBatch = 1u << 16;
    static constexpr u64 kBucketMaxLeaves = 8ull << 20;  // 64 MB of leaf headers
    static constexpr int kBucketCooldown = 16;
    DevBuf<u64> uk, uv;
    DevBuf<u8> uop;
    DevBuf<u32> ul;
    DevBuf<u32> pidx0, pidx1, gid, gstart, gseg;
    DevBuf<u64> rlist;  // ranges whose headers/row offsets need the post-pass
    DevBuf<u32> biglist;  // leaf groups with > kBigSlice updates (lane-parallel kernel)
    DevBuf<u8> gflag;
    DevBuf<u64> touched;  // pairs (b, e)
    DevBuf<u64> tw0, tw1;  // touched ranges as sortable words (touched_ranges)
    // touched words of the last batch: level 0 dense by group index in
    // touched[0, last_ngroups0_), higher levels + the root appended at
    // touched[touched_split_ ...] (last_nrest_ of them)
    int touched_cb_ = 32;
    u64 touched_split_ = 0, last_ngroups0_ = 0, last_nrest_ = 0;
    DevBuf<u64> ik, iv;   // insert lists (pending space)
    DevBuf<u32> ir;
    // slot-space merge scratch (CTA/grid tiers, root path)
    DevBuf<u64> ek, ev, ok, ov;
    DevBuf<u32> es, mb;
    DevBuf<u8> mflag;

    cudaEvent_t ev_[12]{};  // two sets of six stage events, alternating per batch (ev_set_)
};

}  // namespace gpma
