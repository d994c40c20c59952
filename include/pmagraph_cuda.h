/*
 * pmagraph_cuda.h — C ABI of libpmagraph_cuda.so, the B200-native GPMA+ store.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or CUDA
 * types.  Every entry point replaces one public entry of the reference's
 * header-only C++ API (/root/reference/proj/include/pmagraph/...); the file:line
 * of the reference interface it replaces is cited beside each declaration.
 * The C++ wrappers in include/pmagraph/*.hpp restore the reference class and
 * function names on top of these calls, and INTEGRATION.md shows the ctypes
 * and C++ bindings a maintainer adds.
 *
 * Conventions
 *  - Every function returns int: PMA_OK (0) or an error code.  The codes map
 *    onto the exception types the reference throws:
 *      PMA_EINVAL -> std::invalid_argument, PMA_ERANGE -> std::out_of_range,
 *      PMA_ELOGIC -> std::logic_error,      PMA_ECUDA  -> std::runtime_error.
 *    pma_last_error(h)/gpma_last_error(g) return the message of the last
 *    failure on that handle (thread-unsafe, like the reference's single-writer
 *    contract, pma.hpp:9-12).
 *  - Host pointers are borrowed for the call only.  "_device" variants take
 *    device pointers that stay owned by the caller.
 *  - Calls are synchronous: they return after the handle's stream drained, so
 *    wall times measured around them are end-to-end.
 *  - Absent deletes are counted (pma_stats.deletes_missed), never errors,
 *    exactly as segment_engine.hpp:134,294-307 and graph.hpp:140-145.
 *  - Slot states: 0 = Empty, 1 = Valid, 2 = Tombstone (pma.hpp:29).  An Empty
 *    slot downloads as key = value = 0 (pma.hpp:31-33).
 *  - Update ops: 0 = insert, 1 = delete (segment_engine.hpp:24).
 */
#ifndef PMAGRAPH_CUDA_H
#define PMAGRAPH_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMA_OK 0
#define PMA_EINVAL 1
#define PMA_ERANGE 2
#define PMA_ELOGIC 3
#define PMA_ECUDA 4

#define PMA_MAX_LEVELS 64

/* DensityProfile (pma.hpp:52-78).  NULL anywhere a profile is accepted means
 * the reference defaults {0.08, 0.92, 0.40, 0.80, allow_shrink = 1}. */
typedef struct pma_profile {
    double leaf_lower;
    double leaf_upper;
    double root_lower;
    double root_upper;
    int32_t allow_shrink;
    int32_t _pad;
} pma_profile;

/* DeletionMode (segment_engine.hpp:35) */
#define PMA_LAZY 0
#define PMA_EAGER 1
/* MergeStrategy (segment_engine.hpp:41); -1 = size-tiered dispatch */
#define PMA_STRATEGY_AUTO (-1)
#define PMA_STRATEGY_SMALL 0
#define PMA_STRATEGY_MEDIUM 1
#define PMA_STRATEGY_LARGE 2

/* SegmentEngineConfig + MergeTiers (segment_engine.hpp:43-60).  `workers` is
 * accepted for drop-in compatibility and ignored: the CUDA grid replaces the
 * WorkerPool, and results are worker-count independent by contract
 * (pma.hpp:9-12).  The merge tier only changes the slot_writes accounting
 * (commit_in_place counts compaction moves, segment_engine.hpp:147-230); the
 * slot arrays are identical for every tier (segment_engine.hpp:37-40). */
typedef struct pma_engine_config {
    int32_t deletion_mode;   /* PMA_LAZY | PMA_EAGER */
    uint32_t workers;        /* ignored */
    uint64_t small_max;      /* MergeTiers::small_max  (default 32)   */
    uint64_t medium_max;     /* MergeTiers::medium_max (default 1024) */
    int32_t force_strategy;  /* PMA_STRATEGY_* */
    int32_t _pad;
} pma_engine_config;

/* UpdateStats (update_stats.hpp:13-35) as a fixed POD.  touched_ranges are
 * fetched separately with pma_touched_ranges().  Timing fields are host
 * steady-clock nanoseconds around the device work (wall_ns) and the summed
 * device time of the per-round segment kernels (segment_phase_ns). */
typedef struct pma_stats {
    uint64_t batch_size;
    uint64_t rounds;
    uint64_t slot_writes;
    uint64_t wall_ns;
    uint64_t segment_phase_ns;
    uint64_t grow_events;
    uint64_t shrink_events;
    uint64_t deletes_missed;
    uint64_t tombstones_added;
    uint64_t num_touched_ranges;
    int32_t resized;
    int32_t num_levels; /* segments_per_level.size() */
    uint64_t segments_per_level[PMA_MAX_LEVELS];
} pma_stats;

/* PmaLayout + counters (pma.hpp:82-123, 209-214, 529). */
typedef struct pma_layout_info {
    uint64_t capacity;
    uint64_t leaf_size;
    int32_t height;
    int32_t _pad;
    uint64_t valid_count;
    uint64_t tombstone_count;
    uint64_t slot_writes;
} pma_layout_info;

/* Device-event timings of the most recent call on a handle (milliseconds),
 * for the bench's roofline: the dominant kernel's summed duration and launch
 * count, plus the whole device-side span. */
typedef struct pma_timing {
    double device_ms;      /* first to last event of the call on the stream */
    double sort_ms;        /* key sort + duplicate resolution             */
    double search_ms;      /* leaf assignment                             */
    double rounds_ms;      /* all per-round kernels (decide/commit/scatter) */
    double refresh_ms;     /* leaf-header + row-offset refresh            */
    uint64_t kernel_launches;
    uint64_t merge_slots;  /* slots rewritten by merge commits (algorithmic scatter) */
    uint64_t tombstone_flips;
    double level_ms[16];   /* commit-kernel time per tree level (rounds) */
    uint64_t level_groups[16]; /* groups examined per level */
    uint64_t level_big[16];    /* hub groups sent to the CTA kernel per level */
    uint64_t level_max_slice[16]; /* largest update slice per level */
    uint64_t commit_bytes; /* algorithmic HBM bytes of the commit kernels */
    uint64_t level_bytes[16]; /* the same, per tree level */
    uint64_t front_end;    /* 0 radix sort, 1 leaf buckets, 2 leaf buckets overflowed -> radix sort redo */
    uint64_t grid_merges;  /* segments merged by the grid tier (pma_set_grid_segment) */
} pma_timing;

typedef struct pma_handle pma_handle;

/* ---- PackedMemoryArray (pma.hpp:125-612) ------------------------------- */

/* PackedMemoryArray(DensityProfile) (pma.hpp:129-132): empty array of
 * kMinCapacity = 16 slots on CUDA device `device`. */
int pma_create(const pma_profile* profile, int device, pma_handle** out);
int pma_destroy(pma_handle* h);
const char* pma_last_error(const pma_handle* h);

/* PackedMemoryArray::from_sorted (pma.hpp:160-187).  keys strictly
 * increasing, else PMA_EINVAL with the reference's message. */
int pma_from_sorted(pma_handle* h, const uint64_t* keys, const uint64_t* values, size_t n,
                    double fill_target);

/* Exact state restore (generalises from_slot_layout, pma.hpp:191-207, to
 * tombstones): capacity must be a power of two >= 16.  Counters are derived
 * from the states; slot_writes is reset to 0. */
int pma_load_slots(pma_handle* h, size_t capacity, const uint64_t* keys, const uint64_t* values,
                   const uint8_t* states);

/* slots() (pma.hpp:214) as SoA: capacity entries each; any pointer may be NULL. */
int pma_download(pma_handle* h, uint64_t* keys, uint64_t* values, uint8_t* states);

/* layout(), capacity(), valid_count(), tombstone_count(), slot_writes()
 * (pma.hpp:209-214, 529). */
int pma_get_layout(const pma_handle* h, pma_layout_info* out);
int pma_reset_slot_writes(pma_handle* h); /* pma.hpp:530 */

/* min_entries/max_entries/thresholds (pma.hpp:217-230); PMA_ERANGE outside
 * [0, height] with the reference's message (pma.hpp:533-538). */
int pma_bounds(const pma_handle* h, int level, uint64_t* min_entries, uint64_t* max_entries,
               double* rho, double* tau);

/* batch_update(PackedMemoryArray&, std::vector<Update>, const
 * SegmentEngineConfig&, WorkerPool*) -> UpdateStats (segment_engine.hpp:365-470).
 * Host arrays of n updates; cfg NULL = defaults. */
int pma_batch_update(pma_handle* h, const uint64_t* keys, const uint64_t* values,
                     const uint8_t* ops, size_t n, const pma_engine_config* cfg, pma_stats* out);
/* Same, with the update arrays already resident in device memory. */
int pma_batch_update_device(pma_handle* h, const uint64_t* d_keys, const uint64_t* d_values,
                            const uint8_t* d_ops, size_t n, const pma_engine_config* cfg,
                            pma_stats* out);

/* UpdateStats::touched_ranges of the last batch: pairs (begin, end) into
 * `pairs` (2*cap entries); *count receives the total number of ranges. */
int pma_touched_ranges(pma_handle* h, uint64_t* pairs, size_t cap, size_t* count);

/* Size every per-batch buffer for batches of up to max_updates updates (and
 * the slot-space scratch of the CTA/grid tiers) now, so that no device
 * allocation lands inside a later batch_update / apply_batch (the
 * std::vector::reserve of the batch pipeline; no reference counterpart,
 * state unchanged).  Buffers only grow. */
int pma_reserve_batch(pma_handle* h, size_t max_updates);

/* Segments of at least min_slots slots (default 65536) are merged by the
 * grid tier — device-wide compaction, ranking, scatter and placement over the
 * segment (commit_in_place's range, segment_engine.hpp:147-230) — instead of
 * one CTA per segment; smaller ones by the warp / CTA tiers.  The slot arrays
 * and UpdateStats are identical either way (a tuning knob, >= 64). */
int pma_set_grid_segment(pma_handle* h, uint64_t min_slots);

/* try_insert_plus(pma, level, seg, slice, cfg, result) (segment_engine.hpp:
 * 320-341) for one group on the device: the n updates (sorted by key,
 * duplicates resolved, all inside segment `seg` of `level`) are decided by the
 * same rules as the batch engine's rounds and, when allowed, committed (lazy
 * tombstones, or a merge + even re-dispatch).  *outcome: 0 deferred (nothing
 * changed), 1 tombstones committed, 2 merged.  PMA_ERANGE for a level or
 * segment outside the layout. */
int pma_try_insert_plus(pma_handle* h, int level, size_t seg, const uint64_t* keys, const uint64_t* values,
                        const uint8_t* ops, size_t n, const pma_engine_config* cfg, int* outcome,
                        uint64_t* deletes_missed, uint64_t* tombstones_added);

/* Parity digest of slots() (pma.hpp:214) without downloading it: one u64 per
 * segment of `level` (capacity / (leaf_size << level) values), the wrapping
 * sum over the segment's slots i of mix(key + mix(value ^ (i * 0x9E3779B97F4A7C15
 * + state))), mix = the splitmix64 finaliser.  Pins keys, values, states and
 * gap positions; tests/golden/hashing.py computes the same from a host copy.
 * PMA_ERANGE when level > height. */
int pma_slot_hash(pma_handle* h, int level, uint64_t* hashes);

/* binary_search_leaf for n keys (pma.hpp:234-245); any order. */
int pma_binary_search_leaf(pma_handle* h, const uint64_t* keys, size_t n, uint64_t* leaves);

/* search(key) (pma.hpp:247-251) for n keys: found[i] = 1 and values[i] set
 * when the key is Valid. */
int pma_search(pma_handle* h, const uint64_t* keys, size_t n, uint64_t* values, uint8_t* found);

/* count_valid_in(begin, end) (pma.hpp:425-429). */
int pma_count_valid_in(pma_handle* h, size_t begin, size_t end, uint64_t* count);

/* Sequential single-key operations (pma.hpp:294-360, 365-386, 471-479).
 * Their semantics differ from a one-update batch (in-place overwrite and
 * tombstone revival; retry from the leaf after a grow) and are reproduced
 * exactly.  Executed by device kernels; no CPU fallback. */
int pma_insert(pma_handle* h, uint64_t key, uint64_t value);
int pma_erase(pma_handle* h, uint64_t key, int* erased);
int pma_mark_tombstone(pma_handle* h, uint64_t key, int* marked);
int pma_redispatch(pma_handle* h, int level, size_t seg_index, const uint64_t* keys,
                   const uint64_t* values, size_t n);

int pma_last_timing(const pma_handle* h, pma_timing* out);

/* ---- DynamicGraph (graph.hpp:62-240) ------------------------------------ */

/* GraphConfig (graph.hpp:54-60).  engine must be the segment engine (0); the
 * lock engine (GPMA, lock_engine.hpp) is out of scope. */
typedef struct gpma_graph_config {
    int32_t engine;         /* 0 = UpdateEngine::kSegment */
    int32_t deletion_mode;  /* PMA_LAZY | PMA_EAGER */
    uint32_t workers;       /* ignored */
    int32_t _pad;
    double fill_target;     /* 0.5 */
    pma_profile profile;
} gpma_graph_config;

typedef struct gpma_graph gpma_graph;

/* DynamicGraph::from_edges (graph.hpp:66-92).  weights may be NULL (1.0). */
int gpma_from_edges(const gpma_graph_config* cfg, int device, size_t num_vertices,
                    const uint32_t* src, const uint32_t* dst, const double* weights, size_t n,
                    gpma_graph** out);
/* Same with device-resident edge arrays. */
int gpma_from_edges_device(const gpma_graph_config* cfg, int device, size_t num_vertices,
                           const uint32_t* d_src, const uint32_t* d_dst, const double* d_weights,
                           size_t n, gpma_graph** out);
int gpma_destroy(gpma_graph* g);
const char* gpma_last_error(const gpma_graph* g);

/* The graph's PackedMemoryArray (graph.hpp:96); owned by the graph. */
pma_handle* gpma_pma(gpma_graph* g);
uint64_t gpma_num_vertices(const gpma_graph* g);
uint64_t gpma_num_edges(const gpma_graph* g); /* graph.hpp:95 */

/* DynamicGraph::apply_batch (graph.hpp:130-162): inserts (src,dst,weight),
 * deletes (src,dst); guard deletes are dropped and counted as missed; row
 * offsets refreshed on the device.  weights may be NULL (1.0). */
int gpma_apply_batch(gpma_graph* g, const uint32_t* ins_src, const uint32_t* ins_dst,
                     const double* ins_w, size_t n_ins, const uint32_t* del_src,
                     const uint32_t* del_dst, size_t n_del, pma_stats* out);
int gpma_apply_batch_device(gpma_graph* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                            const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                            const uint32_t* d_del_dst, size_t n_del, pma_stats* out);

/* pma_reserve_batch for the graph: every per-batch buffer of apply_batch
 * for batches of up to max_updates inserts + deletes, so no allocation lands
 * inside a later call (no reference counterpart; state unchanged). */
int gpma_reserve_batch(gpma_graph* g, size_t max_updates);

/* row_offsets() (graph.hpp:97): num_vertices + 1 entries. */
int gpma_row_offsets(gpma_graph* g, uint64_t* out);
/* rebuild_row_offsets() (graph.hpp:182-190). */
int gpma_rebuild_row_offsets(gpma_graph* g);
/* csr_snapshot() (graph.hpp:192-206): row_offsets (|V|+1), col (num_edges),
 * vals (num_edges). */
int gpma_csr_snapshot(gpma_graph* g, uint64_t* row_offsets, uint32_t* col, double* vals);

/* ---- analytics (analytics.hpp:17-158) ----------------------------------- */

#define GPMA_UNREACHED 0xFFFFFFFFu /* kUnreached, analytics.hpp:17 */

/* bfs(g, root) (analytics.hpp:22-48): dist has num_vertices entries;
 * PMA_EINVAL when root >= num_vertices. *reached (may be NULL) = vertices
 * with a finite distance. */
int gpma_bfs(gpma_graph* g, uint32_t root, uint32_t* dist, uint64_t* reached);
/* connected_components(g) (analytics.hpp:53-82): min-id label per component
 * of the undirected closure. */
int gpma_cc(gpma_graph* g, uint32_t* labels);
/* pagerank(g, PageRankOptions) (analytics.hpp:90-143).  warm may be NULL. */
int gpma_pagerank(gpma_graph* g, double damping, double epsilon, size_t max_iters,
                  const double* warm, double* ranks, uint64_t* iterations, int* converged);
/* spmv(g, x) (analytics.hpp:147-158); summation in ascending destination
 * order per row, no FMA contraction: bit-exact with the reference. */
int gpma_spmv(gpma_graph* g, const double* x, double* y);

int gpma_last_timing(const gpma_graph* g, pma_timing* out);
/* Sum of the pma_timing records of every update batch since the last reset
 * (level_max_slice: the maximum), and how many batches it covers; reset != 0
 * starts a new sum after copying.  Lets a driver time a loop of batches
 * without reading each batch's record (which waits for a batch's deferred
 * refresh tail). */
int gpma_timing_sum(gpma_graph* g, pma_timing* out, uint64_t* batches, int reset);

/* The cudaStream_t (as void*) every call on this handle runs on, so callers
 * can bracket calls with CUDA events on the launching stream. */
void* gpma_cuda_stream(gpma_graph* g);
void* pma_cuda_stream(pma_handle* h);

/* ---- key-range sharding across GPUs ------------------------
 * One GPMA+ per GPU over the source range [lo, hi) (keys are src << 32 | dst,
 * so a source range is a key range; segments never cross shards).  The
 * reference has no multi-GPU interface: these entry points are the device
 * side of the paper's partitioned deployment; the
 * collectives (NCCL all-to-all / all-reduce) run in the caller between these
 * synchronous calls, on device pointers.  Vertex ids stay global. */

/* DynamicGraph::from_edges (graph.hpp:66-92) restricted to the sources
 * [lo, hi): edges with other sources are skipped (so every shard may be fed
 * the same global edge list), guards only for [lo, hi), row offsets over
 * [lo, hi] (gpma_row_offsets returns hi - lo + 1 entries).  apply_batch on a
 * shard rejects inserts whose source lies outside [lo, hi). */
int gpma_shard_from_edges_device(const gpma_graph_config* cfg, int device, size_t num_vertices, uint32_t lo,
                                 uint32_t hi, const uint32_t* d_src, const uint32_t* d_dst, const double* d_weights,
                                 size_t n, gpma_graph** out);
int gpma_shard_range(const gpma_graph* g, uint64_t* lo, uint64_t* hi);

/* Routing: one rank's share of a batch (inserts then deletes, device
 * arrays) stably partitioned by owner rank (d_bounds[r] <= src <
 * d_bounds[r+1], world + 1 entries, world <= 64; ids >= |V| go to the last
 * rank) into EdgeKeys d_out_keys (owner-major, arrival order kept inside each
 * owner; bit 63 set on deletes, so |V| <= 2^31), with the insert weights in
 * d_out_w (NULL: none; deletes get 1.0); counts[r] (host, world + 1 entries)
 * = updates for rank r, and counts[world] = inserts naming a vertex >= |V|:
 * when any sender reports one, every rank must reject the batch before any
 * shard applies (check_ids throws invalid_argument before any mutation,
 * graph.hpp:133-137).  A delete naming a vertex >= |V| travels as a key no
 * graph holds, so it is counted missed (graph.hpp:140-145) and never aliases
 * a real edge through the delete bit.  One all-to-all of these words
 * (8 B / update) is the whole exchange. */
int gpma_route_batch(gpma_graph* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst, const double* d_ins_w,
                     size_t n_ins, const uint32_t* d_del_src, const uint32_t* d_del_dst, size_t n_del,
                     const uint32_t* d_bounds, int world, uint64_t* d_out_keys, double* d_out_w, uint64_t* counts);

/* As gpma_route_batch, but the per-rank counts go to device memory d_counts
 * (world + 1 u64, as above) and nothing is synchronised: with gpma_set_stream on the
 * caller's stream, routing, the NCCL exchange and the apply are
 * stream-ordered without host round trips. */
int gpma_route_batch_async(gpma_graph* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst, const double* d_ins_w,
                           size_t n_ins, const uint32_t* d_del_src, const uint32_t* d_del_dst, size_t n_del,
                           const uint32_t* d_bounds, int world, uint64_t* d_out_keys, double* d_out_w,
                           uint64_t* d_counts);

/* Run every later call on this handle on `stream` (a cudaStream_t; NULL is
 * the legacy default stream), or back on the handle's own stream when `own`
 * is non-zero.  Calls stay host-synchronous where they return host results. */
int gpma_set_stream(gpma_graph* g, void* stream, int own);

/* DynamicGraph::apply_batch (graph.hpp:130-162) on a routed batch: n
 * EdgeKeys with bit 63 = delete (inserts keep their arrival order among
 * themselves, which is all "last insert wins" needs), weights d_w (NULL =
 * 1.0) parallel to the keys. */
int gpma_apply_batch_routed_device(gpma_graph* g, const uint64_t* d_keys, const double* d_w, size_t n,
                                   pma_stats* stats);

/* BFS (analytics.hpp:22-48), one level: mark (flags[v] = 1, |V| bytes,
 * zeroed by the call) the out-neighbours of the owned frontier vertices; the
 * caller max-reduces the flags across shards, then the owners admit their
 * unreached flagged vertices at `depth` (dist_local: hi - lo entries) as the
 * next frontier (global ids, count to *nf). */
int gpma_shard_bfs_mark(gpma_graph* g, const uint32_t* d_frontier, uint32_t nf, uint8_t* d_flags);
int gpma_shard_bfs_update(gpma_graph* g, const uint8_t* d_flags, uint32_t* d_dist_local, uint32_t depth,
                          uint32_t* d_next, uint32_t* nf);

/* Connected components (analytics.hpp:53-82) as min-label propagation over
 * replicated labels (|V| entries): hook the owned edges (atomic min), the
 * caller min-reduces the labels across shards, then pointer jumping makes
 * every label its root; *changed = any label differs from d_prev.  The
 * fixpoint labels are the component minima — the reference's labels. */
int gpma_shard_cc_hook(gpma_graph* g, uint32_t* d_labels);
int gpma_cc_jump(gpma_graph* g, uint32_t* d_labels, size_t n, const uint32_t* d_prev, int* changed);

/* PageRank (analytics.hpp:84-143): out-degrees of the owned rows (|V|
 * entries, zeroed by the call; the caller sum-reduces them once); per
 * iteration the owners push d*x[u]/outdeg[u] into d_y (zeroed by the call),
 * the caller sum-reduces d_y, then gpma_pr_finish adds the base term
 * ((1-d)/n + d*dangling/n) and returns the L1 residual (replicated). */
int gpma_shard_outdeg(gpma_graph* g, uint32_t* d_outdeg);
int gpma_shard_pr_push(gpma_graph* g, const double* d_x, const uint32_t* d_outdeg, double damping, double* d_y);
int gpma_pr_finish(gpma_graph* g, const double* d_x, double* d_y, size_t n, const uint32_t* d_outdeg, double damping,
                   double* l1);

/* SpMV (analytics.hpp:147-158) of the owned rows: d_y_local[u - lo] for u in
 * [lo, hi), same ordered accumulation as gpma_spmv. */
int gpma_shard_spmv(gpma_graph* g, const double* d_x, double* d_y_local);

/* ---- shard group: the sharded store with its collectives in the library
 * (SURVEY §8b gpma_shard_group_*, §8e).  One process per GPU; each rank owns
 * the source range [bounds[rank], bounds[rank+1]) (world + 1 host entries,
 * bounds[0] = 0, bounds[world] = num_vertices <= 2^31).  The library issues
 * the NCCL collectives itself on the shard's stream: per batch a count
 * exchange + a grouped send/recv all-to-all of EdgeKeys (+ weights) and one
 * scalar all-reduce (bad inserts reject the batch on every rank before any
 * shard applies); BFS reduce-scatters candidate flags to the owners and
 * gathers the distances, CC all-reduces MIN labels, PageRank all-reduces SUM
 * contributions.  NCCL is bound at run time (libnccl.so.2): without it these
 * entries return PMA_ECUDA, everything else works.  Errors:
 * gpma_shard_group_last_error(). */
typedef struct gpma_shard_group gpma_shard_group;
/* ncclGetUniqueId into 128 bytes (rank 0 creates it; the caller broadcasts it). */
int gpma_nccl_unique_id(void* id128);
/* An NCCL communicator of `world` ranks from a unique id (ncclCommInitRank;
 * the ncclComm_t as void*), for callers without NCCL bindings; several shard
 * groups (e.g. rebuilt graphs) may share it.  Destroy after every group. */
int gpma_nccl_comm_create(const void* id128, int world, int rank, int device, void** comm);
int gpma_nccl_comm_destroy(void* comm);
/* DynamicGraph::from_edges (graph.hpp:66-92) for this rank's shard; the
 * communicator is the caller's ncclComm_t (nccl_comm, not owned) or created
 * from nccl_id128 (owned).  Every rank may pass the same global edge list. */
int gpma_shard_group_create(const gpma_graph_config* cfg, int device, size_t num_vertices, const uint32_t* bounds,
                            int world, int rank, const void* nccl_id128, void* nccl_comm, const uint32_t* d_src,
                            const uint32_t* d_dst, const double* d_weights, size_t n, gpma_shard_group** out);
int gpma_shard_group_destroy(gpma_shard_group* g);
const char* gpma_shard_group_last_error(const gpma_shard_group* g);
/* This rank's shard as a graph handle (row offsets, slots, stats, stream). */
gpma_graph* gpma_shard_group_graph(gpma_shard_group* g);
/* DynamicGraph::apply_batch (graph.hpp:130-162) of this rank's share of a
 * global batch (device arrays): routed to the owners, applied by each owner.
 * stats: this shard's UpdateStats; *routed: updates this shard applied;
 * *sent: updates this rank sent to other ranks. */
int gpma_shard_group_apply_batch(gpma_shard_group* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                                 const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                                 const uint32_t* d_del_dst, size_t n_del, pma_stats* stats, uint64_t* routed,
                                 uint64_t* sent);
/* bfs (analytics.hpp:22-48): dist (host, num_vertices, may be NULL) on every rank. */
int gpma_shard_group_bfs(gpma_shard_group* g, uint32_t root, uint32_t* dist, uint64_t* reached);
/* connected_components (analytics.hpp:53-82): labels (host, num_vertices). */
int gpma_shard_group_cc(gpma_shard_group* g, uint32_t* labels);
/* pagerank (analytics.hpp:84-143) on every rank (host vectors). */
int gpma_shard_group_pagerank(gpma_shard_group* g, double damping, double epsilon, size_t max_iters,
                              const double* warm, double* ranks, uint64_t* iterations, int* converged);
/* spmv (analytics.hpp:147-158): y on every rank (host vectors). */
int gpma_shard_group_spmv(gpma_shard_group* g, const double* x, double* y);

/* Drive every kernel once on small synthetic inputs so CUDA's lazy module
 * loading never lands inside a timed region (call once per process/device). */
int gpma_warmup(int device);

/* ---- Fused routing (partition + transfer in one kernel over peer memory)
 * Instead of gpma_route_batch + an all-to-all: (1) gpma_route_count counts
 * this rank's slice per owner (d_counts[world + 1], [world] = inserts naming
 * a vertex >= |V| as in gpma_route_batch; stream-ordered); (2) the
 * caller exchanges the counts (world x world) and derives, for every owner r,
 * this sender's first slot in r's receive buffer (the sum of the counts of
 * the lower senders for r) and the size of its own receive batch; (3)
 * gpma_route_scatter_peer writes the slice straight into the owners' receive
 * buffers (device pointers: same device, peer-enabled devices, or IPC
 * mappings from gpma_ipc_open); (4) after every sender finished, each owner
 * calls gpma_apply_batch_routed_device on its buffer.  The receive order is
 * the all-to-all's (sender-rank order, arrival order within a sender). */
int gpma_route_count(gpma_graph* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst, size_t n_ins,
                     const uint32_t* d_del_src, const uint32_t* d_del_dst, size_t n_del, const uint32_t* d_bounds,
                     int world, uint64_t* d_counts);
int gpma_route_scatter_peer(gpma_graph* g, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                            const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                            const uint32_t* d_del_dst, size_t n_del, const uint32_t* d_bounds, int world,
                            uint64_t* const* d_dst_keys, double* const* d_dst_w, const uint64_t* d_dst_offsets);
/* cudaMalloc + cudaIpcGetMemHandle (64-byte handle out) / open / close / free */
int gpma_ipc_alloc(int device, size_t bytes, void** d_ptr, void* handle64);
int gpma_ipc_open(int device, const void* handle64, void** d_ptr);
int gpma_ipc_close(void* d_ptr);
int gpma_ipc_free(void* d_ptr);

/* Link diagnostic: best-of-`reps` rate of moving `bytes` of page-locked host
 * memory to the device by cudaMemcpyAsync (copy engines) and by SM loads in
 * place (zero-copy, as gpma_apply_batch reads pinned batches).  GB/s. */
int gpma_probe_h2d(int device, const void* host, size_t bytes, int reps, double* memcpy_gbps,
                   double* zero_copy_gbps);

/* ---- Rebuild-CSR baseline (the paper's rebuild-per-batch comparison point)
 * RebuildCsrGraph (baselines.hpp:85-181) on the device: sorted unique edge
 * list + CSR arrays rebuilt from scratch after every batch.  Same contract as
 * the reference: construction rejects ids >= num_vertices with PMA_EINVAL
 * ("RebuildCsrGraph: vertex id out of range", baselines.hpp:91-93) and keeps
 * the last of duplicate edges (dedupe_last_wins, :160-167); a batch resolves
 * duplicates last-insert-wins (segment_engine.hpp:346-363), counts absent
 * deletes in deletes_missed and reports slot_writes = 2|E| + |V| + 1
 * (:153).  Vertex ids of a batch must be < num_vertices (the reference
 * indexes counts[] with them, :171). */
typedef struct gpma_rebuild gpma_rebuild;

/* RebuildCsrGraph(num_vertices, edges) — baselines.hpp:87-98 (host arrays; w may be NULL = 1.0) */
int gpma_rebuild_create(int device, size_t num_vertices, const uint32_t* src, const uint32_t* dst, const double* w,
                        size_t n, gpma_rebuild** out);
int gpma_rebuild_create_device(int device, size_t num_vertices, const uint32_t* d_src, const uint32_t* d_dst,
                               const double* d_w, size_t n, gpma_rebuild** out);
int gpma_rebuild_destroy(gpma_rebuild* r);
const char* gpma_rebuild_last_error(const gpma_rebuild* r);
/* RebuildCsrGraph::apply_batch — baselines.hpp:114-155 */
int gpma_rebuild_apply_batch(gpma_rebuild* r, const uint32_t* ins_src, const uint32_t* ins_dst, const double* ins_w,
                             size_t n_ins, const uint32_t* del_src, const uint32_t* del_dst, size_t n_del,
                             pma_stats* stats);
int gpma_rebuild_apply_batch_device(gpma_rebuild* r, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                                    const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                                    const uint32_t* d_del_dst, size_t n_del, pma_stats* stats);
/* RebuildCsrGraph::csr_snapshot — baselines.hpp:157-158: row_offsets has
 * num_vertices + 1 entries, col / vals num_edges */
int gpma_rebuild_csr(gpma_rebuild* r, uint64_t* row_offsets, uint32_t* col, double* vals);
uint64_t gpma_rebuild_num_edges(const gpma_rebuild* r);
void* gpma_rebuild_cuda_stream(gpma_rebuild* r);

/* ---- data-parallel primitives (primitives.hpp:21-84) ------------------
 * The library's own device primitives behind the batch pipeline, exposed on
 * their own: a onesweep LSD radix sort (8-bit digits, digits every key shares
 * are skipped as primitives.hpp:38-46 does) and a single-pass exclusive scan.
 * Errors: gpma_primitives_last_error(). */

/* sort_by_key / sort_pairs_by_key (primitives.hpp:21-60): stable ascending
 * sort of n 64-bit keys by key bits [begin_bit, end_bit) (0, 64 = the whole
 * key), the u32 payload (may be NULL) moving with its key; equal keys keep
 * their input order.  Sorted in place; host arrays, or device arrays with
 * the _device variant. */
int gpma_sort_by_key(int device, uint64_t* keys, uint32_t* payload, size_t n, int begin_bit, int end_bit);
int gpma_sort_by_key_device(int device, uint64_t* d_keys, uint32_t* d_payload, size_t n, int begin_bit,
                            int end_bit);
/* exclusive_scan (primitives.hpp:74-84): d_out[0] = 0, d_out[i] = d_out[i-1]
 * + d_in[i-1], n u32 device values (the totals must fit 32 bits). */
int gpma_exclusive_scan_device(int device, const uint32_t* d_in, uint32_t* d_out, size_t n);
const char* gpma_primitives_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PMAGRAPH_CUDA_H */
