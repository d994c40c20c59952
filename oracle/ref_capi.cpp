// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Exposes the UNMODIFIED reference implementation (header-only C++20 under
// /root/reference/proj/include/pmagraph, compiled from where it lies by
// oracle/Makefile) through a C ABI, so tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg can drive it via ctypes.
// Nothing here is copied from the reference: this file only calls its public
// API (pma.hpp, segment_engine.hpp, graph.hpp, analytics.hpp, streaming.hpp,
// generators.hpp, baselines.hpp).  The POD structs are shared with the product ABI
// (include/pmagraph_cuda.h) so results compare field by field.
//
// Output: oracle/_ref/libpmagraph_ref.so (git-ignored, travels to the GPU box).

#include <pmagraph/analytics.hpp>
#include <pmagraph/baselines.hpp>
#include <pmagraph/generators.hpp>
#include <pmagraph/graph.hpp>
#include <pmagraph/io.hpp>
#include <pmagraph/pma.hpp>
#include <pmagraph/segment_engine.hpp>
#include <pmagraph/streaming.hpp>

#include <chrono>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>

#include "pmagraph_cuda.h"

using namespace pmagraph;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return PMA_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PMA_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return PMA_ERANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return PMA_ELOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PMA_ECUDA;
    }
}

DensityProfile to_profile(const pma_profile* p) {
    DensityProfile d;
    if (p != nullptr) {
        d.leaf_lower = p->leaf_lower;
        d.leaf_upper = p->leaf_upper;
        d.root_lower = p->root_lower;
        d.root_upper = p->root_upper;
        d.allow_shrink = p->allow_shrink != 0;
    }
    return d;
}

SegmentEngineConfig to_engine(const pma_engine_config* c) {
    SegmentEngineConfig cfg;
    if (c != nullptr) {
        cfg.deletion_mode = c->deletion_mode == PMA_EAGER ? DeletionMode::kEager : DeletionMode::kLazy;
        cfg.workers = c->workers == 0 ? 1 : c->workers;
        cfg.tiers.small_max = c->small_max;
        cfg.tiers.medium_max = c->medium_max;
        if (c->force_strategy >= 0) cfg.force_strategy = static_cast<MergeStrategy>(c->force_strategy);
    }
    return cfg;
}

void fill_stats(const UpdateStats& s, pma_stats* out) {
    if (out == nullptr) return;
    std::memset(out, 0, sizeof(*out));
    out->batch_size = s.batch_size;
    out->rounds = s.rounds;
    out->slot_writes = s.slot_writes;
    out->wall_ns = s.wall_ns;
    out->segment_phase_ns = s.segment_phase_ns;
    out->grow_events = s.grow_events;
    out->shrink_events = s.shrink_events;
    out->deletes_missed = s.deletes_missed;
    out->tombstones_added = s.tombstones_added;
    out->num_touched_ranges = s.touched_ranges.size();
    out->resized = s.resized ? 1 : 0;
    out->num_levels = static_cast<int32_t>(s.segments_per_level.size());
    for (std::size_t i = 0; i < s.segments_per_level.size() && i < PMA_MAX_LEVELS; ++i) {
        out->segments_per_level[i] = s.segments_per_level[i];
    }
}

void download(const PackedMemoryArray& p, uint64_t* keys, uint64_t* values, uint8_t* states) {
    const auto& slots = p.slots();
    for (std::size_t i = 0; i < slots.size(); ++i) {
        if (keys) keys[i] = slots[i].key;
        if (values) values[i] = slots[i].value;
        if (states) states[i] = static_cast<uint8_t>(slots[i].state);
    }
}

}  // namespace

struct ref_pma {
    PackedMemoryArray pma;
    UpdateStats last;
};

struct ref_graph {
    std::optional<DynamicGraph> g;
    UpdateStats last;
};

struct ref_stream {
    EdgeStream s;
};

struct ref_window {
    const ref_stream* stream;
    std::optional<SlidingWindow> w;
    SlideBatch last;
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// ---- PackedMemoryArray -----------------------------------------------------

int ref_pma_create(const pma_profile* profile, ref_pma** out) {
    return guarded([&] { *out = new ref_pma{PackedMemoryArray(to_profile(profile)), {}}; });
}

void ref_pma_destroy(ref_pma* h) { delete h; }

int ref_pma_from_sorted(ref_pma* h, const uint64_t* keys, const uint64_t* values, size_t n,
                        double fill_target) {
    return guarded([&] {
        std::vector<Entry> e(n);
        for (size_t i = 0; i < n; ++i) e[i] = Entry{keys[i], values ? values[i] : 0};
        h->pma = PackedMemoryArray::from_sorted(e, fill_target, h->pma.profile());
    });
}

// Exact restore through public API: from_slot_layout for every non-empty
// slot, then mark_tombstone for the tombstones, then reset_slot_writes.
int ref_pma_load_slots(ref_pma* h, size_t capacity, const uint64_t* keys, const uint64_t* values,
                       const uint8_t* states) {
    return guarded([&] {
        std::vector<std::tuple<std::size_t, std::uint64_t, std::uint64_t>> placements;
        for (size_t i = 0; i < capacity; ++i) {
            if (states[i] != 0) placements.emplace_back(i, keys[i], values[i]);
        }
        h->pma = PackedMemoryArray::from_slot_layout(capacity, placements, h->pma.profile());
        for (size_t i = 0; i < capacity; ++i) {
            if (states[i] == 2) h->pma.mark_tombstone_at(i);
        }
        h->pma.reset_slot_writes();
    });
}

int ref_pma_download(ref_pma* h, uint64_t* keys, uint64_t* values, uint8_t* states) {
    return guarded([&] { download(h->pma, keys, values, states); });
}

int ref_pma_get_layout(ref_pma* h, pma_layout_info* out) {
    return guarded([&] {
        out->capacity = h->pma.capacity();
        out->leaf_size = h->pma.layout().leaf_size();
        out->height = h->pma.layout().height();
        out->valid_count = h->pma.valid_count();
        out->tombstone_count = h->pma.tombstone_count();
        out->slot_writes = h->pma.slot_writes();
    });
}

int ref_pma_reset_slot_writes(ref_pma* h) {
    return guarded([&] { h->pma.reset_slot_writes(); });
}

int ref_pma_bounds(ref_pma* h, int level, uint64_t* mn, uint64_t* mx, double* rho, double* tau) {
    return guarded([&] {
        const auto [lo, hi] = h->pma.thresholds(level);
        if (mn) *mn = h->pma.min_entries(level);
        if (mx) *mx = h->pma.max_entries(level);
        if (rho) *rho = lo;
        if (tau) *tau = hi;
    });
}

int ref_pma_batch_update(ref_pma* h, const uint64_t* keys, const uint64_t* values, const uint8_t* ops,
                         size_t n, const pma_engine_config* cfg, pma_stats* out) {
    return guarded([&] {
        std::vector<Update> ups(n);
        for (size_t i = 0; i < n; ++i) {
            ups[i] = Update{keys[i], values ? values[i] : 0,
                            ops[i] == 0 ? UpdateOp::kInsert : UpdateOp::kDelete};
        }
        h->last = batch_update(h->pma, std::move(ups), to_engine(cfg));
        fill_stats(h->last, out);
    });
}

int ref_pma_touched_ranges(ref_pma* h, uint64_t* pairs, size_t cap, size_t* count) {
    return guarded([&] {
        const auto& tr = h->last.touched_ranges;
        *count = tr.size();
        for (size_t i = 0; i < tr.size() && i < cap; ++i) {
            pairs[2 * i] = tr[i].first;
            pairs[2 * i + 1] = tr[i].second;
        }
    });
}

int ref_pma_binary_search_leaf(ref_pma* h, const uint64_t* keys, size_t n, uint64_t* leaves) {
    return guarded([&] {
        for (size_t i = 0; i < n; ++i) leaves[i] = h->pma.binary_search_leaf(keys[i]);
    });
}

int ref_pma_assign_leaves_sorted(ref_pma* h, const uint64_t* keys, size_t n, uint64_t* leaves) {
    return guarded([&] {
        std::vector<std::size_t> out(n);
        h->pma.assign_leaves_sorted(std::span<const std::uint64_t>(keys, n), out);
        for (size_t i = 0; i < n; ++i) leaves[i] = out[i];
    });
}

int ref_pma_search(ref_pma* h, const uint64_t* keys, size_t n, uint64_t* values, uint8_t* found) {
    return guarded([&] {
        for (size_t i = 0; i < n; ++i) {
            const auto v = h->pma.search(keys[i]);
            found[i] = v.has_value() ? 1 : 0;
            values[i] = v.value_or(0);
        }
    });
}

int ref_pma_count_valid_in(ref_pma* h, size_t b, size_t e, uint64_t* count) {
    return guarded([&] { *count = h->pma.count_valid_in(b, e); });
}

int ref_pma_insert(ref_pma* h, uint64_t key, uint64_t value) {
    return guarded([&] { h->pma.insert(key, value); });
}

int ref_pma_erase(ref_pma* h, uint64_t key, int* erased) {
    return guarded([&] { *erased = h->pma.erase(key) ? 1 : 0; });
}

int ref_pma_mark_tombstone(ref_pma* h, uint64_t key, int* marked) {
    return guarded([&] { *marked = h->pma.mark_tombstone(key) ? 1 : 0; });
}

int ref_pma_redispatch(ref_pma* h, int level, size_t seg, const uint64_t* keys, const uint64_t* values,
                       size_t n) {
    return guarded([&] {
        std::vector<Entry> e(n);
        for (size_t i = 0; i < n; ++i) e[i] = Entry{keys[i], values ? values[i] : 0};
        h->pma.redispatch(level, seg, e);
    });
}

// ---- DynamicGraph ----------------------------------------------------------

static GraphConfig to_graph_config(const gpma_graph_config* c) {
    GraphConfig cfg;
    if (c != nullptr) {
        cfg.engine = c->engine == 0 ? UpdateEngine::kSegment : UpdateEngine::kLock;
        cfg.deletion_mode = c->deletion_mode == PMA_EAGER ? DeletionMode::kEager : DeletionMode::kLazy;
        cfg.workers = c->workers == 0 ? 1 : c->workers;
        cfg.fill_target = c->fill_target;
        cfg.profile = to_profile(&c->profile);
    }
    return cfg;
}

int ref_graph_from_edges(const gpma_graph_config* cfg, size_t nv, const uint32_t* src, const uint32_t* dst,
                         const double* w, size_t n, ref_graph** out) {
    return guarded([&] {
        std::vector<WeightedEdge> edges(n);
        for (size_t i = 0; i < n; ++i) edges[i] = WeightedEdge{src[i], dst[i], w ? w[i] : 1.0};
        auto* g = new ref_graph{};
        try {
            g->g.emplace(DynamicGraph::from_edges(nv, edges, to_graph_config(cfg)));
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

void ref_graph_destroy(ref_graph* g) { delete g; }

int ref_graph_apply_batch(ref_graph* g, const uint32_t* is, const uint32_t* id, const double* iw, size_t ni,
                          const uint32_t* ds, const uint32_t* dd, size_t nd, pma_stats* out) {
    return guarded([&] {
        std::vector<WeightedEdge> ins(ni);
        for (size_t i = 0; i < ni; ++i) ins[i] = WeightedEdge{is[i], id[i], iw ? iw[i] : 1.0};
        std::vector<std::pair<VertexId, VertexId>> del(nd);
        for (size_t i = 0; i < nd; ++i) del[i] = {ds[i], dd[i]};
        g->last = g->g->apply_batch(ins, del);
        fill_stats(g->last, out);
    });
}

// Host steady-clock time around DynamicGraph::apply_batch (the CPU baseline).
int ref_graph_apply_batch_timed(ref_graph* g, const uint32_t* is, const uint32_t* id, const double* iw,
                                size_t ni, const uint32_t* ds, const uint32_t* dd, size_t nd, unsigned workers,
                                pma_stats* out, double* wall_ms) {
    return guarded([&] {
        std::vector<WeightedEdge> ins(ni);
        for (size_t i = 0; i < ni; ++i) ins[i] = WeightedEdge{is[i], id[i], iw ? iw[i] : 1.0};
        std::vector<std::pair<VertexId, VertexId>> del(nd);
        for (size_t i = 0; i < nd; ++i) del[i] = {ds[i], dd[i]};
        WorkerPool pool(workers == 0 ? 1 : workers);
        const auto t0 = std::chrono::steady_clock::now();
        g->last = g->g->apply_batch(ins, del, &pool);
        const auto t1 = std::chrono::steady_clock::now();
        *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        fill_stats(g->last, out);
    });
}

int ref_graph_touched_ranges(ref_graph* g, uint64_t* pairs, size_t cap, size_t* count) {
    return guarded([&] {
        const auto& tr = g->last.touched_ranges;
        *count = tr.size();
        for (size_t i = 0; i < tr.size() && i < cap; ++i) {
            pairs[2 * i] = tr[i].first;
            pairs[2 * i + 1] = tr[i].second;
        }
    });
}

int ref_graph_layout(ref_graph* g, pma_layout_info* out) {
    return guarded([&] {
        const auto& p = g->g->pma();
        out->capacity = p.capacity();
        out->leaf_size = p.layout().leaf_size();
        out->height = p.layout().height();
        out->valid_count = p.valid_count();
        out->tombstone_count = p.tombstone_count();
        out->slot_writes = p.slot_writes();
    });
}

int ref_graph_download(ref_graph* g, uint64_t* keys, uint64_t* values, uint8_t* states) {
    return guarded([&] { download(g->g->pma(), keys, values, states); });
}

int ref_graph_row_offsets(ref_graph* g, uint64_t* out) {
    return guarded([&] {
        const auto& ro = g->g->row_offsets();
        for (size_t i = 0; i < ro.size(); ++i) out[i] = ro[i];
    });
}

uint64_t ref_graph_num_edges(ref_graph* g) { return g->g->num_edges(); }

int ref_graph_csr_snapshot(ref_graph* g, uint64_t* ro, uint32_t* col, double* val) {
    return guarded([&] {
        const CsrSnapshot s = g->g->csr_snapshot();
        for (size_t i = 0; i < s.row_offsets.size(); ++i) ro[i] = s.row_offsets[i];
        for (size_t i = 0; i < s.col_indices.size(); ++i) {
            col[i] = s.col_indices[i];
            val[i] = s.values[i];
        }
    });
}

// RebuildCsrGraph (baselines.hpp:85-181): the rebuild-the-CSR-per-batch
// baseline of the paper's comparison.
struct ref_rebuild {
    std::optional<RebuildCsrGraph> g;
};

int ref_rebuild_create(size_t nv, const uint32_t* src, const uint32_t* dst, const double* w, size_t n,
                       ref_rebuild** out) {
    return guarded([&] {
        std::vector<WeightedEdge> edges(n);
        for (size_t i = 0; i < n; ++i) edges[i] = WeightedEdge{src[i], dst[i], w ? w[i] : 1.0};
        auto* g = new ref_rebuild{};
        try {
            g->g.emplace(nv, edges);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

void ref_rebuild_destroy(ref_rebuild* g) { delete g; }

uint64_t ref_rebuild_num_edges(ref_rebuild* g) { return g->g->num_edges(); }

int ref_rebuild_apply_batch(ref_rebuild* g, const uint32_t* is, const uint32_t* id, const double* iw, size_t ni,
                            const uint32_t* ds, const uint32_t* dd, size_t nd, pma_stats* out) {
    return guarded([&] {
        std::vector<WeightedEdge> ins(ni);
        for (size_t i = 0; i < ni; ++i) ins[i] = WeightedEdge{is[i], id[i], iw ? iw[i] : 1.0};
        std::vector<std::pair<VertexId, VertexId>> del(nd);
        for (size_t i = 0; i < nd; ++i) del[i] = {ds[i], dd[i]};
        fill_stats(g->g->apply_batch(ins, del), out);
    });
}

int ref_rebuild_csr(ref_rebuild* g, uint64_t* ro, uint32_t* col, double* val) {
    return guarded([&] {
        const CsrSnapshot& c = g->g->csr();
        for (size_t i = 0; i < c.row_offsets.size(); ++i) ro[i] = c.row_offsets[i];
        for (size_t i = 0; i < c.col_indices.size(); ++i) {
            col[i] = c.col_indices[i];
            val[i] = c.values[i];
        }
    });
}

int ref_bfs(ref_graph* g, uint32_t root, uint32_t* dist, double* wall_ms) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const auto d = bfs(*g->g, root);
        const auto t1 = std::chrono::steady_clock::now();
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(dist, d.data(), d.size() * sizeof(uint32_t));
    });
}

int ref_cc(ref_graph* g, uint32_t* labels, double* wall_ms) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const auto l = connected_components(*g->g);
        const auto t1 = std::chrono::steady_clock::now();
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(labels, l.data(), l.size() * sizeof(uint32_t));
    });
}

int ref_pagerank(ref_graph* g, double damping, double eps, size_t max_iters, const double* warm, double* ranks,
                 uint64_t* iters, int* converged, double* wall_ms) {
    return guarded([&] {
        PageRankOptions o;
        o.damping = damping;
        o.epsilon = eps;
        o.max_iters = max_iters;
        std::vector<double> w;
        if (warm != nullptr) {
            w.assign(warm, warm + g->g->num_vertices());
            o.warm_start = &w;
        }
        const auto t0 = std::chrono::steady_clock::now();
        const PageRankResult r = pagerank(*g->g, o);
        const auto t1 = std::chrono::steady_clock::now();
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::memcpy(ranks, r.ranks.data(), r.ranks.size() * sizeof(double));
        *iters = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

int ref_spmv(ref_graph* g, const double* x, double* y) {
    return guarded([&] {
        std::vector<double> xv(x, x + g->g->num_vertices());
        const auto r = spmv(*g->g, xv);
        std::memcpy(y, r.data(), r.size() * sizeof(double));
    });
}

// ---- streams (generators.hpp, streaming.hpp) --------------------------------

int ref_gen_rmat(size_t nv, size_t ne, double a, double b, double c, double d, uint64_t seed, ref_stream** out) {
    return guarded([&] { *out = new ref_stream{gen_rmat(nv, ne, RmatParams{a, b, c, d}, seed)}; });
}

int ref_gen_erdos_renyi(size_t nv, double p, uint64_t seed, ref_stream** out) {
    return guarded([&] { *out = new ref_stream{gen_erdos_renyi(nv, p, seed)}; });
}

// assign_random_timestamps (streaming.hpp:58-67) applied in place.
int ref_stream_shuffle(ref_stream* s, uint64_t seed) {
    return guarded([&] { s->s = assign_random_timestamps(std::move(s->s.edges), s->s.num_vertices, seed); });
}

int ref_stream_from_arrays(size_t nv, const uint32_t* src, const uint32_t* dst, const double* w, size_t n,
                           ref_stream** out) {
    return guarded([&] {
        auto* s = new ref_stream{};
        s->s.num_vertices = nv;
        s->s.edges.resize(n);
        for (size_t i = 0; i < n; ++i) s->s.edges[i] = TimestampedEdge{src[i], dst[i], w ? w[i] : 1.0, i};
        *out = s;
    });
}

void ref_stream_destroy(ref_stream* s) { delete s; }
uint64_t ref_stream_size(ref_stream* s) { return s->s.edges.size(); }
uint64_t ref_stream_num_vertices(ref_stream* s) { return s->s.num_vertices; }

int ref_stream_edges(ref_stream* s, uint32_t* src, uint32_t* dst, double* w, uint64_t* ts) {
    return guarded([&] {
        const auto& e = s->s.edges;
        for (size_t i = 0; i < e.size(); ++i) {
            if (src) src[i] = e[i].src;
            if (dst) dst[i] = e[i].dst;
            if (w) w[i] = e[i].weight;
            if (ts) ts[i] = e[i].ts;
        }
    });
}

int ref_window_create(ref_stream* s, ref_window** out) {
    return guarded([&] {
        auto* w = new ref_window{s, std::nullopt, {}};
        w->w.emplace(s->s);
        *out = w;
    });
}

void ref_window_destroy(ref_window* w) { delete w; }
uint64_t ref_window_size(ref_window* w) { return w->w->window_size(); }
uint64_t ref_window_remaining(ref_window* w) { return w->w->remaining(); }

// slide(batch) (streaming.hpp:107-123); sizes of the result via out params,
// contents via ref_window_last_*.
int ref_window_slide(ref_window* w, size_t batch, uint64_t* n_ins, uint64_t* n_del) {
    return guarded([&] {
        w->last = w->w->slide(batch);
        *n_ins = w->last.inserts.size();
        *n_del = w->last.deletions.size();
    });
}

// SlidingWindow::slide_explicit_random (streaming.hpp:129-158) with a caller-owned
// engine (its state advances across calls, as the reference's std::mt19937_64&)
struct ref_rng {
    std::mt19937_64 r;
};
int ref_rng_create(uint64_t seed, ref_rng** out) {
    return guarded([&] { *out = new ref_rng{std::mt19937_64(seed)}; });
}
int ref_rng_destroy(ref_rng* r) {
    delete r;
    return 0;
}
int ref_window_slide_explicit_random(ref_window* w, size_t batch, ref_rng* rng, uint64_t* n_ins, uint64_t* n_del) {
    return guarded([&] {
        w->last = w->w->slide_explicit_random(batch, rng->r);
        *n_ins = w->last.inserts.size();
        *n_del = w->last.deletions.size();
    });
}

int ref_window_last(ref_window* w, uint32_t* is, uint32_t* id, double* iw, uint32_t* ds, uint32_t* dd) {
    return guarded([&] {
        const auto& b = w->last;
        for (size_t i = 0; i < b.inserts.size(); ++i) {
            is[i] = b.inserts[i].src;
            id[i] = b.inserts[i].dst;
            if (iw) iw[i] = b.inserts[i].weight;
        }
        for (size_t i = 0; i < b.deletions.size(); ++i) {
            ds[i] = b.deletions[i].first;
            dd[i] = b.deletions[i].second;
        }
    });
}

// draw_below (streaming.hpp:43-50) over a fresh mt19937_64(seed): the bench's
// BFS-root sequence (bench.hpp:244,266).
int ref_draw_below_sequence(uint64_t seed, uint64_t bound, size_t n, uint64_t* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        for (size_t i = 0; i < n; ++i) out[i] = draw_below(rng, bound);
    });
}

// ---- io.hpp: the reference's file formats, for byte-level comparisons ----
int ref_io_format_double(double v, char* buf, size_t cap) {
    return guarded([&] {
        const std::string s = format_double(v);
        if (s.size() + 1 > cap) throw std::length_error("buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int ref_io_write_pairs(const char* path, int text, const uint64_t* keys, const uint64_t* values, size_t n) {
    return guarded([&] {
        std::vector<Entry> e(n);
        for (size_t i = 0; i < n; ++i) e[i] = Entry{keys[i], values[i]};
        if (text) write_pairs_text(path, e);
        else write_pairs_binary(path, e);
    });
}

namespace {
thread_local std::vector<Entry> g_pairs;
thread_local EdgeStream g_stream;
}  // namespace

int ref_io_read_pairs(const char* path, int text, uint64_t* n) {
    return guarded([&] {
        g_pairs = text ? read_pairs_text(path) : read_pairs_binary(path);
        *n = g_pairs.size();
    });
}

int ref_io_pairs_copy(uint64_t* keys, uint64_t* values) {
    return guarded([&] {
        for (size_t i = 0; i < g_pairs.size(); ++i) {
            keys[i] = g_pairs[i].key;
            values[i] = g_pairs[i].value;
        }
    });
}

int ref_io_write_stream(const char* path, int text, size_t nv, const uint32_t* src, const uint32_t* dst,
                        const double* w, const uint64_t* ts, size_t n) {
    return guarded([&] {
        EdgeStream st;
        st.num_vertices = nv;
        st.edges.resize(n);
        for (size_t i = 0; i < n; ++i) st.edges[i] = TimestampedEdge{src[i], dst[i], w[i], ts[i]};
        if (text) write_stream_text(path, st);
        else write_stream_binary(path, st);
    });
}

// mode: 0 read_stream (format probe), 1 text, 2 binary
int ref_io_read_stream(const char* path, int mode, uint64_t* nv, uint64_t* n) {
    return guarded([&] {
        g_stream = mode == 1 ? read_stream_text(path) : mode == 2 ? read_stream_binary(path) : read_stream(path);
        *nv = g_stream.num_vertices;
        *n = g_stream.edges.size();
    });
}

int ref_io_stream_copy(uint32_t* src, uint32_t* dst, double* w, uint64_t* ts) {
    return guarded([&] {
        for (size_t i = 0; i < g_stream.edges.size(); ++i) {
            src[i] = g_stream.edges[i].src;
            dst[i] = g_stream.edges[i].dst;
            w[i] = g_stream.edges[i].weight;
            ts[i] = g_stream.edges[i].ts;
        }
    });
}

// kind: 0 f64, 1 u32, 2 u64
int ref_io_write_vector(const char* path, int text, int kind, const void* data, size_t n) {
    return guarded([&] {
        auto go = [&](auto* p) {
            using T = std::remove_cv_t<std::remove_pointer_t<decltype(p)>>;
            std::vector<T> v(p, p + n);
            if (text) write_vector_text(path, v);
            else write_vector_binary(path, v);
        };
        if (kind == 0) go(static_cast<const double*>(data));
        else if (kind == 1) go(static_cast<const uint32_t*>(data));
        else go(static_cast<const uint64_t*>(data));
    });
}

}  // extern "C"
