#pragma once
// Drop-in <pmagraph/graph.hpp> (reference graph.hpp:23-262): DynamicGraph on
// the device PMA; apply_batch, row offsets, snapshots run on the GPU.
#include <bit>
#include <cstdint>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "pma.hpp"
#include "segment_engine.hpp"
#include "update_stats.hpp"

namespace pmagraph {

using VertexId = std::uint32_t;

struct EdgeKey {  // graph.hpp:27-37
    static constexpr VertexId kGuardDst = std::numeric_limits<VertexId>::max();
    static std::uint64_t pack(VertexId src, VertexId dst) { return (static_cast<std::uint64_t>(src) << 32) | dst; }
    static VertexId src_of(std::uint64_t key) { return static_cast<VertexId>(key >> 32); }
    static VertexId dst_of(std::uint64_t key) { return static_cast<VertexId>(key & 0xffffffffu); }
    static std::uint64_t guard(VertexId src) { return pack(src, kGuardDst); }
    static bool is_guard(std::uint64_t key) { return dst_of(key) == kGuardDst; }
};

struct WeightedEdge {
    VertexId src = 0;
    VertexId dst = 0;
    double weight = 1.0;
};

struct CsrSnapshot {
    std::vector<std::size_t> row_offsets;
    std::vector<VertexId> col_indices;
    std::vector<double> values;
};

enum class UpdateEngine { kSegment, kLock };

struct GraphConfig {  // graph.hpp:54-60 (kSegment only: GPMA+)
    UpdateEngine engine = UpdateEngine::kSegment;
    DeletionMode deletion_mode = DeletionMode::kLazy;
    unsigned workers = 1;
    double fill_target = 0.5;
    DensityProfile profile{};
};

class DynamicGraph {
public:
    static DynamicGraph from_edges(std::size_t num_vertices, std::span<const WeightedEdge> edges,
                                   GraphConfig config = {}) {
        if (config.engine != UpdateEngine::kSegment)
            throw std::invalid_argument("GraphConfig.engine: only the segment engine (GPMA+) is provided");
        std::vector<std::uint32_t> s(edges.size()), d(edges.size());
        std::vector<double> w(edges.size());
        for (std::size_t i = 0; i < edges.size(); ++i) {
            s[i] = edges[i].src;
            d[i] = edges[i].dst;
            w[i] = edges[i].weight;
        }
        const gpma_graph_config c{0, config.deletion_mode == DeletionMode::kEager ? PMA_EAGER : PMA_LAZY,
                                  config.workers, 0, config.fill_target, config.profile.c()};
        gpma_graph* g = nullptr;
        if (int rc = gpma_from_edges(&c, detail_cuda::default_device(), num_vertices, s.data(), d.data(), w.data(),
                                     s.size(), &g))
            detail_cuda::raise(rc, gpma_last_error(nullptr));
        return DynamicGraph(g, num_vertices, config);
    }

    DynamicGraph(DynamicGraph&& o) noexcept
        : g_(o.g_), nv_(o.nv_), config_(o.config_), pma_(std::move(o.pma_)), ro_(std::move(o.ro_)), ro_ok_(o.ro_ok_) {
        o.g_ = nullptr;
    }
    DynamicGraph& operator=(DynamicGraph&& o) noexcept {
        if (this != &o) {
            if (g_) gpma_destroy(g_);
            g_ = o.g_;
            nv_ = o.nv_;
            config_ = o.config_;
            pma_ = std::move(o.pma_);
            ro_ = std::move(o.ro_);
            ro_ok_ = o.ro_ok_;
            o.g_ = nullptr;
        }
        return *this;
    }
    DynamicGraph(const DynamicGraph&) = delete;
    ~DynamicGraph() {
        if (g_) gpma_destroy(g_);
    }

    std::size_t num_vertices() const { return nv_; }
    std::size_t num_edges() const { return gpma_num_edges(g_); }
    const PackedMemoryArray& pma() const { return pma_; }
    const std::vector<std::size_t>& row_offsets() const {
        if (!ro_ok_) {
            std::vector<std::uint64_t> r(nv_ + 1);
            check(gpma_row_offsets(g_, r.data()));
            ro_.assign(r.begin(), r.end());
            ro_ok_ = true;
        }
        return ro_;
    }
    bool is_entry_exist(std::size_t slot) const {
        const Slot& s = pma_.slots()[slot];
        return s.state == SlotState::kValid && !EdgeKey::is_guard(s.key);
    }
    template <typename Fn>
    void for_each_neighbor(VertexId v, Fn&& fn) const {
        const auto& ro = row_offsets();
        const auto& slots = pma_.slots();
        for (std::size_t i = ro[v]; i < ro[v + 1]; ++i) {
            if (!is_entry_exist(i)) continue;
            fn(EdgeKey::dst_of(slots[i].key), std::bit_cast<double>(slots[i].value));
        }
    }
    std::size_t degree(VertexId v) const {
        std::size_t d = 0;
        for_each_neighbor(v, [&](VertexId, double) { ++d; });
        return d;
    }
    std::optional<double> edge_weight(VertexId src, VertexId dst) const {
        const auto v = pma_.search(EdgeKey::pack(src, dst));
        if (!v) return std::nullopt;
        return std::bit_cast<double>(*v);
    }
    UpdateStats apply_batch(std::span<const WeightedEdge> inserts,
                            std::span<const std::pair<VertexId, VertexId>> deletes, WorkerPool* pool = nullptr) {
        (void)pool;
        std::vector<std::uint32_t> is(inserts.size()), id(inserts.size()), ds(deletes.size()), dd(deletes.size());
        std::vector<double> iw(inserts.size());
        for (std::size_t i = 0; i < inserts.size(); ++i) {
            is[i] = inserts[i].src;
            id[i] = inserts[i].dst;
            iw[i] = inserts[i].weight;
        }
        for (std::size_t i = 0; i < deletes.size(); ++i) {
            ds[i] = deletes[i].first;
            dd[i] = deletes[i].second;
        }
        pma_stats st{};
        pma_.invalidate();
        ro_ok_ = false;
        check(gpma_apply_batch(g_, is.data(), id.data(), iw.data(), is.size(), ds.data(), dd.data(), ds.size(), &st));
        return UpdateStats::from_c(st, gpma_pma(g_));
    }
    void rebuild_row_offsets() {
        ro_ok_ = false;
        check(gpma_rebuild_row_offsets(g_));
    }
    CsrSnapshot csr_snapshot() const {
        CsrSnapshot snap;
        const std::size_t ne = num_edges();
        std::vector<std::uint64_t> ro(nv_ + 1);
        snap.col_indices.resize(ne);
        snap.values.resize(ne);
        check(gpma_csr_snapshot(g_, ro.data(), snap.col_indices.data(), snap.values.data()));
        snap.row_offsets.assign(ro.begin(), ro.end());
        return snap;
    }
    std::vector<WeightedEdge> edge_list() const {
        std::vector<WeightedEdge> out;
        pma_.for_each_valid([&](std::uint64_t key, std::uint64_t value) {
            if (!EdgeKey::is_guard(key))
                out.push_back(WeightedEdge{EdgeKey::src_of(key), EdgeKey::dst_of(key), std::bit_cast<double>(value)});
        });
        return out;
    }
    std::size_t guard_count() const {
        std::size_t n = 0;
        pma_.for_each_valid([&](std::uint64_t key, std::uint64_t) { n += EdgeKey::is_guard(key); });
        return n;
    }
    gpma_graph* handle() const { return g_; }
    void check(int rc) const {
        if (rc) detail_cuda::raise(rc, gpma_last_error(g_));
    }

private:
    DynamicGraph(gpma_graph* g, std::size_t nv, GraphConfig config)
        : g_(g), nv_(nv), config_(config), pma_(gpma_pma(g), config.profile) {}

    gpma_graph* g_ = nullptr;
    std::size_t nv_ = 0;
    GraphConfig config_{};
    PackedMemoryArray pma_;
    mutable std::vector<std::size_t> ro_;
    mutable bool ro_ok_ = false;
};

// Read-only graph view over compact CSR arrays (graph.hpp:244-260).
class CsrView {
public:
    explicit CsrView(const CsrSnapshot& snap) : snap_(&snap) {}
    std::size_t num_vertices() const { return snap_->row_offsets.size() - 1; }
    template <typename Fn>
    void for_each_neighbor(VertexId v, Fn&& fn) const {
        for (std::size_t i = snap_->row_offsets[v]; i < snap_->row_offsets[v + 1]; ++i)
            fn(snap_->col_indices[i], snap_->values[i]);
    }
    const CsrSnapshot& snapshot() const { return *snap_; }

private:
    const CsrSnapshot* snap_;
};

}  // namespace pmagraph
