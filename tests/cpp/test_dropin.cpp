// C++ drop-in check: the reference's public API (pmagraph:: names from
// include/pmagraph/*.hpp) used exactly as the reference's own tests use it,
// running on the GPU through libpmagraph_cuda.so.  Expected values are the
// known answers of proj/tests/test_pma.cpp, test_segment_engine.cpp,
// test_graph.cpp and test_analytics.cpp.  Exit code = number of failures.
#include <pmagraph/analytics.hpp>
#include <pmagraph/graph.hpp>
#include <pmagraph/pma.hpp>
#include <pmagraph/segment_engine.hpp>

#include <cmath>
#include <cstdio>
#include <map>
#include <random>
#include <tuple>
#include <vector>

using namespace pmagraph;

static int failures = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

static PackedMemoryArray fixture() {
    const std::uint64_t keys[] = {2, 8, 10, 11, 14, 17, 20, 25, 30, 33, 36, 40, 45, 50, 60, 70, 80, 90};
    const std::size_t slots[] = {0, 4, 5, 6, 8, 9, 12, 13, 16, 17, 18, 20, 21, 22, 24, 25, 28, 29};
    std::vector<std::tuple<std::size_t, std::uint64_t, std::uint64_t>> p;
    for (int i = 0; i < 18; ++i) p.emplace_back(slots[i], keys[i], keys[i] * 10);
    return PackedMemoryArray::from_slot_layout(32, p);
}

static std::vector<Update> inserts(std::initializer_list<std::uint64_t> keys) {
    std::vector<Update> b;
    for (auto k : keys) b.push_back(Update{k, k * 10, UpdateOp::kInsert});
    return b;
}

int main() {
    {  // thresholds (test_pma.cpp:14-41)
        PackedMemoryArray pma = fixture();
        CHECK(pma.capacity() == 32 && pma.layout().leaf_size() == 4 && pma.layout().height() == 3);
        const std::size_t mins[] = {1, 2, 4, 8}, maxs[] = {3, 6, 12, 24};
        for (int l = 0; l <= 3; ++l) CHECK(pma.min_entries(l) == mins[l] && pma.max_entries(l) == maxs[l]);
        bool threw = false;
        try {
            pma.thresholds(4);
        } catch (const std::out_of_range&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // leaf search (test_pma.cpp:81-89)
        PackedMemoryArray pma = fixture();
        CHECK(pma.binary_search_leaf(48) == 5 && pma.binary_search_leaf(35) == 4 && pma.binary_search_leaf(9) == 1);
        CHECK(pma.binary_search_leaf(1) == 0 && pma.binary_search_leaf(4) == 0 && pma.binary_search_leaf(1000) == 7);
    }
    {  // five-insert batch (test_segment_engine.cpp:53-73)
        PackedMemoryArray pma = fixture();
        const UpdateStats st = batch_update(pma, inserts({1, 4, 9, 35, 48}));
        CHECK(st.rounds == 3);
        CHECK((st.segments_per_level == std::vector<std::size_t>{1, 0, 2, 0}));
        CHECK(st.grow_events == 0 && pma.valid_count() == 23);
        for (std::uint64_t k : {1, 4, 9, 35, 48}) CHECK(pma.search(k) == std::optional<std::uint64_t>(k * 10));
    }
    {  // lazy deletes tombstone (test_segment_engine.cpp:263-286)
        PackedMemoryArray pma = fixture();
        const auto before = pma.slots();
        SegmentEngineConfig cfg;
        cfg.deletion_mode = DeletionMode::kLazy;
        const UpdateStats st = batch_update(
            pma, {Update{30, 0, UpdateOp::kDelete}, Update{45, 0, UpdateOp::kDelete}, Update{999, 0, UpdateOp::kDelete}},
            cfg);
        CHECK(st.rounds == 1 && st.tombstones_added == 2 && st.deletes_missed == 1 && st.touched_ranges.empty());
        CHECK(pma.tombstone_count() == 2 && !pma.search(30).has_value());
        for (std::size_t i = 0; i < before.size(); ++i) CHECK(before[i].key == pma.slots()[i].key);
        batch_update(pma, inserts({31, 46}), cfg);
        CHECK(pma.tombstone_count() == 0 && pma.search(31).has_value());
    }
    {  // growth exactly once (test_segment_engine.cpp:250-261)
        PackedMemoryArray pma;
        const std::size_t root_max = pma.max_entries(pma.layout().height());
        for (std::size_t i = 0; i < root_max; ++i) pma.insert(i * 7, i);
        CHECK(pma.capacity() == PackedMemoryArray::kMinCapacity);
        const UpdateStats st = batch_update(pma, inserts({3, 10, 17, 24}));
        CHECK(st.grow_events == 1 && st.resized && pma.capacity() == 32);
    }
    {  // insert 48 re-dispatches [16,31] (test_pma.cpp:132-153)
        PackedMemoryArray pma = fixture();
        pma.insert(48, 480);
        const std::pair<std::size_t, std::uint64_t> want[] = {{16, 30}, {17, 33}, {18, 36}, {20, 40}, {21, 45}, {23, 48},
                                                             {24, 50}, {26, 60}, {27, 70}, {29, 80}, {30, 90}};
        for (auto [slot, key] : want) CHECK(pma.slots()[slot].state == SlotState::kValid && pma.slots()[slot].key == key);
    }
    {  // random trace vs ordered map (test_segment_engine.cpp:185-216 style)
        std::mt19937_64 rng(41);
        PackedMemoryArray pma;
        std::map<std::uint64_t, std::uint64_t> oracle;
        for (int b = 0; b < 12; ++b) {
            std::vector<Update> batch;
            std::map<std::uint64_t, std::optional<std::uint64_t>> resolved;
            for (int i = 0; i < 300; ++i) {
                const std::uint64_t key = rng() % 20000;
                if (rng() % 10 < 4) {
                    batch.push_back(Update{key, 0, UpdateOp::kDelete});
                    if (!resolved.count(key)) resolved[key] = std::nullopt;
                } else {
                    const std::uint64_t v = rng();
                    batch.push_back(Update{key, v, UpdateOp::kInsert});
                    resolved[key] = v;
                }
            }
            SegmentEngineConfig cfg;
            cfg.deletion_mode = b % 2 ? DeletionMode::kEager : DeletionMode::kLazy;
            batch_update(pma, batch, cfg);
            for (auto& [k, v] : resolved) {
                if (v) oracle[k] = *v;
                else oracle.erase(k);
            }
            const auto entries = pma.to_entries();
            CHECK(entries.size() == oracle.size());
            std::size_t i = 0;
            for (auto& [k, v] : oracle) {
                if (i < entries.size()) CHECK(entries[i].key == k && entries[i].value == v);
                ++i;
            }
        }
    }
    {  // graph worked example + analytics (test_graph.cpp:51-58, test_analytics.cpp)
        const std::vector<WeightedEdge> edges = {{0, 0, 1.0}, {0, 2, 2.0}, {1, 2, 3.0},
                                                 {2, 0, 4.0}, {2, 1, 5.0}, {2, 2, 6.0}};
        DynamicGraph g = DynamicGraph::from_edges(3, edges);
        const CsrSnapshot snap = g.csr_snapshot();
        CHECK((snap.row_offsets == std::vector<std::size_t>{0, 2, 3, 6}));
        CHECK((snap.col_indices == std::vector<VertexId>{0, 2, 2, 0, 1, 2}));
        CHECK((snap.values == std::vector<double>{1, 2, 3, 4, 5, 6}));
        CHECK((bfs(g, 0) == std::vector<std::uint32_t>{0, 2, 1}));
        CHECK((connected_components(g) == std::vector<std::uint32_t>{0, 0, 0}));
        CHECK((spmv(g, {1.0, 1.0, 1.0}) == std::vector<double>{3, 3, 15}));
        std::vector<VertexId> dsts;
        g.for_each_neighbor(2, [&](VertexId v, double) { dsts.push_back(v); });
        CHECK((dsts == std::vector<VertexId>{0, 1, 2}));
        const CsrView view(snap);
        CHECK((bfs(view, 0) == bfs(g, 0)));
        // window-style batch keeps set semantics (test_graph.cpp:116-131)
        const std::vector<WeightedEdge> ins = {{1, 0, 7.0}, {0, 1, 8.0}};
        const std::vector<std::pair<VertexId, VertexId>> del = {{2, 1}, {0, 0}};
        g.apply_batch(ins, del);
        CHECK(g.num_edges() == 6 && g.edge_weight(1, 0) == std::optional<double>(7.0) && !g.edge_weight(2, 1));
        const UpdateStats miss = g.apply_batch({}, std::vector<std::pair<VertexId, VertexId>>{{1, 1}});
        CHECK(miss.deletes_missed == 1);
    }
    {  // pagerank known answers (test_analytics.cpp:74-88)
        DynamicGraph one = DynamicGraph::from_edges(1, {});
        const PageRankResult r = pagerank(one);
        CHECK(r.converged && r.ranks == std::vector<double>{1.0});
        const std::vector<WeightedEdge> pair = {{0, 1, 1.0}, {1, 0, 1.0}};
        DynamicGraph two = DynamicGraph::from_edges(2, pair);
        const PageRankResult r2 = pagerank(two);
        CHECK(r2.converged && std::abs(r2.ranks[0] - 0.5) < 1e-12 && std::abs(r2.ranks[1] - 0.5) < 1e-12);
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
    return failures;
}
