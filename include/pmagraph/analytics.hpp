#pragma once
// Drop-in <pmagraph/analytics.hpp> (reference analytics.hpp:17-158): BFS,
// connected components, PageRank and SpMV run on the GPU over the gapped
// PMA.  A CsrView (compact snapshot) is analysed by loading it as a
// gap-free device graph (same edge set, same results).
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

#include "graph.hpp"

namespace pmagraph {

inline constexpr std::uint32_t kUnreached = std::numeric_limits<std::uint32_t>::max();

struct PageRankResult {
    std::vector<double> ranks;
    std::size_t iterations = 0;
    bool converged = false;
};

struct PageRankOptions {
    double damping = 0.85;
    double epsilon = 1e-3;
    std::size_t max_iters = 200;
    const std::vector<double>* warm_start = nullptr;
};

inline std::vector<std::uint32_t> bfs(const DynamicGraph& g, std::uint32_t root) {
    std::vector<std::uint32_t> dist(g.num_vertices());
    g.check(gpma_bfs(g.handle(), root, dist.data(), nullptr));
    return dist;
}

inline std::vector<std::uint32_t> connected_components(const DynamicGraph& g) {
    std::vector<std::uint32_t> lab(g.num_vertices());
    g.check(gpma_cc(g.handle(), lab.data()));
    return lab;
}

inline PageRankResult pagerank(const DynamicGraph& g, PageRankOptions opts = {}) {
    const std::size_t n = g.num_vertices();
    if (n == 0) throw std::invalid_argument("pagerank: empty vertex set");
    if (opts.warm_start && opts.warm_start->size() != n)
        throw std::invalid_argument("pagerank: warm start size mismatch");
    PageRankResult r;
    r.ranks.resize(n);
    std::uint64_t it = 0;
    int conv = 0;
    g.check(gpma_pagerank(g.handle(), opts.damping, opts.epsilon, opts.max_iters,
                          opts.warm_start ? opts.warm_start->data() : nullptr, r.ranks.data(), &it, &conv));
    r.iterations = it;
    r.converged = conv != 0;
    return r;
}

inline std::vector<double> spmv(const DynamicGraph& g, const std::vector<double>& x) {
    if (x.size() != g.num_vertices()) throw std::invalid_argument("spmv: dimension mismatch");
    std::vector<double> y(x.size());
    g.check(gpma_spmv(g.handle(), x.data(), y.data()));
    return y;
}

namespace detail_cuda {
inline DynamicGraph device_graph(const CsrView& v) {
    std::vector<WeightedEdge> edges;
    const auto& s = v.snapshot();
    for (std::size_t u = 0; u + 1 < s.row_offsets.size(); ++u)
        for (std::size_t i = s.row_offsets[u]; i < s.row_offsets[u + 1]; ++i)
            edges.push_back(WeightedEdge{static_cast<VertexId>(u), s.col_indices[i], s.values[i]});
    return DynamicGraph::from_edges(v.num_vertices(), edges);
}
}  // namespace detail_cuda

inline std::vector<std::uint32_t> bfs(const CsrView& v, std::uint32_t root) { return bfs(detail_cuda::device_graph(v), root); }
inline std::vector<std::uint32_t> connected_components(const CsrView& v) {
    return connected_components(detail_cuda::device_graph(v));
}
inline PageRankResult pagerank(const CsrView& v, PageRankOptions opts = {}) {
    return pagerank(detail_cuda::device_graph(v), opts);
}
inline std::vector<double> spmv(const CsrView& v, const std::vector<double>& x) {
    return spmv(detail_cuda::device_graph(v), x);
}

}  // namespace pmagraph
