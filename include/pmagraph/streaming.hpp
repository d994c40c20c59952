#pragma once
// Drop-in <pmagraph/streaming.hpp> (reference streaming.hpp:1-193): the
// sliding window runs on the device (pmagraph_stream.h: FIFO slides by the
// next-occurrence trick, explicit random eviction with the caller's
// mt19937_64 draws, multiplicity-filtered deletions); the host EdgeStream
// keeps the weights and timestamps, so SlideBatch carries exactly the
// reference's inserts, deletions and expiries.
#include <cstdint>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../pmagraph_stream.h"
#include "graph.hpp"

namespace pmagraph {

struct TimestampedEdge {
    VertexId src = 0;
    VertexId dst = 0;
    double weight = 1.0;
    std::uint64_t ts = 0;
};

struct EdgeStream {
    std::size_t num_vertices = 0;
    std::vector<TimestampedEdge> edges;  // non-decreasing ts

    void validate() const {
        for (std::size_t i = 1; i < edges.size(); ++i)
            if (edges[i].ts < edges[i - 1].ts)
                throw std::invalid_argument("EdgeStream: timestamps must be non-decreasing");
    }
};

// Portable bounded draw (streaming.hpp:43-50): mt19937_64 is fully
// specified, its distributions are not.
inline std::uint64_t draw_below(std::mt19937_64& rng, std::uint64_t bound) {
    const std::uint64_t limit = bound * (UINT64_MAX / bound);
    std::uint64_t x;
    do {
        x = rng();
    } while (x >= limit);
    return x % bound;
}

inline double draw_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// assign_random_timestamps (streaming.hpp:58-67): the same seeded
// Fisher-Yates draws as the device stream's gpma_stream_shuffle.
inline EdgeStream assign_random_timestamps(std::vector<TimestampedEdge> edges, std::size_t num_vertices,
                                           std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    for (std::size_t i = edges.size(); i > 1; --i) {
        const std::size_t j = static_cast<std::size_t>(draw_below(rng, i));
        std::swap(edges[i - 1], edges[j]);
    }
    for (std::size_t i = 0; i < edges.size(); ++i) edges[i].ts = i;
    return EdgeStream{num_vertices, std::move(edges)};
}

struct SlideBatch {
    std::vector<WeightedEdge> inserts;
    std::vector<std::pair<VertexId, VertexId>> deletions;  // multiplicity-filtered
    std::vector<TimestampedEdge> expiries;                 // raw edges leaving the window
    bool final_partial = false;
};

class SlidingWindow {
public:
    explicit SlidingWindow(const EdgeStream& stream, int device = 0) : stream_(&stream) {
        if (stream.edges.size() < 2) throw std::invalid_argument("SlidingWindow: stream needs at least two edges");
        stream.validate();
        std::vector<std::uint32_t> s(stream.edges.size()), d(stream.edges.size());
        for (std::size_t i = 0; i < s.size(); ++i) {
            s[i] = stream.edges[i].src;
            d[i] = stream.edges[i].dst;
        }
        gpma_stream* gs = nullptr;
        check(gpma_stream_from_arrays(stream.num_vertices, s.data(), d.data(), s.size(), &gs));
        s_.reset(gs);
        gpma_window* gw = nullptr;
        check(gpma_window_create(gs, device, &gw));
        w_.reset(gw);
    }

    // Window of the first half of the stream, graph built from its edge set
    // (streaming.hpp:89-99).
    static std::pair<SlidingWindow, DynamicGraph> init_window(const EdgeStream& stream, GraphConfig config = {}) {
        SlidingWindow window(stream);
        const std::size_t half = (stream.edges.size() + 1) / 2;
        std::vector<WeightedEdge> edges;
        edges.reserve(half);
        for (std::size_t i = 0; i < half; ++i)
            edges.push_back(WeightedEdge{stream.edges[i].src, stream.edges[i].dst, stream.edges[i].weight});
        DynamicGraph graph = DynamicGraph::from_edges(stream.num_vertices, edges, config);
        return {std::move(window), std::move(graph)};
    }

    std::size_t window_size() const { return static_cast<std::size_t>(gpma_window_size(w_.get())); }
    std::size_t remaining() const {
        gpma_window_info_t i{};
        gpma_window_info(w_.get(), &i);
        return static_cast<std::size_t>(i.stream_size - i.cursor);
    }
    bool exhausted() const { return remaining() == 0; }

    // FIFO slide (streaming.hpp:107-123).
    SlideBatch slide(std::size_t batch) {
        gpma_slide_t sl{};
        check(gpma_window_slide(w_.get(), batch, &sl));
        return collect(sl);
    }

    // Explicit random eviction (streaming.hpp:129-158) with the caller's
    // generator: its state goes to the device window's draws and comes back
    // advanced exactly as the reference's would.
    SlideBatch slide_explicit_random(std::size_t batch, std::mt19937_64& rng) {
        gpma_rng* r = nullptr;
        check(gpma_rng_create(0, &r));
        std::unique_ptr<gpma_rng, int (*)(gpma_rng*)> guard(r, &gpma_rng_destroy);
        std::ostringstream os;
        os << rng;
        check(gpma_rng_set_state(r, os.str().c_str()));
        gpma_slide_t sl{};
        check(gpma_window_slide_explicit_random(w_.get(), batch, r, &sl));
        std::size_t len = 0;
        check(gpma_rng_get_state(r, nullptr, 0, &len));
        std::string text(len, '\0');
        check(gpma_rng_get_state(r, text.data(), len, &len));
        std::istringstream is(text);
        is >> rng;
        return collect(sl);
    }

    std::vector<std::pair<VertexId, VertexId>> distinct_edges() const {
        std::size_t n = 0;
        check(gpma_window_distinct_edges(w_.get(), nullptr, nullptr, 0, &n));
        std::vector<std::uint32_t> s(n), d(n);
        check(gpma_window_distinct_edges(w_.get(), s.data(), d.data(), n, &n));
        std::vector<std::pair<VertexId, VertexId>> out(n);
        for (std::size_t i = 0; i < n; ++i) out[i] = {s[i], d[i]};
        return out;
    }

private:
    static void check(int rc) {
        if (rc == PMA_OK) return;
        const std::string m = gpma_stream_last_error();
        if (rc == PMA_EINVAL) throw std::invalid_argument(m);
        if (rc == PMA_ERANGE) throw std::out_of_range(m);
        throw std::runtime_error(m);
    }

    SlideBatch collect(const gpma_slide_t& sl) const {
        SlideBatch out;
        out.final_partial = sl.final_partial != 0;
        out.inserts.reserve(sl.n_ins);
        for (std::uint64_t i = 0; i < sl.n_ins; ++i) {
            const TimestampedEdge& e = stream_->edges[sl.ins_offset + i];
            out.inserts.push_back(WeightedEdge{e.src, e.dst, e.weight});
        }
        std::vector<std::uint32_t> ds(sl.n_del), dd(sl.n_del);
        if (sl.n_del) check(gpma_window_deletions_host(w_.get(), sl.del_offset, sl.n_del, ds.data(), dd.data()));
        out.deletions.resize(sl.n_del);
        for (std::uint64_t i = 0; i < sl.n_del; ++i) out.deletions[i] = {ds[i], dd[i]};
        std::size_t ne = 0;
        check(gpma_window_last_expiries(w_.get(), nullptr, 0, &ne));
        std::vector<std::uint32_t> pos(ne);
        check(gpma_window_last_expiries(w_.get(), pos.data(), ne, &ne));
        out.expiries.reserve(ne);
        for (const std::uint32_t p : pos) out.expiries.push_back(stream_->edges[p]);
        return out;
    }

    struct StreamDel {
        void operator()(gpma_stream* s) const { gpma_stream_destroy(s); }
    };
    struct WindowDel {
        void operator()(gpma_window* w) const { gpma_window_destroy(w); }
    };
    const EdgeStream* stream_;
    std::unique_ptr<gpma_stream, StreamDel> s_;
    std::unique_ptr<gpma_window, WindowDel> w_;
};

}  // namespace pmagraph
