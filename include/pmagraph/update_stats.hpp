#pragma once
// Drop-in <pmagraph/update_stats.hpp> (reference update_stats.hpp:13-35).
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../pmagraph_cuda.h"

namespace pmagraph {

struct UpdateStats {
    std::size_t batch_size = 0;
    std::size_t rounds = 0;
    std::uint64_t slot_writes = 0;
    std::uint64_t wall_ns = 0;
    std::uint64_t segment_phase_ns = 0;
    std::vector<std::size_t> segments_per_level;
    std::size_t grow_events = 0;
    std::size_t shrink_events = 0;
    std::size_t deletes_missed = 0;
    std::size_t tombstones_added = 0;
    std::vector<std::pair<std::size_t, std::size_t>> touched_ranges;
    bool resized = false;

    static std::string csv_header() { return "batch_size,rounds,slot_writes,wall_ns"; }
    std::string csv_row() const {
        return std::to_string(batch_size) + "," + std::to_string(rounds) + "," + std::to_string(slot_writes) + "," +
               std::to_string(wall_ns);
    }

    static UpdateStats from_c(const pma_stats& s, pma_handle* h) {
        UpdateStats u;
        u.batch_size = s.batch_size;
        u.rounds = s.rounds;
        u.slot_writes = s.slot_writes;
        u.wall_ns = s.wall_ns;
        u.segment_phase_ns = s.segment_phase_ns;
        u.segments_per_level.assign(s.segments_per_level, s.segments_per_level + s.num_levels);
        u.grow_events = s.grow_events;
        u.shrink_events = s.shrink_events;
        u.deletes_missed = s.deletes_missed;
        u.tombstones_added = s.tombstones_added;
        u.resized = s.resized != 0;
        if (h && s.num_touched_ranges) {
            std::vector<std::uint64_t> pairs(2 * s.num_touched_ranges);
            std::size_t n = 0;
            pma_touched_ranges(h, pairs.data(), s.num_touched_ranges, &n);
            for (std::size_t i = 0; i < n; ++i) u.touched_ranges.emplace_back(pairs[2 * i], pairs[2 * i + 1]);
        }
        return u;
    }
};

}  // namespace pmagraph
