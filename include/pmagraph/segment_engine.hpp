#pragma once
// Drop-in <pmagraph/segment_engine.hpp>: GPMA+ batch_update
// (reference segment_engine.hpp:24-60, 365-470) on the device.
#include <chrono>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <vector>

#include "pma.hpp"
#include "primitives.hpp"
#include "update_stats.hpp"
#include "worker_pool.hpp"

namespace pmagraph {

enum class UpdateOp : std::uint8_t { kInsert, kDelete };
struct Update {
    std::uint64_t key = 0;
    std::uint64_t value = 0;
    UpdateOp op = UpdateOp::kInsert;
};
enum class DeletionMode { kLazy, kEager };
enum class MergeStrategy { kSmall, kMedium, kLarge };
struct MergeTiers {
    std::size_t small_max = 32;
    std::size_t medium_max = 1024;
};
inline MergeStrategy select_merge_strategy(std::size_t seg_size, const MergeTiers& tiers = {}) {
    if (seg_size <= tiers.small_max) return MergeStrategy::kSmall;
    if (seg_size <= tiers.medium_max) return MergeStrategy::kMedium;
    return MergeStrategy::kLarge;
}
struct SegmentEngineConfig {
    DeletionMode deletion_mode = DeletionMode::kLazy;
    unsigned workers = 1;
    MergeTiers tiers{};
    std::optional<MergeStrategy> force_strategy;

    pma_engine_config c() const {
        return pma_engine_config{deletion_mode == DeletionMode::kEager ? PMA_EAGER : PMA_LAZY, workers,
                                 tiers.small_max, tiers.medium_max,
                                 force_strategy ? static_cast<int>(*force_strategy) : PMA_STRATEGY_AUTO, 0};
    }
};

// ---- the engine's building blocks (segment_engine.hpp:62-363) -------------
// The device engine runs these steps as kernels over the whole batch; the
// host forms below keep the reference's public helper API.

struct PendingUpdates {
    std::vector<Update> entries;
    std::vector<std::size_t> segments;
    int round_level = 0;
};

struct SegmentGroup {
    std::vector<std::size_t> unique_segments;
    std::vector<std::size_t> offsets;  // first update index per unique segment
    std::vector<std::size_t> counts;
};

// unique_segments (segment_engine.hpp:78-86): RLE of sorted segment ids +
// exclusive scan of the run lengths.
inline SegmentGroup unique_segments(std::span<const std::size_t> segs) {
    const RleResult rle = run_length_encode(std::vector<std::uint64_t>(segs.begin(), segs.end()));
    SegmentGroup group;
    group.unique_segments.assign(rle.unique_values.begin(), rle.unique_values.end());
    group.counts = rle.run_lengths;
    group.offsets = exclusive_scan(rle.run_lengths);
    return group;
}

// advance_round (segment_engine.hpp:90-105): drop committed groups, lift the
// survivors' segment ids to their parents.
inline void advance_round(PendingUpdates& pending, const SegmentGroup& group, std::span<const char> committed) {
    std::size_t w = 0;
    for (std::size_t g = 0; g < group.unique_segments.size(); ++g) {
        if (committed[g]) continue;
        for (std::size_t i = 0; i < group.counts[g]; ++i) {
            const std::size_t r = group.offsets[g] + i;
            pending.entries[w] = pending.entries[r];
            pending.segments[w] = pending.segments[r] >> 1;
            ++w;
        }
    }
    pending.entries.resize(w);
    pending.segments.resize(w);
    ++pending.round_level;
}

// resolve_duplicates (segment_engine.hpp:346-363) on a sorted batch: any
// insert makes the key present with the last insert's value.
inline void resolve_duplicates(std::vector<Update>& sorted) {
    std::size_t w = 0;
    for (std::size_t i = 0; i < sorted.size();) {
        std::size_t j = i;
        Update eff{sorted[i].key, 0, UpdateOp::kDelete};
        for (; j < sorted.size() && sorted[j].key == sorted[i].key; ++j) {
            if (sorted[j].op == UpdateOp::kInsert) {
                eff.value = sorted[j].value;
                eff.op = UpdateOp::kInsert;
            }
        }
        sorted[w++] = eff;
        i = j;
    }
    sorted.resize(w);
}

namespace detail {
struct GroupResult {
    bool committed = false;
    bool moved_slots = false;
    std::uint32_t deletes_missed = 0;
    std::uint32_t tombstones_added = 0;
};
}  // namespace detail

enum class TryOutcome : std::uint8_t { kCommitted, kDeferred };

// try_insert_plus (segment_engine.hpp:320-341): one group decided and, when
// the density bounds allow, committed — on the device (pma_try_insert_plus).
inline TryOutcome try_insert_plus(PackedMemoryArray& pma, int level, std::size_t seg, std::span<const Update> slice,
                                  const SegmentEngineConfig& cfg, detail::GroupResult& result) {
    std::vector<std::uint64_t> k(slice.size()), v(slice.size());
    std::vector<std::uint8_t> o(slice.size());
    for (std::size_t i = 0; i < slice.size(); ++i) {
        k[i] = slice[i].key;
        v[i] = slice[i].value;
        o[i] = slice[i].op == UpdateOp::kInsert ? 0 : 1;
    }
    const pma_engine_config c = cfg.c();
    int outcome = 0;
    std::uint64_t missed = 0, tombs = 0;
    pma.invalidate();
    pma.check(pma_try_insert_plus(pma.handle(), level, seg, k.data(), v.data(), o.data(), k.size(), &c, &outcome,
                                  &missed, &tombs));
    if (outcome == 0) return TryOutcome::kDeferred;
    result = detail::GroupResult{true, outcome == 2, static_cast<std::uint32_t>(missed),
                                 static_cast<std::uint32_t>(tombs)};
    return TryOutcome::kCommitted;
}

inline UpdateStats batch_update(PackedMemoryArray& pma, std::vector<Update> updates,
                                const SegmentEngineConfig& cfg = {}, WorkerPool* pool = nullptr) {
    (void)pool;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::uint64_t> k(updates.size()), v(updates.size());
    std::vector<std::uint8_t> o(updates.size());
    for (std::size_t i = 0; i < updates.size(); ++i) {
        k[i] = updates[i].key;
        v[i] = updates[i].value;
        o[i] = updates[i].op == UpdateOp::kInsert ? 0 : 1;
    }
    const pma_engine_config c = cfg.c();
    pma_stats st{};
    pma.invalidate();
    pma.check(pma_batch_update(pma.handle(), k.data(), v.data(), o.data(), k.size(), &c, &st));
    UpdateStats u = UpdateStats::from_c(st, pma.handle());
    u.wall_ns = static_cast<std::uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
    return u;
}

}  // namespace pmagraph
