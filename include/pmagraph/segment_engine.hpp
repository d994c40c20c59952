#pragma once
// Drop-in <pmagraph/segment_engine.hpp>: GPMA+ batch_update
// (reference segment_engine.hpp:24-60, 365-470) on the device.
#include <chrono>
#include <cstdint>
#include <optional>
#include <vector>

#include "pma.hpp"
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
