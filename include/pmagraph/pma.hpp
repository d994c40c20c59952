#pragma once
// Drop-in replacement for the reference's <pmagraph/pma.hpp>
// (/root/reference/proj/include/pmagraph/pma.hpp:29-612): the same class and
// function names over the device-resident B200 implementation
// (libpmagraph_cuda.so, include/pmagraph_cuda.h).  Link with
// -lpmagraph_cuda.  Every operation runs on the GPU; slots() downloads a host
// mirror that is invalidated by any mutation.

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../pmagraph_cuda.h"

namespace pmagraph {

namespace detail_cuda {
[[noreturn]] inline void raise(int code, const char* msg) {
    switch (code) {
        case PMA_EINVAL: throw std::invalid_argument(msg);
        case PMA_ERANGE: throw std::out_of_range(msg);
        case PMA_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
inline int& default_device() {
    static int dev = 0;
    return dev;
}
}  // namespace detail_cuda

inline void set_device(int device) { detail_cuda::default_device() = device; }

enum class SlotState : std::uint8_t { kEmpty = 0, kValid = 1, kTombstone = 2 };  // pma.hpp:29

struct Slot {  // pma.hpp:34-40
    std::uint64_t key = 0;
    std::uint64_t value = 0;
    SlotState state = SlotState::kEmpty;
    friend bool operator==(const Slot&, const Slot&) = default;
};

struct Entry {  // pma.hpp:42-47
    std::uint64_t key = 0;
    std::uint64_t value = 0;
    friend bool operator==(const Entry&, const Entry&) = default;
};

struct DensityProfile {  // pma.hpp:52-78
    double leaf_lower = 0.08;
    double leaf_upper = 0.92;
    double root_lower = 0.40;
    double root_upper = 0.80;
    bool allow_shrink = true;

    double lower_at(int level, int height) const {
        if (height == 0) return root_lower;
        return leaf_lower + (root_lower - leaf_lower) * static_cast<double>(level) / height;
    }
    double upper_at(int level, int height) const {
        if (height == 0) return root_upper;
        return leaf_upper + (root_upper - leaf_upper) * static_cast<double>(level) / height;
    }
    pma_profile c() const { return pma_profile{leaf_lower, leaf_upper, root_lower, root_upper, allow_shrink ? 1 : 0, 0}; }
};

class PmaLayout {  // pma.hpp:82-123
public:
    PmaLayout() : PmaLayout(16) {}
    explicit PmaLayout(std::size_t capacity) : capacity_(capacity), leaf_size_(leaf_size_for(capacity)) {
        height_ = 0;
        for (std::size_t s = leaf_size_; s < capacity_; s <<= 1) ++height_;
    }
    static std::size_t leaf_size_for(std::size_t capacity) {
        int log2cap = 0;
        while ((std::size_t{1} << (log2cap + 1)) <= capacity) ++log2cap;
        std::size_t leaf = 4;
        while (leaf * 2 <= static_cast<std::size_t>(log2cap)) leaf *= 2;
        return leaf;
    }
    std::size_t capacity() const { return capacity_; }
    std::size_t leaf_size() const { return leaf_size_; }
    int height() const { return height_; }
    std::size_t seg_size(int level) const { return leaf_size_ << level; }
    std::size_t num_segments(int level) const { return capacity_ / seg_size(level); }
    std::size_t seg_begin(int level, std::size_t index) const { return index * seg_size(level); }
    std::size_t num_leaves() const { return capacity_ / leaf_size_; }
    std::size_t leaf_of_slot(std::size_t slot) const { return slot / leaf_size_; }

private:
    std::size_t capacity_ = 16;
    std::size_t leaf_size_ = 4;
    int height_ = 2;
};

class PackedMemoryArray {
public:
    static constexpr std::size_t kMinCapacity = 16;

    explicit PackedMemoryArray(DensityProfile profile = {}) : profile_(profile) {
        const pma_profile p = profile_.c();
        pma_handle* h = nullptr;
        if (int rc = pma_create(&p, detail_cuda::default_device(), &h)) detail_cuda::raise(rc, pma_last_error(nullptr));
        h_ = h;
        owned_ = true;
    }
    // Non-owning view of a graph's array (DynamicGraph::pma()).
    PackedMemoryArray(pma_handle* view, DensityProfile profile) : h_(view), owned_(false), profile_(profile) {}
    ~PackedMemoryArray() {
        if (owned_ && h_) pma_destroy(h_);
    }
    PackedMemoryArray(PackedMemoryArray&& o) noexcept
        : h_(o.h_), owned_(o.owned_), profile_(o.profile_), mirror_(std::move(o.mirror_)), mirror_ok_(o.mirror_ok_) {
        o.h_ = nullptr;
        o.owned_ = false;
    }
    PackedMemoryArray& operator=(PackedMemoryArray&& o) noexcept {
        if (this != &o) {
            if (owned_ && h_) pma_destroy(h_);
            h_ = o.h_;
            owned_ = o.owned_;
            profile_ = o.profile_;
            mirror_ = std::move(o.mirror_);
            mirror_ok_ = o.mirror_ok_;
            o.h_ = nullptr;
            o.owned_ = false;
        }
        return *this;
    }
    // Deep copy through a slot download + restore (the reference copies the array).
    PackedMemoryArray(const PackedMemoryArray& o) : PackedMemoryArray(o.profile_) { copy_from(o); }
    PackedMemoryArray& operator=(const PackedMemoryArray& o) {
        if (this != &o) {
            PackedMemoryArray tmp(o);
            *this = std::move(tmp);
        }
        return *this;
    }

    static PackedMemoryArray from_sorted(std::span<const Entry> sorted, double fill_target, DensityProfile profile = {}) {
        PackedMemoryArray p(profile);
        std::vector<std::uint64_t> k(sorted.size()), v(sorted.size());
        for (std::size_t i = 0; i < sorted.size(); ++i) {
            k[i] = sorted[i].key;
            v[i] = sorted[i].value;
        }
        p.check(pma_from_sorted(p.h_, k.data(), v.data(), k.size(), fill_target));
        return p;
    }

    static PackedMemoryArray from_slot_layout(
        std::size_t capacity, std::span<const std::tuple<std::size_t, std::uint64_t, std::uint64_t>> placements,
        DensityProfile profile = {}) {
        PackedMemoryArray p(profile);
        std::vector<std::uint64_t> k(capacity, 0), v(capacity, 0);
        std::vector<std::uint8_t> s(capacity, 0);
        std::uint64_t last = 0;
        bool first = true;
        for (const auto& [slot, key, value] : placements) {
            if (slot >= capacity) throw std::invalid_argument("from_slot_layout: slot out of range");
            if (!first && key <= last) throw std::invalid_argument("from_slot_layout: keys must increase in slot order");
            first = false;
            last = key;
            k[slot] = key;
            v[slot] = value;
            s[slot] = 1;
        }
        p.check(pma_load_slots(p.h_, capacity, k.data(), v.data(), s.data()));
        return p;
    }

    PmaLayout layout() const { return PmaLayout(info().capacity); }
    const DensityProfile& profile() const { return profile_; }
    std::size_t capacity() const { return info().capacity; }
    std::size_t valid_count() const { return info().valid_count; }
    std::size_t tombstone_count() const { return info().tombstone_count; }
    std::uint64_t slot_writes() const { return info().slot_writes; }
    void reset_slot_writes() { pma_reset_slot_writes(h_); }

    const std::vector<Slot>& slots() const {
        if (!mirror_ok_) {
            const std::size_t cap = capacity();
            std::vector<std::uint64_t> k(cap), v(cap);
            std::vector<std::uint8_t> s(cap);
            check(pma_download(h_, k.data(), v.data(), s.data()));
            mirror_.resize(cap);
            for (std::size_t i = 0; i < cap; ++i) mirror_[i] = Slot{k[i], v[i], static_cast<SlotState>(s[i])};
            mirror_ok_ = true;
        }
        return mirror_;
    }

    std::pair<double, double> thresholds(int level) const {
        double rho = 0, tau = 0;
        check(pma_bounds(h_, level, nullptr, nullptr, &rho, &tau));
        return {rho, tau};
    }
    std::size_t min_entries(int level) const {
        std::uint64_t mn = 0;
        check(pma_bounds(h_, level, &mn, nullptr, nullptr, nullptr));
        return mn;
    }
    std::size_t max_entries(int level) const {
        std::uint64_t mx = 0;
        check(pma_bounds(h_, level, nullptr, &mx, nullptr, nullptr));
        return mx;
    }
    std::size_t binary_search_leaf(std::uint64_t key) const {
        std::uint64_t leaf = 0;
        check(pma_binary_search_leaf(h_, &key, 1, &leaf));
        return leaf;
    }
    void assign_leaves_sorted(std::span<const std::uint64_t> keys, std::span<std::size_t> out) const {
        std::vector<std::uint64_t> o(keys.size());
        check(pma_binary_search_leaf(h_, keys.data(), keys.size(), o.data()));
        for (std::size_t i = 0; i < o.size(); ++i) out[i] = o[i];
    }
    std::optional<std::uint64_t> search(std::uint64_t key) const {
        std::uint64_t v = 0;
        std::uint8_t f = 0;
        check(pma_search(h_, &key, 1, &v, &f));
        if (!f) return std::nullopt;
        return v;
    }
    std::optional<std::size_t> find_slot(std::uint64_t key) const {
        const auto& s = slots();
        const std::size_t leaf = binary_search_leaf(key);
        const std::size_t ls = layout().leaf_size();
        for (std::size_t i = leaf * ls; i < (leaf + 1) * ls; ++i)
            if (s[i].state != SlotState::kEmpty && s[i].key == key) return i;
        return std::nullopt;
    }
    void insert(std::uint64_t key, std::uint64_t value) {
        mirror_ok_ = false;
        check(pma_insert(h_, key, value));
    }
    bool erase(std::uint64_t key) {
        mirror_ok_ = false;
        int r = 0;
        check(pma_erase(h_, key, &r));
        return r != 0;
    }
    bool mark_tombstone(std::uint64_t key) {
        mirror_ok_ = false;
        int r = 0;
        check(pma_mark_tombstone(h_, key, &r));
        return r != 0;
    }
    void redispatch(int level, std::size_t seg_index, std::span<const Entry> extra) {
        mirror_ok_ = false;
        std::vector<std::uint64_t> k(extra.size()), v(extra.size());
        for (std::size_t i = 0; i < extra.size(); ++i) {
            k[i] = extra[i].key;
            v[i] = extra[i].value;
        }
        check(pma_redispatch(h_, level, seg_index, k.data(), v.data(), k.size()));
    }
    std::pair<std::size_t, std::size_t> seg_range(int level, std::size_t seg_index) const {
        const PmaLayout l = layout();
        const std::size_t b = l.seg_begin(level, seg_index);
        return {b, b + l.seg_size(level)};
    }
    std::size_t count_valid_in(std::size_t begin, std::size_t end) const {
        std::uint64_t c = 0;
        check(pma_count_valid_in(h_, begin, end, &c));
        return c;
    }
    template <typename Fn>
    void for_each_valid(Fn&& fn) const {
        for (const Slot& s : slots())
            if (s.state == SlotState::kValid) fn(s.key, s.value);
    }
    std::vector<Entry> to_entries() const {
        std::vector<Entry> out;
        for_each_valid([&](std::uint64_t k, std::uint64_t v) { out.push_back(Entry{k, v}); });
        return out;
    }

    pma_handle* handle() const { return h_; }
    void invalidate() const { mirror_ok_ = false; }
    void check(int rc) const {
        if (rc) detail_cuda::raise(rc, pma_last_error(h_));
    }

private:
    pma_layout_info info() const {
        pma_layout_info li{};
        pma_get_layout(h_, &li);
        return li;
    }
    void copy_from(const PackedMemoryArray& o) {
        const std::size_t cap = o.capacity();
        std::vector<std::uint64_t> k(cap), v(cap);
        std::vector<std::uint8_t> s(cap);
        o.check(pma_download(o.h_, k.data(), v.data(), s.data()));
        check(pma_load_slots(h_, cap, k.data(), v.data(), s.data()));
    }

    pma_handle* h_ = nullptr;
    bool owned_ = false;
    DensityProfile profile_{};
    mutable std::vector<Slot> mirror_;
    mutable bool mirror_ok_ = false;
};

}  // namespace pmagraph
