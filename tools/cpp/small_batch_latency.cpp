// Library-only latency of small sliding-window batches through the C ABI
// (no Python): C2's stream and window, slides of B arrivals applied with
// gpma_apply_batch_device, host steady_clock around each call.
//   tools/cpp/small_batch_latency [B ...]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pmagraph_cuda.h"
#include "pmagraph_stream.h"

int main(int argc, char** argv) {
    std::vector<size_t> bs;
    for (int i = 1; i < argc; ++i) bs.push_back(size_t(std::atoll(argv[i])));
    if (bs.empty()) bs = {100, 1000, 10000};
    gpma_warmup(0);
    gpma_stream* st = nullptr;
    if (gpma_stream_rmat(1u << 21, 30600000, 0.57, 0.19, 0.19, 0.05, 1, &st) || gpma_stream_shuffle(st, 2)) {
        std::fprintf(stderr, "stream: %s\n", gpma_stream_last_error());
        return 1;
    }
    for (size_t B : bs) {
        gpma_window* w = nullptr;
        gpma_window_create(st, 0, &w);
        const int n = 200;
        gpma_window_reserve(w, size_t(n + 8) * B + 16);
        gpma_window_info_t info{};
        gpma_window_info(w, &info);
        gpma_graph* g = nullptr;
        if (gpma_from_edges_device(nullptr, 0, 1u << 21, info.stream_src, info.stream_dst, nullptr,
                                   info.initial_size, &g)) {
            std::fprintf(stderr, "graph: %s\n", gpma_last_error(nullptr));
            return 1;
        }
        gpma_reserve_batch(g, 2 * B + 16);
        std::vector<gpma_slide_t> sl(n + 8);
        for (auto& s : sl) gpma_window_slide(w, B, &s);
        gpma_window_info(w, &info);
        std::vector<double> us;
        pma_stats ps;
        for (size_t i = 0; i < sl.size(); ++i) {
            const auto& s = sl[i];
            const auto t0 = std::chrono::steady_clock::now();
            const int rc = gpma_apply_batch_device(g, info.stream_src + s.ins_offset, info.stream_dst + s.ins_offset,
                                                   nullptr, s.n_ins, info.del_src + s.del_offset,
                                                   info.del_dst + s.del_offset, s.n_del, &ps);
            const auto t1 = std::chrono::steady_clock::now();
            if (rc) {
                std::fprintf(stderr, "apply: %s\n", gpma_last_error(g));
                return 1;
            }
            if (i >= 8) us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        std::sort(us.begin(), us.end());
        pma_timing tm{};
        gpma_last_timing(g, &tm);
        std::printf("B=%zu: C ABI wall per batch median %.1f us, p10 %.1f, p90 %.1f (device %.1f us, %llu updates)\n", B,
                    us[us.size() / 2], us[us.size() / 10], us[us.size() * 9 / 10], tm.device_ms * 1e3,
                    (unsigned long long)ps.batch_size);
        std::printf("  last call: sort %.1f us, search %.1f, rounds %.1f, refresh %.1f\n", tm.sort_ms * 1e3,
                    tm.search_ms * 1e3, tm.rounds_ms * 1e3, tm.refresh_ms * 1e3);
        gpma_destroy(g);
        gpma_window_destroy(w);
    }
    gpma_stream_destroy(st);
    return 0;
}
