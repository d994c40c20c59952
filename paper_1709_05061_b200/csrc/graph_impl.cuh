// graph_impl.cuh — DynamicGraph (graph.hpp:62-240) over the device PMA.
#pragma once

#include "pma_impl.cuh"

namespace gpma {

class Graph {
public:
    Graph(const gpma_graph_config* cfg, int device, u64 nv, u64 lo = 0, u64 hi = ~0ull);
    ~Graph();
    Pma pma;
    u64 nv;      // global vertex count (ids)
    u64 lo, hi;  // owned source range: a shard of a key-range sharded graph, or [0, nv)
    u64 nloc() const { return hi - lo; }
    bool is_shard() const { return lo != 0 || hi != nv; }
    EngineCfg ecfg;
    double fill_target = 0.5;
    DevBuf<u64> ro;  // row offsets, |V| + 1 (graph.hpp:97)

    void from_edges_device(const u32* d_src, const u32* d_dst, const double* d_w, u64 n);
    void apply_batch_device(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                            u64 nd, pma_stats* out);
    void row_offsets(u64* out);
    u64 num_edges() const;
    void csr_snapshot(u64* ro, u32* col, double* val);

    void bfs(u32 root, u32* dist, u64* reached);
    void cc(u32* labels);
    void pagerank(double d, double eps, u64 max_iters, const double* warm, double* ranks, u64* iters, int* converged);
    void spmv(const double* x, double* y);

    // key-range sharding (shard.cu): routing partition and the device steps of
    // the sharded analytics (collectives run in the caller between them)
    void reserve_batch(u64 n);  // every per-batch buffer of apply_batch for n updates
    void route_partition(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                         u64 nd, const u32* d_bounds, int world, u64* okeys, double* ow, u64* h_counts,
                         u64* d_counts = nullptr);
    void route_scatter_peer(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd,
                            u64 nd, const u32* d_bounds, int world, u64* const* dst_keys, double* const* dst_w,
                            const u64* dst_off);
    u64 rt_ntiles = 0;
    // apply_batch with routed EdgeKeys, bit 63 = delete (arrival order kept among inserts)
    void apply_batch_mixed_device(const u64* keys, const double* w, u64 n, pma_stats* out);
    void apply_batch_impl(const u32* is, const u32* id, const u64* mk, const double* iw, u64 ni, const u32* ds,
                          const u32* dd, u64 nd, pma_stats* out);
    void shard_bfs_mark(const u32* frontier, u32 nf, u8* flags);
    void shard_bfs_update(const u8* flags, u32* dist_local, u32 depth, u32* next, u32* nf_out);
    void shard_cc_hook(u32* labels);
    void cc_jump(u32* labels, u64 n, const u32* prev, int* changed);
    void shard_outdeg(u32* outdeg);
    void shard_pr_push(const double* x, const u32* outdeg, double d, double* y);
    void pr_finish(const double* x, double* y, u64 n, const u32* outdeg, double d, double* l1);
    void shard_spmv(const double* x, double* y_local);
    double pr_iter_ms_ = 0.0;
    std::string err;

public:  // (extended __device__ lambdas need public enclosing functions)
    Ctr* scratch_ctr();
    cudaEvent_t pma_ev(int i);
    void record_timing(u64 launches);
    Ctr* d_ctr_ = nullptr;
    DevBuf<u64> bk, bv;
    DevBuf<u8> bo;
    DevBuf<u32> dist, bvis, q0, q1, h0, h1, g0, g1, qn, outdeg;
    DevBuf<double> px, py, pshare, psc, pl1;
    DevBuf<u32> pdone;
    DevBuf<u32> rt_counts, hot_table, hot_ids, hot_hist;
    u32 nhot_ = 0;
    bool hot_ready_ = false;
    void prepare_hot(const u32* outdeg, u64 n);
    DevBuf<u64> rt_offsets, rt_totals;
    u32 h_nf_store_[2] = {0, 0};
    std::vector<u32> h_lv_;  // per-level frontier counts of one BFS window
    u32* h_nf_ = h_nf_store_;
    cudaEvent_t evs_[4]{};
};

}  // namespace gpma
