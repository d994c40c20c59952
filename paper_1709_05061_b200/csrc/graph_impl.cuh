// graph_impl.cuh — DynamicGraph (graph.hpp:62-240) over the device PMA.
#pragma once

#include "pma_impl.cuh"

namespace gpma {

class Graph {
public:
    Graph(const gpma_graph_config* cfg, int device, u64 nv);
    ~Graph();
    Pma pma;
    u64 nv;
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
    double pr_iter_ms_ = 0.0;
    std::string err;

public:  // (extended __device__ lambdas need public enclosing functions)
    Ctr* scratch_ctr();
    cudaEvent_t pma_ev(int i);
    void record_timing(u64 launches);
    Ctr* d_ctr_ = nullptr;
    DevBuf<u64> bk, bv;
    DevBuf<u8> bo;
    DevBuf<u32> dist, q0, q1, qn, outdeg;
    DevBuf<double> px, py, pshare, psc;
    u32 h_nf_store_ = 0;
    u32* h_nf_ = &h_nf_store_;
    cudaEvent_t evs_[4]{};
};

}  // namespace gpma
