#pragma once
// Drop-in <pmagraph/worker_pool.hpp> (reference worker_pool.hpp:17-94).  The
// CUDA grid replaces the bulk-synchronous thread pool; results are
// worker-count independent by contract (pma.hpp:9-12), so the pool is a
// placeholder that keeps signatures source-compatible.
namespace pmagraph {
class WorkerPool {
public:
    explicit WorkerPool(unsigned workers) : workers_(workers == 0 ? 1 : workers) {}
    unsigned workers() const { return workers_; }

private:
    unsigned workers_;
};
}  // namespace pmagraph
