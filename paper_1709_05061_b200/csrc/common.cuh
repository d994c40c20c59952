// common.cuh — shared device/host helpers for libpmagraph_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "pmagraph_cuda.h"

namespace gpma {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = long long;
using ull = unsigned long long;

constexpr u8 kEmpty = 0;
constexpr u8 kValid = 1;
constexpr u8 kTombstone = 2;
constexpr u8 kOpInsert = 0;
constexpr u8 kOpDelete = 1;
constexpr u8 kOpSkip = 2;  // guard deletes dropped by apply_batch (graph.hpp:141-147)
constexpr u64 kGuardDst = 0xFFFFFFFFull;
constexpr int kNumSMs = 148;
constexpr unsigned FULL = 0xffffffffu;

// Error carrying the reference exception class as a PMA_* code.
struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GPMA_CUDA(call)                                                                           \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw ::gpma::ApiError(PMA_ECUDA, std::string(#call " failed: ") + cudaGetErrorString(e_) + \
                                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")");        \
    } while (0)

#define GPMA_LAUNCH_CHECK() GPMA_CUDA(cudaGetLastError())

inline unsigned grid_for(u64 n, unsigned block, unsigned cap = 148u * 16u) {
    u64 g = (n + block - 1) / block;
    if (g == 0) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// CTAs of `kernel` (block threads, dynamic smem) resident on the whole GPU at
// once: the grid of a persistent grid-stride kernel — a partial last wave
// leaves SMs idle while the slowest CTAs finish.
template <class K>
inline unsigned resident_grid(K kernel, int block, size_t smem = 0) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    return unsigned((per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148));
}

// Programmatic dependent launch (captured small-batch chains): a kernel of
// the chain lets its successor's CTAs be scheduled at once
// (launch_dependents) and waits for its predecessor's completion and memory
// (wait) before touching anything the predecessor wrote.  Both are no-ops for
// an ordinary launch, so the kernels call them unconditionally.
static __device__ int g_pdl_early = 0;  // 1: successors scheduled at entry (GPMA_PDL_EARLY=1; measured slower)
__device__ __forceinline__ void pdl_enter() {
    if (g_pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Host side: while pdl_chain() is set on this thread (a small-batch capture),
// launch_k adds the programmatic-serialization attribute, so the captured
// edge to the previous kernel becomes a programmatic one.
inline bool& pdl_chain() {
    static thread_local bool on = false;
    return on;
}
template <typename... P, typename... A>
inline void launch_k(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (pdl_chain()) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    GPMA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}

// stage / span stamp: the complement of %globaltimer kept by atomicMax, so
// the earliest caller wins and 0 means "not stamped" (thread 0 of each CTA)
__device__ __forceinline__ void stamp_first(ull* slot) {
    if (slot && threadIdx.x == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        atomicMax(slot, ~g);
    }
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Streaming (evict-first) 64-bit loads/stores for single-touch traffic.
__device__ __forceinline__ u64 ld_cs(const u64* p) { return __ldcs(reinterpret_cast<const unsigned long long*>(p)); }

// Edge-key helpers (graph.hpp:27-37).
__host__ __device__ __forceinline__ u64 pack_edge(u32 src, u32 dst) { return (u64(src) << 32) | dst; }
__host__ __device__ __forceinline__ u32 src_of(u64 key) { return u32(key >> 32); }
__host__ __device__ __forceinline__ u32 dst_of(u64 key) { return u32(key & 0xFFFFFFFFull); }
__host__ __device__ __forceinline__ bool is_guard(u64 key) { return (key & 0xFFFFFFFFull) == kGuardDst; }

// Growable device buffer (grow-only; contents not preserved on growth).
// NVTX ranges (SURVEY §5 tracing): one per batch / analytic call and one per
// stage of a batch, for nsys / ncu --nvtx; no-ops when no tool is attached
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope&) = delete;
    NvtxScope& operator=(const NvtxScope&) = delete;
};
// the current stage of a batch: each call closes the previous one
struct NvtxStages {
    bool open = false;
    void next(const char* name) {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    ~NvtxStages() {
        if (open) nvtxRangePop();
    }
};

template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        size_t c = n < 1024 ? 1024 : n + n / 4;
        GPMA_CUDA(cudaMalloc(&ptr, c * sizeof(T)));
        cap = c;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace gpma
