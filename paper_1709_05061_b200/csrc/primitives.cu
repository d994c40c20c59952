// primitives.cu — the reference's data-parallel building blocks
// (primitives.hpp:21-84) as C-ABI entry points over the library's own
// device primitives (radix.cuh: onesweep sort, single-pass exclusive sum).
// The batch pipeline calls the same templates directly; these entries make
// them usable (and testable) on their own, host or device arrays.
#include <mutex>
#include <string>

#include "pmagraph_cuda.h"
#include "radix.cuh"

using namespace gpma;

namespace {
thread_local std::string g_prim_err;

struct PrimCtx {
    cudaStream_t stream = nullptr;
    RadixWorkspace rws;
    ScanWorkspace sws;
    DevBuf<u64> k, kalt;
    DevBuf<u32> v, valt;
};

std::mutex g_mu;
PrimCtx* g_ctx[64] = {};

PrimCtx& ctx(int device) {
    if (device < 0 || device >= 64) throw ApiError(PMA_EINVAL, "device index out of range");
    GPMA_CUDA(cudaSetDevice(device));
    if (!g_ctx[device]) {
        auto* c = new PrimCtx;
        GPMA_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        g_ctx[device] = c;
    }
    return *g_ctx[device];
}

template <class F>
int prim_guard(F&& f) {
    try {
        std::lock_guard<std::mutex> lk(g_mu);
        f();
        return PMA_OK;
    } catch (const ApiError& e) {
        g_prim_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_prim_err = e.what();
        return PMA_ECUDA;
    }
}

void check_bits(int begin_bit, int end_bit) {
    if (begin_bit < 0 || end_bit > 64 || begin_bit > end_bit)
        throw ApiError(PMA_EINVAL, "sort_by_key: bit range outside [0, 64]");
}

// keys/payload in c.k / c.v (device); result back in the same buffers
void sort_in_ctx(PrimCtx& c, u64* keys, u32* pay, u64 n, int b, int e) {
    c.kalt.reserve(n);
    if (pay) c.valt.reserve(n);
    const int alt = radix_sort(c.stream, c.rws, keys, c.kalt.ptr, pay, pay ? c.valt.ptr : nullptr, n, b, e);
    if (alt) {
        GPMA_CUDA(cudaMemcpyAsync(keys, c.kalt.ptr, n * 8, cudaMemcpyDeviceToDevice, c.stream));
        if (pay) GPMA_CUDA(cudaMemcpyAsync(pay, c.valt.ptr, n * 4, cudaMemcpyDeviceToDevice, c.stream));
    }
}
}  // namespace

extern "C" {

const char* gpma_primitives_last_error(void) { return g_prim_err.c_str(); }

int gpma_sort_by_key_device(int device, uint64_t* d_keys, uint32_t* d_payload, size_t n, int begin_bit,
                            int end_bit) {
    return prim_guard([&] {
        check_bits(begin_bit, end_bit);
        PrimCtx& c = ctx(device);
        sort_in_ctx(c, d_keys, d_payload, n, begin_bit, end_bit);
        GPMA_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int gpma_sort_by_key(int device, uint64_t* keys, uint32_t* payload, size_t n, int begin_bit, int end_bit) {
    return prim_guard([&] {
        check_bits(begin_bit, end_bit);
        if (n == 0) return;
        PrimCtx& c = ctx(device);
        c.k.reserve(n);
        GPMA_CUDA(cudaMemcpyAsync(c.k.ptr, keys, n * 8, cudaMemcpyHostToDevice, c.stream));
        if (payload) {
            c.v.reserve(n);
            GPMA_CUDA(cudaMemcpyAsync(c.v.ptr, payload, n * 4, cudaMemcpyHostToDevice, c.stream));
        }
        sort_in_ctx(c, c.k.ptr, payload ? c.v.ptr : nullptr, n, begin_bit, end_bit);
        GPMA_CUDA(cudaMemcpyAsync(keys, c.k.ptr, n * 8, cudaMemcpyDeviceToHost, c.stream));
        if (payload) GPMA_CUDA(cudaMemcpyAsync(payload, c.v.ptr, n * 4, cudaMemcpyDeviceToHost, c.stream));
        GPMA_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int gpma_exclusive_scan_device(int device, const uint32_t* d_in, uint32_t* d_out, size_t n) {
    return prim_guard([&] {
        PrimCtx& c = ctx(device);
        exclusive_sum(c.stream, c.sws, d_in, d_out, n);
        GPMA_CUDA(cudaStreamSynchronize(c.stream));
    });
}

}  // extern "C"
