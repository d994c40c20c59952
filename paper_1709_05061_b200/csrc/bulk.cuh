// bulk.cuh — sm_100a bulk-copy (TMA engine, non-tensor) + mbarrier helpers.
//
// cp.async.bulk moves a contiguous, 16-byte aligned run of bytes between HBM
// and shared memory on the TMA engine: one instruction per run instead of one
// load + store per 16 bytes per thread, no registers held while in flight,
// completion signalled on an mbarrier (loads) or a bulk group (stores).  The
// PMA's unit of work is a 128-byte leaf line (16 keys or 16 values), exactly
// one bulk copy.
#pragma once

#include "common.cuh"

namespace gpma {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// arrive (count 1) and raise the expected transaction bytes of the phase
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(u64* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// HBM -> smem, completes `bytes` transaction bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// smem -> HBM (bulk group of the issuing thread)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }

// the thread's committed bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// generic-proxy smem writes -> visible to the async proxy (bulk stores, or
// bulk loads overwriting the buffer)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace gpma
