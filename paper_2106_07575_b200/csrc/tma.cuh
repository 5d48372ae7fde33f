// Minimal sm_90+/sm_100a async-copy plumbing: mbarriers and 1-D bulk copies (TMA engine,
// SASS UBLKCP) from global to shared memory, completion tracked by transaction bytes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pty {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// Bounded wait: a protocol bug becomes a launch failure (trap) after ~seconds, never a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, phase)) {
        if (++spins == (1u << 26)) __trap();
    }
}

// dst (shared) <- src (global), bytes multiple of 16, both 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk L2 prefetch (TMA engine, no shared memory / registers involved); bytes multiple of 16.
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Threads 0..pieces-1 of the CTA each prefetch one 16 KB piece of [src, src + bytes).
__device__ __forceinline__ void prefetch_l2_frame(const void* src, uint32_t bytes, int tid) {
    constexpr uint32_t PIECE = 16384;
    const uint32_t pieces = (bytes + PIECE - 1) / PIECE;
    if ((uint32_t)tid < pieces) {
        const uint32_t off = (uint32_t)tid * PIECE;
        prefetch_l2(static_cast<const char*>(src) + off, bytes - off < PIECE ? bytes - off : PIECE);
    }
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace pty
