// sgpu_common.cuh — warp primitives and sm_100a PTX wrappers shared by the
// libsgpu kernels (mbarrier + cp.async.bulk staging, lane masks).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sgpu.h"

namespace sg {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// Dynamic work distribution (K1 kernels): ctr[0] hands out work items one
// warp at a time; ctr[1] counts warps that have made their failing fetch.
// The last warp of the launch resets both, so every launch - and every
// replay of a captured CUDA graph - starts from zero.  Warp-collective.
__device__ __forceinline__ uint64_t work_fetch(unsigned long long* ctr, uint32_t lane) {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1ull);
    return (uint64_t)__shfl_sync(FULL, v, 0);
}
// reset_list: also reset the deferred-list count ctr[2] (every warp of this
// launch read it before it counted itself done)
__device__ __forceinline__ void work_done(unsigned long long* ctr, uint32_t lane, bool reset_list = false) {
    if (lane == 0) {
        const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(ctr + 1, 1ull) == warps - 1) {  // no fetch of this launch is left
            atomicExch(ctr, 0ull);
            atomicExch(ctr + 1, 0ull);
            if (reset_list) atomicExch(ctr + 2, 0ull);
        }
    }
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Lexicographic warp minimum of a 64-bit key via two 32-bit REDUX ops.
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
    uint32_t hi = __reduce_min_sync(FULL, (uint32_t)(v >> 32));
    uint32_t lo = __reduce_min_sync(FULL, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0xFFFFFFFFu);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src);
    uint32_t hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

// ---- L2 eviction-priority hints -----------------------------------------
// Streamed inputs are read once (evict_first); scattered per-app outputs are
// written piecemeal over a simulation, so their sectors are kept in L2
// (evict_last) until complete instead of being evicted partially written.

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ldg_stream(const void* ptr, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ void stg_keep(uint32_t* ptr, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(ptr), "r"(v), "l"(pol) : "memory");
}

// ---- mbarrier + 1-D bulk async copy (TMA engine, no tensor map) ----------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_addr(bar)),
        "r"(bytes)
        : "memory");
}

// Bulk copy global -> shared completing on an mbarrier (size % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_addr(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

}  // namespace sg
