// sgpu_warpsort.cuh — warp-collective helpers shared by the lane (K1 v5)
// and octet (K1 v8) kernels' staging: 64-bit shuffles and an ascending
// bitonic sort of 32*K keys held K per lane.
#pragma once

#include <cstdint>

#include "sgpu_common.cuh"

namespace sg {

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
    const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m);
    const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int m) {
    const uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, m);
    const uint32_t hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t shfl_xor_key(uint32_t v, int m) { return __shfl_xor_sync(FULL, v, m); }
__device__ __forceinline__ uint64_t shfl_xor_key(uint64_t v, int m) { return shfl_xor_u64(v, m); }

// Ascending bitonic sort of 32*K keys held K per lane (element k*32 + lane).
template <int K, class KeyT>
__device__ __forceinline__ void warp_bitonic_sort(KeyT (&v)[K], uint32_t lane) {
    constexpr uint32_t N = 32u * K;
#pragma unroll
    for (uint32_t size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                const uint32_t ks = stride >> 5;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    if ((k & ks) == 0) {
                        const int kp = k | ks;
                        const bool up = (((uint32_t)k * 32u + lane) & size) == 0;
                        const KeyT a = v[k], b = v[kp];
                        const bool sw = up ? (a > b) : (a < b);
                        v[k] = sw ? b : a;
                        v[kp] = sw ? a : b;
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const KeyT o = shfl_xor_key(v[k], (int)stride);
                    const bool up = (((uint32_t)k * 32u + lane) & size) == 0;
                    const bool low = (lane & stride) == 0;
                    v[k] = (up == low) ? (v[k] < o ? v[k] : o) : (v[k] < o ? o : v[k]);
                }
            }
        }
    }
}

// Sort 64-bit keys (~0 = padding) with 32-bit compare-exchanges when every
// real key is below 2^32 - 1 (warp-uniform `narrow`): half the shuffles.
template <int K>
__device__ __forceinline__ void warp_sort_keys(uint64_t (&v)[K], bool narrow, uint32_t lane) {
    if (narrow) {
        uint32_t w[K];
#pragma unroll
        for (int k = 0; k < K; k++) w[k] = v[k] == ~0ull ? ~0u : (uint32_t)v[k];
        warp_bitonic_sort<K>(w, lane);
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = w[k] == ~0u ? ~0ull : (uint64_t)w[k];
    } else {
        warp_bitonic_sort<K>(v, lane);
    }
}

}  // namespace sg
