// sgpu_aux.cu — K2 stats_reduce, K3 trace_gen, K4 select_grants_batch.
#include "sgpu_common.cuh"
#include "sgpu_internal.h"

namespace sg {

// ------------------------------------------------------------ K2 reduce
// Sums / maxima of integer per-trace statistics.  Integer sums are exact and
// order-independent, so the result is deterministic regardless of the grid.

constexpr int kReduceThreads = 256;

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

__global__ void __launch_bounds__(kReduceThreads)
stats_reduce_kernel(const sg_trace_stats* __restrict__ st, uint64_t count, sg_aggr* out) {
    uint64_t s[SG_AGGR_NSUM] = {0};
    uint64_t m[16 - SG_AGGR_NSUM] = {0};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4* p = reinterpret_cast<const uint4*>(st + i);
        const uint4 a = __ldg(p), b = __ldg(p + 1);
        // a = {makespan, busy, I.lo, I.hi}; b = {grants, pops, maxh|unf<<16, status}
        const uint32_t maxh = b.z & 0xFFFFu, unf = b.z >> 16;
        s[0] += 1;
        s[1] += a.x;
        s[2] += a.y;
        s[3] += ((uint64_t)a.w << 32) | a.z;
        s[4] += b.x;
        s[5] += b.y;
        s[6] += unf;
        s[7] += maxh;
        s[8] += unf != 0;
        s[9] += b.w != 0;
        m[0] = max(m[0], (uint64_t)a.x);
        m[1] = max(m[1], (uint64_t)maxh);
        m[2] |= b.w;
    }
    __shared__ uint64_t sh[kReduceThreads / 32][16];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < SG_AGGR_NSUM; k++) {
        const uint64_t v = warp_sum_u64(s[k]);
        if (l == 0) sh[w][k] = v;
    }
#pragma unroll
    for (int k = 0; k < 16 - SG_AGGR_NSUM; k++) {
        uint64_t v = m[k];
        if (k == 2) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(FULL, v, o);
        } else {
            v = warp_max_u64(v);
        }
        if (l == 0) sh[w][SG_AGGR_NSUM + k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 16) {
        const int k = threadIdx.x;
        uint64_t v = sh[0][k];
        for (int j = 1; j < kReduceThreads / 32; j++) {
            if (k < SG_AGGR_NSUM) v += sh[j][k];
            else if (k == SG_AGGR_NSUM + 2) v |= sh[j][k];
            else v = max(v, sh[j][k]);
        }
        unsigned long long* o = reinterpret_cast<unsigned long long*>(out) + k;
        if (k < SG_AGGR_NSUM) atomicAdd(o, (unsigned long long)v);
        else if (k == SG_AGGR_NSUM + 2) atomicOr(o, (unsigned long long)v);
        else atomicMax(o, (unsigned long long)v);
    }
}

cudaError_t launch_reduce(const sg_trace_stats* stats, uint64_t count, sg_aggr* out,
                          cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(sg_aggr), stream);
    if (e != cudaSuccess || count == 0) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (count + kReduceThreads - 1) / kReduceThreads;
    if (blocks > (uint64_t)sms * 4) blocks = (uint64_t)sms * 4;
    stats_reduce_kernel<<<(unsigned)blocks, kReduceThreads, 0, stream>>>(stats, count, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------ K3 generator
// Bit-identical twin of paper_1712_04495_b200/tracegen.py:generate.

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t uniform_u32(uint64_t h, uint32_t lo, uint32_t hi) {
    const uint64_t span = (uint64_t)hi - lo + 1;
    return (uint32_t)(lo + (((h >> 32) * span) >> 32));
}

__global__ void __launch_bounds__(256)
trace_gen_kernel(const sg_gen_params p, uint64_t trace_begin, uint64_t n_traces, uint64_t k0,
                 uint4* __restrict__ out) {
    const uint64_t total = n_traces * p.apps_per_trace;
    // (trace, app) of element g: 32-bit division while g fits (all BASELINE
    // shapes; 64-bit division is a long emulated sequence)
    const bool narrow = total <= 0xFFFFFFFFull;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t t, app;
        if (narrow) {
            const uint32_t t32 = (uint32_t)g / p.apps_per_trace;
            t = t32;
            app = (uint32_t)g - t32 * p.apps_per_trace;
        } else {
            t = g / p.apps_per_trace;
            app = g - t * p.apps_per_trace;
        }
        const uint64_t kt = mix64(k0 ^ (trace_begin + t));
        const uint64_t ha = mix64(kt ^ ((app << 3) | 0));
        const uint64_t hm = mix64(kt ^ ((app << 3) | 1));
        const uint64_t hb = mix64(kt ^ ((app << 3) | 2));
        const uint64_t hp = mix64(kt ^ ((app << 3) | 3)) >> 32;
        uint32_t arrival;
        if (p.arrival_kind == SG_ARR_CUBIC) {
            const uint64_t u = ha >> 40;
            const uint64_t c = (((u * u) >> 24) * u) >> 24;
            arrival = (uint32_t)(p.arr_lo + ((c * ((uint64_t)p.arr_hi - p.arr_lo + 1)) >> 24));
        } else {
            arrival = uniform_u32(ha, p.arr_lo, p.arr_hi);
        }
        uint32_t prio;
        if (p.prio_kind == SG_PRIO_SKEWED) {
            const uint64_t total_w = (1ull << p.prio_levels) - 1;
            const uint64_t r = (hp * total_w) >> 32;
            uint64_t cum = 0;
            prio = 0;
            for (uint32_t k = 0; k < p.prio_levels; k++) {
                cum += 1ull << (p.prio_levels - 1 - k);
                prio += r >= cum;
            }
        } else {
            prio = (uint32_t)((hp * p.prio_levels) >> 32);
        }
        const uint32_t dev = (uint32_t)app % p.ndev;
        out[g] = make_uint4(arrival, uniform_u32(hm, p.mem_lo, p.mem_hi),
                            uniform_u32(hb, p.busy_lo, p.busy_hi), prio | (dev << 8));
    }
}

cudaError_t launch_generate(const sg_gen_params& p, uint64_t trace_begin, uint64_t n_traces,
                            sg_app* out, cudaStream_t stream) {
    const uint64_t total = n_traces * p.apps_per_trace;
    if (total == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (total + 255) / 256;
    if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
    const uint64_t k0 = mix64(p.seed);
    trace_gen_kernel<<<(unsigned)blocks, 256, 0, stream>>>(p, trace_begin, n_traces, k0,
                                                           reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

// ------------------------------------------------------------ K4 select_grants
// One warp per queue: memshare/policy.py:52-74 with int64 byte sizes.

__global__ void __launch_bounds__(256)
select_grants_kernel(uint64_t n_queues, const uint64_t* __restrict__ qoff,
                     const int64_t* __restrict__ nbytes, const int32_t* __restrict__ prio,
                     const int64_t* __restrict__ free_bytes, const uint32_t* __restrict__ kind,
                     uint8_t* __restrict__ granted) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t o0 = qoff[0];
    for (uint64_t q = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n_queues;
         q += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t b = qoff[q] - o0, e = qoff[q + 1] - o0;
        const uint32_t n = (uint32_t)(e - b);
        const uint32_t k = kind[q];
        const bool restrict_top = k >= SG_POLICY_PFIFO;
        const bool fifo = (k & 1u) == 0;
        int32_t top = 0;
        if (restrict_top && n > 0) {
            int32_t best = INT32_MIN;
            for (uint32_t i = lane; i < n; i += 32) best = max(best, prio[b + i]);
            top = __reduce_max_sync(FULL, best);
        }
        int64_t budget = free_bytes[q];
        bool stop = false;
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            const bool valid = i < n;
            const int64_t nb = valid ? nbytes[b + i] : 0;
            const bool cand = valid && !stop && (!restrict_top || prio[b + i] == top);
            uint32_t rem = __ballot_sync(FULL, cand), gm = 0;
            while (rem) {
                const uint32_t head = __ffs(rem) - 1;
                const uint32_t fm = __ballot_sync(FULL, cand && nb <= budget) & rem;
                if (fifo) {
                    if (!((fm >> head) & 1u)) { stop = true; break; }
                    gm |= 1u << head;
                    budget -= __shfl_sync(FULL, nb, head);
                    rem &= rem - 1;
                } else {
                    if (!fm) break;
                    const uint32_t j = __ffs(fm) - 1;
                    gm |= 1u << j;
                    budget -= __shfl_sync(FULL, nb, j);
                    rem &= (j == 31) ? 0u : (0xFFFFFFFFu << (j + 1));
                }
            }
            if (valid) granted[b + i] = (gm >> lane) & 1u;
        }
    }
}

cudaError_t launch_select(uint64_t n_queues, const uint64_t* qoff, const int64_t* nbytes,
                          const int32_t* prio, const int64_t* free_bytes, const uint32_t* kind,
                          uint8_t* granted, cudaStream_t stream) {
    if (n_queues == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (n_queues * 32 + 255) / 256;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    select_grants_kernel<<<(unsigned)blocks, 256, 0, stream>>>(n_queues, qoff, nbytes, prio,
                                                               free_bytes, kind, granted);
    return cudaGetLastError();
}

}  // namespace sg

namespace sg {

// ------------------------------------------------------------ K5 pack16
// Host pipeline transfer format of one chunk (after its simulation): per app
// its busy ticks as u16 (0xFFFF = no memory request, hence no grant) and per
// (policy, app) its end tick as u16 (0xFFFF = SG_NEVER).  Host threads
// expand the end ticks into the caller's u32 array and derive every grant
// as end - busy (sgpu_abi.cu), so 10 B per app cross PCIe instead of 16 B
// of end ticks (and no 16-byte input record is re-read on the host).
// *overflow = 1 if the chunk is not exactly representable (a requesting
// app's busy >= 0xFFFF or an end tick >= 0xFFFF other than SG_NEVER): the
// host then copies that chunk's u32 end rows instead.  The end rows of
// policy p start at end + p * stride.

__global__ void __launch_bounds__(256)
pack16_kernel(const uint4* __restrict__ apps, const uint32_t* __restrict__ end, uint64_t na, uint64_t stride,
              uint32_t npol, uint16_t* __restrict__ b16, uint16_t* __restrict__ e16, uint32_t* overflow) {
    uint32_t bad = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 f = __ldcs(apps + i);  // arrival, mem, busy, attr
        bad |= (f.y != 0u) & (f.z >= 0xFFFFu);
        b16[i] = f.y == 0u ? (uint16_t)0xFFFFu : (uint16_t)f.z;
        for (uint32_t p = 0; p < npol; p++) {
            const uint32_t e = __ldcs(end + p * stride + i);
            bad |= (e != SG_NEVER) & (e >= 0xFFFFu);
            e16[p * na + i] = (uint16_t)(e == SG_NEVER ? 0xFFFFu : e);
        }
    }
    if (__any_sync(FULL, bad != 0) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1u);
}

cudaError_t launch_pack16(const sg_app* apps, const uint32_t* end, uint64_t na, uint64_t stride, uint32_t npol,
                          uint16_t* b16, uint16_t* e16, uint32_t* overflow, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(overflow, 0, sizeof(uint32_t), stream);
    if (e != cudaSuccess || na == 0) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (na + 255) / 256;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    pack16_kernel<<<(unsigned)blocks, 256, 0, stream>>>(reinterpret_cast<const uint4*>(apps), end, na, stride,
                                                         npol, b16, e16, overflow);
    return cudaGetLastError();
}

}  // namespace sg
