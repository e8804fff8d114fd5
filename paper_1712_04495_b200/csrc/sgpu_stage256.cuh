// sgpu_stage256.cuh — warp-collective staging of one 129..256-app T0 trace
// for the octet kernel (K1 v8, shared memory) and the global-table lane
// kernel (K1 v9, global memory): SoA records in (arrival, index) order,
// class masks of the distinct priorities (highest first), the fit table
// (256-bit rows at every FS-th rank, as 8 u32 = 4 u64 words), the
// rank-lookup buckets (u16, LB of them, then lo / hi / scale as u32), and
// meta (u32): [0] n, [1] fail, [2] apps arriving at t = 0, [3] classes,
// [4..5] sum(arrival + busy) (the speed-up numerator), [6] 32-bit lane keys
// suffice.  Pointers are generic: the slot lives in shared or global memory.
#pragma once

#include "sgpu_lanesim.cuh"
#include "sgpu_warpsort.cuh"

namespace sg {

constexpr uint32_t kStage256FS = 4;      // fit-table stride (ranks)
constexpr uint32_t kStage256MaxCls = 8;  // priority classes per trace

struct Slot256 {
    uint32_t *s_a, *s_mem, *s_bw;  // N + 1 entries (s_mem[N] = ~0)
    uint32_t* s_ms;                // optional: requests in rank order, N + 4 (~0 past the end)
    uint16_t *s_por, *s_lt;        // N + 4 ranks; LB buckets + 3 u32
    uint32_t *s_tbl, *s_cm, *meta; // (N / FS + 1) x 8; classes x 8; 8
    uint16_t* s_rank;              // scratch, N entries
    uint32_t* s_lt32;              // optional: packed bucket entries (request << 9 | rank), LB of them + 3 u32
    uint32_t rs;                   // record stride of s_mem / s_bw in u32 (2: interleaved pairs)
};

template <uint32_t LB, uint32_t FS = kStage256FS>
__device__ __forceinline__ void stage256(const SimParams& P, bool need_cls, const Slot256& S, uint64_t t,
                                         uint32_t lane) {
    constexpr uint32_t N = 256;
    constexpr uint32_t kOctFS = FS;
    constexpr int K = 8;  // apps per lane
    uint64_t a0;
    uint32_t na;
    if (P.trace_offsets) {
        const uint64_t o0 = P.trace_offsets[0];
        a0 = P.trace_offsets[t] - o0;
        na = (uint32_t)(P.trace_offsets[t + 1] - P.trace_offsets[t]);
    } else {
        a0 = t * P.apps_per_trace;
        na = P.apps_per_trace;
    }
    const uint4* src = reinterpret_cast<const uint4*>(P.apps + a0);
    uint32_t* s_a = S.s_a;
    uint32_t* s_mem = S.s_mem;
    uint32_t* s_bw = S.s_bw;
    uint16_t* s_por = S.s_por;
    uint16_t* s_lt = S.s_lt;
    uint32_t* s_tbl = S.s_tbl;
    uint32_t* s_cm = S.s_cm;
    uint32_t* meta = S.meta;
    uint16_t* s_rank = S.s_rank;  // position -> rank (scratch)

    uint64_t key[K];
    bool big = false;
    uint32_t amax = 0, seq_lo = 0, seq_hi = 0, bsum = 0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        key[k] = kInf;
        if (i < na) {
            const uint4 f = ldg_stream(src + i, l2_policy_evict_first());
            key[k] = ((uint64_t)f.x << 10) | i;
            big = big || f.x >= (1u << 31) || f.z >= (1u << kBusyBits);
            amax = max(amax, f.x);
            // speed-up numerator (arrival + busy), summed in 16-bit halves
            seq_lo += (f.x & 0xFFFFu) + (f.z & 0xFFFFu);
            seq_hi += (f.x >> 16) + min(f.z >> 16, 1u << 16);
            bsum += min(f.z, 1u << kBusyBits);
        }
    }
    uint32_t fail = __any_sync(FULL, big) ? 1u : 0u;
    seq_lo = __reduce_add_sync(FULL, seq_lo);
    seq_hi = __reduce_add_sync(FULL, seq_hi);
    amax = __reduce_max_sync(FULL, amax);
    bsum = __reduce_add_sync(FULL, bsum);
    warp_sort_keys<K>(key, amax < (1u << 22), lane);
    __syncwarp();
    // SoA records in arrival order
    uint32_t memk[K], prk[K];
    uint32_t zc = 0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t e = (uint32_t)k * 32u + lane;
        memk[k] = ~0u;
        prk[k] = 0;
        const bool v = key[k] != kInf;
        if (v) {
            const uint32_t i = (uint32_t)key[k] & kAppMask;
            const uint4 f = __ldg(src + i);  // just loaded: an L1 hit
            s_a[e] = f.x;
            s_mem[e * S.rs] = f.y;
            s_bw[e * S.rs] = (f.z & ((1u << kBusyBits) - 1u)) | (i << kBusyBits);
            memk[k] = f.y;
            prk[k] = f.w & 0xFFu;
        }
        zc += __popc(__ballot_sync(FULL, v && (key[k] >> 10) == 0));
    }
    // priority classes (policy.py:58-63): the distinct priorities, highest
    // first; class word k of class c = the ballot of position k*32 + lane
    if (need_cls) {
        uint32_t pmax = 0, pres = 0;
#pragma unroll
        for (int k = 0; k < K; k++) {
            pmax = max(pmax, key[k] != kInf ? prk[k] : 0u);
            pres |= key[k] != kInf && prk[k] < 32 ? 1u << prk[k] : 0u;
        }
        pmax = __reduce_max_sync(FULL, pmax);
        pres = __reduce_or_sync(FULL, pres);
        const uint32_t ncls = __popc(pres);
        if (pmax >= 32 || ncls > kStage256MaxCls) {
            fail = 1;
        } else {
            uint32_t cls[K];
#pragma unroll
            for (int k = 0; k < K; k++) {
                cls[k] = ~0u;
                if (key[k] != kInf) {
                    cls[k] = __popc((uint32_t)((uint64_t)pres >> (prk[k] + 1u)));
                    s_bw[((uint32_t)k * 32u + lane) * S.rs] |= cls[k] << kClsShift;
                }
            }
            for (uint32_t c = 0; c < ncls; c++) {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const uint32_t w = __ballot_sync(FULL, cls[k] == c);
                    if (lane == 0) s_cm[c * 8u + (uint32_t)k] = w;
                }
            }
            if (lane == 0) meta[3] = ncls;
        }
    }
    // fit table: requests ascending; T[r] = positions of the r smallest
    uint64_t mk[K];
    uint32_t mx = 0, mn = ~0u;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t e = (uint32_t)k * 32u + lane;
        mk[k] = memk[k] != ~0u ? (((uint64_t)memk[k] << 8) | e) : kInf;
        mx = max(mx, memk[k] != ~0u ? memk[k] : 0u);
        mn = min(mn, memk[k]);
    }
    mx = __reduce_max_sync(FULL, mx);
    mn = __reduce_min_sync(FULL, mn);
    if (mn > mx) mn = mx;  // empty trace
    warp_sort_keys<K>(mk, mx < (1u << 24), lane);
    const uint64_t sc = ((uint64_t)LB << 32) / ((uint64_t)(mx - mn) + 1ull);
    const uint32_t scale = sc > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)sc;
    uint32_t bcarry = 0;  // bucket of the last rank of the previous row (+1)
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t r = (uint32_t)k * 32u + lane;
        const bool valid = mk[k] != kInf;
        const uint32_t pos = (uint32_t)mk[k] & 0xFFu;
        s_por[r] = valid ? (uint16_t)pos : (uint16_t)N;
        if (S.s_ms) S.s_ms[r] = valid ? (uint32_t)(mk[k] >> 8) : ~0u;
        if (valid) s_rank[pos] = (uint16_t)r;
        // LT[j] = first rank whose bucket is >= j: rank r owns (b[r-1], b[r]]
        const uint32_t b = valid ? min((uint32_t)(((uint64_t)((uint32_t)(mk[k] >> 8) - mn) * scale) >> 32),
                                       LB - 1u) + 1u
                                 : LB + 1u;
        uint32_t bp = __shfl_up_sync(FULL, b, 1);
        if (lane == 0) bp = bcarry;
        const uint32_t ent = (min(valid ? (uint32_t)(mk[k] >> 8) : kLtSat, kLtSat) << 9) | r;
        for (uint32_t j = bp; j < min(b, LB + 1u); j++)
            if (j < LB) {
                if (S.s_lt32)
                    S.s_lt32[j] = ent;
                else
                    s_lt[j] = (uint16_t)r;
            }
        bcarry = __shfl_sync(FULL, b, 31);
    }
    for (uint32_t j = bcarry + lane; j < LB; j += 32u) {
        if (S.s_lt32)
            S.s_lt32[j] = (kLtSat << 9) | N;
        else
            s_lt[j] = (uint16_t)N;
    }
    __syncwarp();
    // rows R = 0..N/FS: word w of T[FS R] = positions 32w + b whose rank < FS R
    {
        uint32_t myrank[8];
#pragma unroll
        for (uint32_t w = 0; w < 8; w++) {
            const uint32_t p = 32u * w + lane;
            myrank[w] = p < na ? s_rank[p] : 0xFFFFu;
        }
        for (uint32_t R = 0; R <= N / kOctFS; R++) {
            uint32_t word = 0;
#pragma unroll
            for (uint32_t w = 0; w < 8; w++) {
                const uint32_t b = __ballot_sync(FULL, myrank[w] < kOctFS * R);
                word = lane == w ? b : word;
            }
            if (lane < 8) s_tbl[R * 8u + lane] = word;
        }
    }
    if (lane == 0) {
        uint32_t* prm = S.s_lt32 ? S.s_lt32 + LB : reinterpret_cast<uint32_t*>(s_lt + LB);
        prm[0] = mn;
        prm[1] = mx;
        prm[2] = scale;
        s_mem[N * S.rs] = ~0u;
        meta[0] = na;
        meta[1] = fail;
        meta[2] = zc;
        const uint64_t seq = (uint64_t)seq_lo + ((uint64_t)seq_hi << 16);
        meta[4] = (uint32_t)seq;
        meta[5] = (uint32_t)(seq >> 32);
        // every event time <= max arrival + busy sum: 32-bit lane keys
        // (LaneKey<8, true>) suffice below their limit
        meta[6] = (uint64_t)amax + bsum < LaneKey<8, true>::LIM ? 1u : 0u;
    }
    if (lane < FS) s_por[N + lane] = (uint16_t)N;
    if (lane < 4 && S.s_ms) S.s_ms[N + lane] = ~0u;
    __syncwarp();
}

}  // namespace sg
