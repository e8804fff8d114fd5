// sgpu_lane.cu — K1 v5 `trace_sim_lane`: one LANE simulates one (trace,
// device, policy) of a T0 (burst) batch, 32 simulations per warp in SIMT.
// This file stages traces into shared memory and launches; the per-lane
// simulator itself (LaneSim) is in sgpu_lanesim.cuh.
//
// Same semantics as trace_sim_kernel (sgpu_sim.cu),
// restated for a single thread.  The T0 shape (cpu(arrival) -> alloc ->
// busy -> free, memshare/harness.py:478-490) makes these reductions exact:
//
//  * Arrival stream.  The initial pops run in index order at t = 0
//    (harness.py:560-562); an app with arrival a > 0 only pushes (a, c), with
//    c increasing in the app index, so arrivals pop in (a, index) order: a
//    per-trace sort, shared by every lane of the trace, replaces those heap
//    entries.  Heap counters are restated as order-preserving virtual
//    counters (LaneKey): the initial pop of app i owns counter i (its
//    arrival push, or the one busy end its inline run at t = 0 pushes), and
//    every later push counts up from N.  Comparing (t, virtual counter) is
//    therefore the reference's (t, counter) order (harness.py:505-508,
//    563-565).  32-bit keys when every time of the group's traces fits,
//    else 64-bit keys.
//  * Wake-ups.  grant_waiters pushes each granted waiter at (now, ++counter)
//    (harness.py:558): later than every pending entry of time `now`, earlier
//    than any entry of a later time.  They sit in a per-lane FIFO, drained in
//    one inner loop once no arrival / busy end of time `now` remains.  The
//    heap keeps busy ends only: a 4-ary heap of depth 2 per lane in shared
//    memory, laid out [slot][lane] so a warp's accesses are bank-conflict
//    free whatever slot each lane touches.
//  * Wait queue.  An app enqueues at most once, at its arrival pop, so the
//    queue (harness.py:532-536) is a presence bitmask over arrival positions,
//    in registers; queue order is position order.  select_grants
//    (policy.py:52-74) works on masks, one step per loop iteration: the
//    priority kinds restrict to the top class (per-trace class masks,
//    policy.py:58-63), FIFO grants the head while it fits, MMU takes first
//    fits with a shrinking budget.  For traces of <= 128 apps each step is
//    O(1): a per-trace table T[r] of the positions whose request is among the
//    r smallest gives the set that fits `budget` as T[#requests <= budget]
//    (bucket lookup), and the next first fit is the lowest bit of
//    mask & class & T above the last grant.
//
// 32-bit event keys when every time of the group's traces fits, else 64-bit
// keys, whose heap holds kLaneHeapW events in the same 2.5 KB region.  Two
// launches per batch: a trace whose 64-bit-key lanes overflow that heap is
// appended to a deferred list and re-simulated by the second (retry) pass
// with a kLaneHeapN-event 64-bit heap (a 5 KB region, lower occupancy); on
// C2's 32-bit-key traces that pass finds nothing to do.  Lanes that still
// cannot take the lane path (heap or FIFO capacity exceeded, too many
// priority classes, times near the 32-bit tick range) are re-simulated by
// the whole warp with the exact warp-per-trace TraceSim (sgpu_tracesim.cuh)
// right after, in the same kernel.
#include <cstring>

#include "sgpu_lanesim.cuh"
#include "sgpu_warpsort.cuh"

namespace sg {

constexpr uint32_t kLaneClassMasks = 64;    // class masks per warp, split over its trace slots
constexpr int kLaneWarpsPerBlock = 2;      // two warps share a block's 1 KB smem reservation
// Resident two-warp blocks per SM the register allocation is sized for.
// Nine (18 warps) caps registers at 96 per thread: a small loss at 64 apps
// (C2: 18.13 -> 18.30 ms), where eight blocks keep ~114 registers.  At 128
// apps shared memory allows five blocks, so registers are left free up to
// that (C4: 3.96e7 -> 4.03e7 trace-sims/s against the 96-register build;
// one-box A/Bs).
template <int K> struct LaneMinBlocks { static constexpr int v = K == 2 ? 8 : K == 4 ? 5 : 9; };
// With few traces per warp (npol * ndev >= 8, e.g. C5's 8 devices x 4
// policies) shared memory allows more blocks and registers limit residency:
// a 64-app variant capped for ten blocks (<= 96 registers) is used there.
constexpr int kLaneHiBlocks2 = 10;
// The 64-bit-key retry pass: a 5 KB heap per warp, so fewer resident blocks.
template <int K> struct LaneMinBlocksR { static constexpr int v = K == 2 ? 6 : K == 4 ? 4 : 7; };
struct LaneParams {
    SimParams sp;          // inputs/outputs + the fallback TraceSim layout (off_* relative to the warp region)
    uint32_t G;            // traces per warp (32 / lpt)
    uint32_t lpt;          // lanes per trace = npol * ndev
    uint32_t need_cls;     // a priority policy is requested: build class masks
    uint32_t need_tbl;     // an MMU-type policy on <= 64-app traces: build the fit table
    uint32_t cm_per_trace; // class-mask capacity of one trace slot
    uint32_t meta_stride;  // u16 per trace slot of the meta array
    // per-warp shared-memory layout (bytes)
    uint32_t off_a, off_mem, off_bw, off_por, off_lt, off_tbl, off_cm, off_meta, off_fb,
        warp_bytes;
};

// Per-trace-slot strides (in elements) of the shared arrays.  The u32
// record arrays hold N entries + the s_mem[N] sentinel; an odd stride skews
// the slots of a warp onto different banks.
template <uint32_t N, uint32_t FS> struct SlotStride {
    static constexpr uint32_t S32 = N + 1;          // u32 record arrays
    static constexpr uint32_t POR = N + 4;          // rank -> position (u8) + 4 sentinels
    static constexpr uint32_t LTB = LtBuckets<FS>::v + 12;  // rank lookup: u8 buckets + 3 u32 params
    static constexpr uint32_t T4 = (N / FS + 1) * ((N + 63) / 64);  // fit table (NW words per entry)
};

// meta per trace slot (u16), for ndev devices: [0] n, [1] fail (big times /
// too many classes), [2] 32-bit keys allowed, [3 + d] (d = 0..ndev) device
// bounds in arrival order, [4 + ndev + d] apps of device d arriving at t = 0,
// [4 + 2 ndev + d] (d = 0..ndev) class-mask index bounds per device
__host__ __device__ constexpr uint32_t meta_dev(uint32_t d) { return 3u + d; }
__host__ __device__ constexpr uint32_t meta_z(uint32_t ndev, uint32_t d) { return 4u + ndev + d; }
__host__ __device__ constexpr uint32_t meta_cls(uint32_t ndev, uint32_t d) { return 4u + 2u * ndev + d; }
__host__ __device__ constexpr uint32_t meta_u16(uint32_t ndev) { return (5u + 3u * ndev + 7u) & ~7u; }
// ndev > 1 only (one spare u16 after the class bounds; ndev == 1 ignores the
// device field): the trace holds an app with device index >= ndev
__host__ __device__ constexpr uint32_t meta_baddev(uint32_t ndev) { return 5u + 3u * ndev; }
static_assert(meta_baddev(2) < meta_u16(2) && meta_baddev(3) < meta_u16(3) && meta_baddev(4) < meta_u16(4) &&
                  meta_baddev(5) < meta_u16(5) && meta_baddev(6) < meta_u16(6) && meta_baddev(7) < meta_u16(7) &&
                  meta_baddev(8) < meta_u16(8),
              "meta layout");

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void lane_trace_range(const SimParams& P, uint64_t t, uint64_t& a0,
                                                 uint32_t& na) {
    if (P.trace_offsets) {
        const uint64_t o0 = P.trace_offsets[0];
        a0 = P.trace_offsets[t] - o0;
        na = (uint32_t)(P.trace_offsets[t + 1] - P.trace_offsets[t]);
    } else {
        a0 = t * P.apps_per_trace;
        na = P.apps_per_trace;
    }
}

// Exclusive prefix over lanes 0..7 of a per-device count held by lane d.
__device__ __forceinline__ uint32_t dev_scan_incl(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const uint32_t u = __shfl_up_sync(FULL, v, o);
        if (lane >= (uint32_t)o) v += u;
    }
    return v;
}

// Stage trace t into slot g (scratch: the warp's fb region): SoA records in
// (device, arrival, index) order, class masks of each device's priority
// classes (highest first), the fit table (every FS-th rank).  Warp-collective.
template <int K, uint32_t FS>
__device__ __forceinline__ void stage_trace(const LaneParams& L, uint8_t* ws, uint32_t g, uint64_t t,
                                            uint32_t lane) {
    const SimParams& P = L.sp;
    constexpr uint32_t N = 32u * K;
    constexpr uint32_t NW = (N + 63u) / 64u;
    uint64_t a0;
    uint32_t na;
    lane_trace_range(P, t, a0, na);
    uint4* raw = reinterpret_cast<uint4*>(ws + L.off_fb);
    using SS = SlotStride<N, FS>;
    uint32_t* s_a = reinterpret_cast<uint32_t*>(ws + L.off_a) + g * SS::S32;
    uint32_t* s_mem = reinterpret_cast<uint32_t*>(ws + L.off_mem) + g * SS::S32;
    uint32_t* s_bw = reinterpret_cast<uint32_t*>(ws + L.off_bw) + g * SS::S32;
    uint16_t* meta = reinterpret_cast<uint16_t*>(ws + L.off_meta) + g * L.meta_stride;
    const uint32_t ndev = P.ndev;

    uint64_t key[K];
    bool big = false, bad_dev = false;
    uint32_t bsum = 0;  // busy sum (each busy < 2^21 unless `big`)
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        key[k] = kInf;
        if (i < na) {
            const uint4 f = ldg_stream(reinterpret_cast<const uint4*>(P.apps + a0) + i, l2_policy_evict_first());
            raw[i] = f;
            uint32_t dv = ndev > 1 ? (f.w >> 8) & 0xFFu : 0u;
            if (dv >= ndev) {  // simulated on device 0, flagged SG_ST_BAD_DEVICE
                dv = 0;
                bad_dev = true;
            }
            key[k] = ((uint64_t)dv << 42) | ((uint64_t)f.x << 10) | i;
            big = big || f.x >= (1u << 31) || f.z >= (1u << kBusyBits);
            bsum += min(f.z, 1u << kBusyBits);
        }
    }
    uint32_t fail = __any_sync(FULL, big) ? 1u : 0u;
    bsum = __reduce_add_sync(FULL, bsum);
    uint32_t amax = 0;
#pragma unroll
    for (int k = 0; k < K; k++) amax = max(amax, key[k] != kInf ? (uint32_t)(key[k] >> 10) : 0u);
    amax = __reduce_max_sync(FULL, amax);
    // every event time is <= max arrival + busy sum: 32-bit keys suffice
    // when that stays below LaneKey::LIM
    const bool narrow = (uint64_t)amax + bsum < LaneKey<K, true>::LIM;
    bool wide_big = false;  // 64-bit keys and more than kLaneHeapW apps can be busy at once
    warp_sort_keys<K>(key, ndev == 1 && amax < (1u << 22), lane);  // device bits sit above bit 41
    __syncwarp();
    // SoA records in arrival order
    uint32_t memk[K], prk[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t e = (uint32_t)k * 32u + lane;
        memk[k] = ~0u;
        prk[k] = 0;
        if (key[k] != kInf) {
            const uint32_t i = (uint32_t)key[k] & kAppMask;
            const uint4 f = raw[i];
            s_a[e] = f.x;
            s_mem[e] = f.y;
            s_bw[e] = (f.z & ((1u << kBusyBits) - 1u)) | (i << kBusyBits);
            memk[k] = f.y;
            prk[k] = f.w & 0xFFu;
        }
    }
    // device bounds and arrivals at t = 0, per device (lane d holds device d)
    uint32_t cnt_d = 0, z_d = 0;
    for (uint32_t d = 0; d < ndev; d++) {
        uint32_t c = 0, zc = 0;
#pragma unroll
        for (int k = 0; k < K; k++) {
            const bool v = key[k] != kInf && (uint32_t)(key[k] >> 42) == d;
            c += __popc(__ballot_sync(FULL, v));
            zc += __popc(__ballot_sync(FULL, v && ((key[k] >> 10) & 0xFFFFFFFFull) == 0));
        }
        if (lane == d) { cnt_d = c; z_d = zc; }
    }
    const uint32_t dincl = dev_scan_incl(cnt_d, lane);
    uint32_t pmax = 0;
#pragma unroll
    for (int k = 0; k < K; k++) pmax = max(pmax, key[k] != kInf ? prk[k] : 0u);
    pmax = __reduce_max_sync(FULL, pmax);
    if (L.need_cls && ndev == 1 && pmax < 32) {
        // one device, priorities below 32: the classes (policy.py:58-63) are
        // the distinct priorities, highest first; class index = number of
        // distinct priorities above the app's own
        uint64_t* cm = reinterpret_cast<uint64_t*>(ws + L.off_cm) + g * (L.cm_per_trace * NW);
        uint32_t pres = 0;
#pragma unroll
        for (int k = 0; k < K; k++) pres |= key[k] != kInf ? 1u << prk[k] : 0u;
        pres = __reduce_or_sync(FULL, pres);
        const uint32_t ncls_total = __popc(pres);
        if (ncls_total > L.cm_per_trace || ncls_total > kLaneMaxCls) {
            fail = 1;
        } else {
            uint32_t cls[K];
#pragma unroll
            for (int k = 0; k < K; k++) {
                cls[k] = ~0u;
                if (key[k] != kInf) {
                    cls[k] = __popc((uint32_t)((uint64_t)pres >> (prk[k] + 1u)));
                    s_bw[(uint32_t)k * 32u + lane] |= cls[k] << kClsShift;
                }
            }
            for (uint32_t c = 0; c < ncls_total; c++) {
#pragma unroll
                for (uint32_t w = 0; w < NW; w++) {
                    const uint32_t lo = __ballot_sync(FULL, cls[min(2u * w, (uint32_t)K - 1u)] == c && 2u * w < (uint32_t)K);
                    const uint32_t hi = __ballot_sync(FULL, cls[min(2u * w + 1u, (uint32_t)K - 1u)] == c && 2u * w + 1u < (uint32_t)K);
                    if (lane == 0) cm[c * NW + w] = ((uint64_t)hi << 32) | lo;
                }
            }
            if (lane == 0) meta[meta_cls(1, 1)] = (uint16_t)ncls_total;
        }
    } else if (L.need_cls) {
        // classes = (device, priority) groups, highest priority first
        // (policy.py:58-63); one mask of arrival positions per class
        uint64_t* cm = reinterpret_cast<uint64_t*>(ws + L.off_cm) + g * (L.cm_per_trace * NW);
        uint32_t ck[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const uint32_t e = (uint32_t)k * 32u + lane;
            ck[k] = key[k] != kInf ? (((uint32_t)(key[k] >> 42) << 18) | ((255u - prk[k]) << 10) | e) : ~0u;
        }
        warp_bitonic_sort<K>(ck, lane);
        uint32_t bnd[K];
        uint32_t ncls_total = 0;
#pragma unroll
        for (int k = 0; k < K; k++) {
            uint32_t prev = __shfl_up_sync(FULL, ck[k], 1);
            const uint32_t pk = __shfl_sync(FULL, ck[k > 0 ? k - 1 : 0], 31);
            if (lane == 0) prev = k > 0 ? pk : ~0u;
            const bool valid = ck[k] != ~0u;
            bnd[k] = __ballot_sync(FULL, valid && (prev == ~0u || (prev >> 10) != (ck[k] >> 10)));
            ncls_total += __popc(bnd[k]);
        }
        // classes per device (lane d: device d) and their index bounds
        uint32_t nc_d = 0;
        for (uint32_t d = 0; d < ndev; d++) {
            uint32_t c = 0;
#pragma unroll
            for (int k = 0; k < K; k++)
                c += __popc(bnd[k] & __ballot_sync(FULL, ck[k] != ~0u && (ck[k] >> 18) == d));
            if (lane == d) nc_d = c;
        }
        const uint32_t cincl = dev_scan_incl(nc_d, lane);
        const uint32_t cexcl = cincl - nc_d;
        if (ncls_total > L.cm_per_trace || __any_sync(FULL, nc_d > kLaneMaxCls)) {
            fail = 1;
        } else {
            for (uint32_t i = lane; i < ncls_total * NW; i += 32) cm[i] = 0ull;
            __syncwarp();
            uint32_t before = 0;  // classes starting before word k
#pragma unroll
            for (int k = 0; k < K; k++) {
                const uint32_t c0 = __shfl_sync(FULL, cexcl, ck[k] != ~0u ? (ck[k] >> 18) & 31u : 0u);
                if (ck[k] != ~0u) {
                    const uint32_t ci = before + __popc(bnd[k] & ((2u << lane) - 1u)) - 1u;
                    const uint32_t apos = ck[k] & 0x3FFu;
                    atomicOr(reinterpret_cast<unsigned long long*>(&cm[ci * NW + (apos >> 6)]),
                             1ull << (apos & 63u));
                    // the app's class within its device, for the lane's class set
                    s_bw[apos] |= (ci - c0) << kClsShift;
                }
                before += __popc(bnd[k]);
            }
            if (lane < ndev) meta[meta_cls(ndev, lane + 1)] = (uint16_t)cincl;
        }
    }
    if (L.need_tbl) {
        // fit table: requests ascending; T[r] = positions of the r smallest,
        // kept at every 4th rank plus the rank -> position list
        uint8_t* s_por = ws + L.off_por + g * SS::POR;
        uint8_t* s_lt = ws + L.off_lt + g * SS::LTB;
        uint64_t* s_t4 = reinterpret_cast<uint64_t*>(ws + L.off_tbl) + g * SS::T4;
        uint64_t mk[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const uint32_t e = (uint32_t)k * 32u + lane;
            mk[k] = memk[k] != ~0u ? (((uint64_t)memk[k] << 8) | e) : kInf;
        }
        uint32_t mmax = 0;
#pragma unroll
        for (int k = 0; k < K; k++) mmax = max(mmax, memk[k] != ~0u ? memk[k] : 0u);
        warp_sort_keys<K>(mk, __reduce_max_sync(FULL, mmax) < (1u << 24), lane);
        // rank lookup: LtBuckets buckets spread linearly over [lo, hi]
        uint32_t mx = 0, mn = ~0u;
#pragma unroll
        for (int k = 0; k < K; k++) {
            mx = max(mx, memk[k] != ~0u ? memk[k] : 0u);
            mn = min(mn, memk[k]);
        }
        mx = __reduce_max_sync(FULL, mx);
        mn = __reduce_min_sync(FULL, mn);
        if (mn > mx) mn = mx;  // empty trace
        const uint64_t sc = ((uint64_t)LtBuckets<FS>::v << 32) / ((uint64_t)(mx - mn) + 1ull);
        const uint32_t scale = sc > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)sc;
        uint64_t carry[NW];
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) carry[w] = 0;
        uint32_t bk1[K];  // per rank: its bucket + 1
#pragma unroll
        for (int k = 0; k < K; k++) {
            const uint32_t r = (uint32_t)k * 32u + lane;
            const bool valid = mk[k] != kInf;
            s_por[r] = valid ? (uint8_t)(mk[k] & 0xFFu) : (uint8_t)N;
            // prefix OR over ranks, word by word: v = T[r + 1]
            const uint32_t pos = (uint32_t)mk[k] & 0xFFu;
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) {
                uint64_t v = valid && (pos >> 6) == w ? (1ull << (pos & 63u)) : 0ull;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t u = shfl_up_u64(v, o);
                    if (lane >= (uint32_t)o) v |= u;
                }
                v |= carry[w];
                if ((r + 1u) % FS == 0) s_t4[((r + 1) / FS) * NW + w] = v;
                carry[w] = __shfl_sync(FULL, (uint32_t)v, 31) |
                           ((uint64_t)__shfl_sync(FULL, (uint32_t)(v >> 32), 31) << 32);
            }
            // bucket of rank r, + 1 (LB + 1 past the valid ranks)
            bk1[k] = valid ? lt_bucket<FS>((uint32_t)(mk[k] >> 8) - mn, scale) + 1u : LtBuckets<FS>::v + 1u;
        }
        // LT[j] = first rank whose bucket is >= j = #ranks with bucket < j:
        // the last rank r of each bucket value leaves r + 1 at index
        // bucket + 1, and a prefix maximum over the buckets fills the rest
        // (no loop whose trip count varies across lanes)
        {
            constexpr uint32_t LB = LtBuckets<FS>::v, CH = LB / 32u;
            static_assert(LB % 32u == 0, "buckets per lane");
            uint8_t* lt = s_lt + lane * CH;
#pragma unroll
            for (uint32_t c = 0; c < CH; c++) lt[c] = 0;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < K; k++) {
                const uint32_t r = (uint32_t)k * 32u + lane;
                uint32_t bn = __shfl_down_sync(FULL, bk1[k], 1);
                const uint32_t nx = __shfl_sync(FULL, bk1[k + 1 < K ? k + 1 : k], 0);
                if (lane == 31) bn = k + 1 < K ? nx : LB + 1u;
                if (bn != bk1[k] && bk1[k] < LB) s_lt[bk1[k]] = (uint8_t)(r + 1u);
            }
            __syncwarp();
            uint32_t v[CH], m = 0;
#pragma unroll
            for (uint32_t c = 0; c < CH; c++) {
                m = max(m, (uint32_t)lt[c]);
                v[c] = m;
            }
            uint32_t x = m;  // inclusive max scan over the lanes' chunks
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(FULL, x, o);
                if (lane >= (uint32_t)o) x = max(x, u);
            }
            uint32_t ex = __shfl_up_sync(FULL, x, 1);
            if (lane == 0) ex = 0;
#pragma unroll
            for (uint32_t c = 0; c < CH; c++) lt[c] = (uint8_t)max(v[c], ex);
        }
        if (!narrow && ndev == 1) {
            // busy apps at once <= apps without a request + the most requests
            // that fit the device together (the k smallest): ranks whose
            // prefix sum of sorted requests is <= cap.  Above the main
            // pass's 64-bit heap, the trace goes to the retry pass directly.
            uint64_t run = 0;
            uint32_t fit = 0;
#pragma unroll
            for (int k = 0; k < K; k++) {
                uint64_t v = mk[k] != kInf ? (mk[k] >> 8) : (uint64_t)0xFFFFFFFFu;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t u = shfl_up_u64(v, o);
                    if (lane >= (uint32_t)o) v += u;
                }
                v += run;
                fit += __popc(__ballot_sync(FULL, v <= P.cap[0]));
                run = __shfl_sync(FULL, (uint32_t)v, 31) | ((uint64_t)__shfl_sync(FULL, (uint32_t)(v >> 32), 31) << 32);
            }
            wide_big = fit > kLaneHeapW;
        }
        if (lane < NW) s_t4[lane] = 0ull;
        if (lane == 0) {
            uint32_t* prm = reinterpret_cast<uint32_t*>(s_lt + LtBuckets<FS>::v);
            prm[0] = mn;
            prm[1] = mx;
            prm[2] = scale;
            s_mem[N] = ~0u;
        }
        if (lane < 4) s_por[N + lane] = (uint8_t)N;
    }
    if (lane < ndev) {
        meta[meta_dev(lane + 1)] = (uint16_t)dincl;
        meta[meta_z(ndev, lane)] = (uint16_t)z_d;
    }
    if (ndev > 1) {
        bad_dev = __any_sync(FULL, bad_dev);
        if (lane == 0) meta[meta_baddev(ndev)] = bad_dev ? 1u : 0u;
    }
    if (lane == 0) {
        meta[0] = (uint16_t)na;
        meta[1] = (uint16_t)fail;
        meta[2] = narrow ? 1u : wide_big ? 2u : 0u;  // 32-bit keys / 64-bit, retry pass / 64-bit
        meta[meta_dev(0)] = 0;
        meta[meta_cls(ndev, 0)] = 0;
    }
    __syncwarp();
}

// One lane's simulation of (trace t, device d, policy slot pslot) from the
// staged slot g with a heap of HW 64-bit keys (or kLaneHeapN 32-bit keys).
// Returns false if the lane must be re-run (retry pass / fallback).
// kLaneSync: the lanes re-converge at a ballot every iteration
// (LaneSim's SY; the lane256 kernel needs it, here it is measured)
constexpr bool kLaneSync = false;

template <int K, uint32_t FS, bool NARROW, uint32_t HW = kLaneHeapW>
__device__ __forceinline__ bool lane_run(const LaneParams& L, uint8_t* ws, const uint16_t* meta, uint32_t g,
                                         uint32_t d, uint32_t pslot, uint32_t policy, uint32_t cap_d,
                                         uint64_t t, uint32_t lane, uint32_t runmask) {
    const SimParams& P = L.sp;
    constexpr uint32_t N = 32u * K;
    constexpr uint32_t NW = (N + 63u) / 64u;
    using SS = SlotStride<N, FS>;
    const uint32_t na = meta[0];
    const uint32_t ndev = P.ndev;
    const uint32_t s0 = meta[meta_dev(d)], s1 = meta[meta_dev(d + 1)], z = meta[meta_z(ndev, d)];
    uint64_t a0;
    uint32_t na_unused;
    lane_trace_range(P, t, a0, na_unused);
    LaneSim<K, NARROW, HW, FS, (K <= 4), kLaneSync> sim(P);
    sim.smask = runmask;
    sim.s_a = reinterpret_cast<const uint32_t*>(ws + L.off_a) + g * SS::S32;
    sim.s_mem = reinterpret_cast<const uint32_t*>(ws + L.off_mem) + g * SS::S32;
    sim.s_bw = reinterpret_cast<const uint32_t*>(ws + L.off_bw) + g * SS::S32;
    sim.s_por = ws + L.off_por + g * SS::POR;
    sim.s_lt = ws + L.off_lt + g * SS::LTB;
    sim.lt_lo = reinterpret_cast<const uint32_t*>(sim.s_lt + LtBuckets<FS>::v)[0];
    sim.lt_hi = reinterpret_cast<const uint32_t*>(sim.s_lt + LtBuckets<FS>::v)[1];
    sim.lt_scale = reinterpret_cast<const uint32_t*>(sim.s_lt + LtBuckets<FS>::v)[2];
    sim.s_t4 = reinterpret_cast<const uint64_t*>(ws + L.off_tbl) + g * SS::T4;
    uint32_t c0 = 0, c1 = 0;
    if (L.need_cls) { c0 = meta[meta_cls(ndev, d)]; c1 = meta[meta_cls(ndev, d + 1)]; }
    sim.s_cm = reinterpret_cast<const uint64_t*>(ws + L.off_cm) + g * (L.cm_per_trace * NW) + c0 * NW;
    sim.ncls = c1 - c0;
    sim.heap = reinterpret_cast<typename LaneSim<K, NARROW, HW, FS, (K <= 4), kLaneSync>::Key*>(ws + L.off_fb) + lane;
    const uint64_t out_base = (uint64_t)pslot * P.n_apps_total + a0;
    sim.gp = P.grant ? reinterpret_cast<uint32_t*>(P.grant) + out_base : nullptr;
    sim.ep = P.end ? reinterpret_cast<uint32_t*>(P.end) + out_base : nullptr;
    if (!sim.run(na, s0, s1, z, policy, cap_d)) return false;
    // S = cpu + busy ticks of the lane's device range (arrival < 2^31 and
    // busy < 2^21 on this path), only when the speed-up is requested
    uint64_t seq = 0;
    if (P.speedup)
        for (uint32_t q = s0; q < s1; q++) seq += (uint64_t)sim.s_a[q] + bw_busy(sim.s_bw[q]);
    const uint32_t st = ndev > 1 && meta[meta_baddev(ndev)] ? SG_ST_BAD_DEVICE : 0u;
    sim.finish(((uint64_t)pslot * P.n_traces + t) * P.ndev + d, s1 - s0, st, seq);
    return true;
}

// Main pass: pre-write the group's output rows with full-sector stores
// (groups of >= 4 traces).  C2: DRAM traffic 7.48 -> 4.35 GB per launch
// (reads 3.16 -> 1.25 GB: no sector fills) for +0.7 % time; with one trace
// per warp (C5) it cost 7.7 % and is off (profiles/r02_prewrite_ab.txt).
constexpr bool kPrewriteRows = true;

// Main pass (RETRY = false): every trace in order.  A trace whose 64-bit-key
// lanes overflow their heap (kLaneHeapW events), or could (its staged
// busy-app bound exceeds kLaneHeapW: meta[2] == 2), is appended to P.retry.
// Retry pass: the traces of P.retry (count P.work[2]) with 64-bit keys and a
// heap of kLaneHeapN events in a larger warp region.  Other failed lanes
// (32-bit-key heap or wake FIFO full, staging limits) are re-run in-kernel
// by the warp-per-trace fallback.
template <int K, bool RETRY, int MB, uint32_t FS>
__global__ void __launch_bounds__(kLaneWarpsPerBlock * 32, MB) trace_sim_lane_kernel(const LaneParams L) {
    const SimParams& P = L.sp;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * L.warp_bytes;
    const uint64_t n_items = RETRY ? *reinterpret_cast<volatile unsigned long long*>(P.work + 2) : P.n_traces;
    const uint64_t n_groups = (n_items + L.G - 1) / L.G;
    auto trace_of = [&](uint64_t i) -> uint64_t { return RETRY ? (uint64_t)P.retry[i] : i; };
    const uint32_t ndev = P.ndev;
    // groups are handed out by one atomic counter (each warp takes the next
    // group when it finishes one): no tail of warps with more groups than
    // others (sgpu_common.cuh work_fetch / work_done)
    auto fetch = [&]() -> uint64_t { return work_fetch(P.work, lane); };

    // lane -> (slot, device, policy slot)
    const uint32_t g = lane / L.lpt;
    const uint32_t rem = lane - g * L.lpt;
    const uint32_t d = rem / P.npol;
    const uint32_t pslot = rem - d * P.npol;
    const uint32_t policy = (P.policy_list >> (4 * pslot)) & 0xFu;
    uint32_t cap_d = P.cap[0];
#pragma unroll
    for (uint32_t j = 1; j < SG_MAX_DEV; j++)
        if (d == j) cap_d = P.cap[j];

    uint64_t grp = fetch();
    while (grp < n_groups) {
        const uint64_t next = fetch();
        const uint64_t t0 = grp * L.G;
        const uint32_t gcount = (uint32_t)min((uint64_t)L.G, n_items - t0);
        for (uint32_t s = 0; s < gcount; s++) stage_trace<K, FS>(L, ws, s, trace_of(t0 + s), lane);
        // warm L2 with the next group's records while this one simulates
        if (!RETRY && next < n_groups && !P.trace_offsets) {
            const uint64_t nt0 = next * L.G;
            const uint64_t nb = min((uint64_t)L.G, P.n_traces - nt0) * P.apps_per_trace * 16u;
            const uint8_t* base = reinterpret_cast<const uint8_t*>(P.apps + nt0 * P.apps_per_trace);
            for (uint64_t off = (uint64_t)lane * 128u; off < nb; off += 32u * 128u) prefetch_l2(base + off);
        }

        if (!RETRY && kPrewriteRows && L.G >= 4u && P.grant && P.end && !P.trace_offsets) {
            // the group's grant / end rows written whole first (coalesced
            // 16-byte stores of SG_NEVER): the lanes' later per-app stores
            // then land in fully written L2 sectors instead of partial ones
            // that cost a DRAM read to fill (every entry is overwritten by
            // the lanes, the fallback or the retry pass)
            const uint64_t a0g = t0 * P.apps_per_trace;
            const uint32_t span = gcount * P.apps_per_trace;
            if (((a0g | span | P.n_apps_total) & 3u) == 0 &&
                ((reinterpret_cast<uintptr_t>(P.grant) | reinterpret_cast<uintptr_t>(P.end)) & 15u) == 0) {
                const uint4 nv = make_uint4(SG_NEVER, SG_NEVER, SG_NEVER, SG_NEVER);
                for (uint32_t x = 0; x < 2u * P.npol; x++) {
                    const uint32_t arr = x >= P.npol ? 1u : 0u, p = x - arr * P.npol;
                    uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(arr ? P.end : P.grant) +
                                                         (uint64_t)p * P.n_apps_total + a0g);
                    for (uint32_t j = lane; j < span / 4u; j += 32u) d4[j] = nv;
                }
            }
        }
        bool fail = false, defer = false;
        const uint16_t* meta = reinterpret_cast<const uint16_t*>(ws + L.off_meta) + g * L.meta_stride;
        const uint64_t my_t = trace_of(t0 + min(g, gcount - 1));
        // 32-bit event keys when every trace of the group allows them (warp-uniform)
        const bool narrow = !RETRY && __all_sync(FULL, g >= gcount || meta[2] == 1);
        // the lanes that enter a LaneSim main loop (for kLaneSync)
        const uint32_t runmask =
            __ballot_sync(FULL, g < gcount && !meta[1] && (RETRY || narrow || meta[2] != 2));
        if (g < gcount) {
            if (meta[1])
                fail = true;
            else if (RETRY)
                fail = !lane_run<K, FS, false, kLaneHeapN>(L, ws, meta, g, d, pslot, policy, cap_d, my_t, lane, runmask);
            else if (narrow)
                fail = !lane_run<K, FS, true>(L, ws, meta, g, d, pslot, policy, cap_d, my_t, lane, runmask);
            else if (meta[2] == 2)
                defer = true;
            else
                defer = !lane_run<K, FS, false>(L, ws, meta, g, d, pslot, policy, cap_d, my_t, lane, runmask);
        }
        if (!RETRY) {
            // a trace with a failed lane goes to the retry pass whole: one
            // entry per trace, appended by its slot's first lane
            const uint32_t any = __ballot_sync(FULL, defer);
            const uint32_t smask = L.lpt >= 32u ? ~0u : (1u << L.lpt) - 1u;
            const bool dslot = ((any >> (g * L.lpt)) & smask) != 0 && g < gcount;
            fail = fail && !dslot;  // the retry pass re-runs every lane of a deferred trace
            const uint32_t dm = __ballot_sync(FULL, dslot && rem == 0);
            if (dm) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(P.work + 2, (unsigned long long)__popc(dm));
                base = __shfl_sync(FULL, base, 0);
                if (dm >> lane & 1u) P.retry[base + __popc(dm & lanemask_lt())] = (uint32_t)my_t;
            }
        }
        __syncwarp();
        // exact fallback: the whole warp re-simulates each failed lane
        for (uint32_t fm = __ballot_sync(FULL, fail); fm; fm &= fm - 1) {
            const uint32_t fl = __ffs(fm) - 1;
            const uint32_t fg = fl / L.lpt;
            const uint32_t frem = fl - fg * L.lpt;
            const uint32_t fd = frem / P.npol;
            const uint32_t fp = frem - fd * P.npol;
            const uint64_t t = trace_of(t0 + fg);
            uint64_t a0;
            uint32_t na;
            lane_trace_range(P, t, a0, na);
            uint8_t* fb = ws;  // the whole warp region: the group's lane simulations are done
            uint4* apps_s = reinterpret_cast<uint4*>(fb + P.off_app);
            for (uint32_t i = lane; i < na; i += 32)
                apps_s[i] = __ldg(reinterpret_cast<const uint4*>(P.apps + a0) + i);
            __syncwarp();
            const uint4* sub = apps_s;
            const uint16_t* idx = nullptr;
            uint32_t nd = na;
            bool bad_dev = false;
            if (ndev > 1) {
                uint4* s_sub = reinterpret_cast<uint4*>(fb + P.off_sub);
                uint16_t* s_idx = reinterpret_cast<uint16_t*>(fb + P.off_idx);
                nd = build_subtrace(apps_s, na, fd, ndev, s_sub, s_idx, lane, bad_dev);
                sub = s_sub;
                idx = s_idx;
            }
            uint32_t fcap = P.cap[0];
#pragma unroll
            for (uint32_t j = 1; j < SG_MAX_DEV; j++)
                if (fd == j) fcap = P.cap[j];
            TraceSim<TickTM, K, false, false> sim(P, lane, fb, sub);
            sim.run(nd, (P.policy_list >> (4 * fp)) & 0xFu, fcap, nullptr);
            if (bad_dev) sim.status |= SG_ST_BAD_DEVICE;
            sim.finish(((uint64_t)fp * P.n_traces + t) * ndev + fd, (uint64_t)fp * P.n_apps_total + a0,
                       idx, nullptr);
        }
        __syncwarp();
        grp = next;
    }
    work_done(P.work, lane, RETRY);
}

static inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }


// Lane path eligibility: T0 ticks mode, no event log, <= 256 apps per trace,
// < 2^32 traces.
// By default traces of <= 128 apps take it (measured on one B200: C4, 128
// apps, 4 policies: 4.1e7 vs 1.4e7 trace-sims/s on the warp kernel);
// 256-app traces are faster on the warp kernel (C3: 3.6e6 vs 1.3e6) unless
// `forced`.
bool lane_eligible(const SimParams& p, bool program_mode, bool f64, bool forced) {
    if (program_mode || f64 || p.events != nullptr || p.npol * p.ndev > 32) return false;
    if (p.n_traces > 0xFFFFFFFFull) return false;  // deferred-trace ids are 32-bit
    if (forced) return p.n_pad <= 256u;
    // one simulation per 128-app trace leaves 7 of 8 lanes of a trace slot
    // idle: the warp kernel is faster there (C4 shape, 1 policy: 38-59 vs
    // 98 ms per 1M traces)
    return p.n_pad <= 64u || (p.n_pad <= 128u && p.npol * p.ndev >= 2);
}

// Grid of one lane-kernel instantiation for L (cached attributes/occupancy).
template <int K, bool RETRY, int MB, uint32_t FS>
static cudaError_t lane_grid(const LaneParams& L, uint64_t* grid) {
    const uint32_t wpb = kLaneWarpsPerBlock;
    const size_t smem = (size_t)L.warp_bytes * wpb;
    int sms = 0, per_sm = 0;
    const cudaError_t err = kernel_config(reinterpret_cast<const void*>(trace_sim_lane_kernel<K, RETRY, MB, FS>),
                                          wpb * 32, smem, &per_sm, &sms);
    if (err != cudaSuccess) return err;
    const uint64_t groups = (L.sp.n_traces + L.G - 1) / L.G;
    const uint64_t need = (groups + wpb - 1) / wpb;
    uint64_t g = (uint64_t)sms * per_sm;
    if (need < g) g = need;
    *grid = g == 0 ? 1 : g;
    return cudaSuccess;
}

// Main pass + retry pass of one variant.  Both configurations are checked
// before the main pass launches: a main pass whose retry pass cannot run
// would leave its deferred-trace count behind.
template <int K, int MB, int MBR, uint32_t FS>
static cudaError_t launch_pair(LaneParams& L, LaneParams& R, cudaStream_t stream, int* grid_out) {
    uint64_t gm = 0, gr = 0;
    cudaError_t err = lane_grid<K, false, MB, FS>(L, &gm);
    if (err == cudaSuccess) err = lane_grid<K, true, MBR, FS>(R, &gr);
    if (err != cudaSuccess) return err;
    if (grid_out) *grid_out = (int)gm;
    const unsigned threads = kLaneWarpsPerBlock * 32;
    trace_sim_lane_kernel<K, false, MB, FS><<<(unsigned)gm, threads, (size_t)L.warp_bytes * kLaneWarpsPerBlock, stream>>>(L);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    trace_sim_lane_kernel<K, true, MBR, FS><<<(unsigned)gr, threads, (size_t)R.warp_bytes * kLaneWarpsPerBlock, stream>>>(R);
    err = cudaGetLastError();
    if (err != cudaSuccess) {
        // the main pass may have deferred traces: clear the count for the
        // stream's next launch
        cudaMemsetAsync(L.sp.work + 2, 0, sizeof(unsigned long long), stream);
    }
    return err;
}

// Per-warp shared-memory layout of the lane kernel; `heap_bytes` is the
// busy-end heap region of the warp's 32 lanes, `fs` the fit-table stride.
static void lane_layout(LaneParams& L, uint32_t heap_bytes, uint32_t fs) {
    const uint32_t N = L.sp.n_pad;
    const uint32_t NW = (N + 63u) / 64u;
    // the heaps and the staging scratch share one region; the fallback
    // TraceSim overlays the whole warp region once the group's lanes are done
    const uint32_t fb = max(heap_bytes, N * 16u);
    const uint32_t LB = fs == 2 ? LtBuckets<2>::v : LtBuckets<4>::v;
    const uint32_t S32 = N + 1, POR = N + 4, LTB = LB + 12, T4 = (N / fs + 1) * NW;  // SlotStride<N, fs>
    L.meta_stride = meta_u16(L.sp.ndev);
    uint32_t o = 0;
    L.off_a = o;
    o = align16(o + L.G * S32 * 4u);
    L.off_mem = o;
    o = align16(o + L.G * S32 * 4u);
    L.off_bw = o;
    o = align16(o + L.G * S32 * 4u);
    L.off_por = o;
    o = align16(o + (L.need_tbl ? L.G * POR : 0u));
    L.off_lt = o;
    o = align16(o + (L.need_tbl ? L.G * LTB : 0u));
    L.off_tbl = o;
    o = align16(o + (L.need_tbl ? L.G * T4 * 8u : 0u));
    L.off_cm = o;
    o = align16(o + (L.need_cls ? L.G * (L.cm_per_trace * NW) * 8u : 0u));
    L.off_meta = o;
    o = align16(o + L.G * L.meta_stride * 2u);
    L.off_fb = o;
    o = align16(o + fb);
    L.warp_bytes = max(o, align16(L.sp.warp_bytes));
    if (const char* pad = getenv("SGPU_LANE_SMEM_PAD")) L.warp_bytes += align16((uint32_t)atoi(pad));  // occupancy experiments
}

// Main pass + retry pass.  The variant: at 64 apps with few traces per warp
// (shared memory allows >= kLaneHiBlocks2 blocks with the 4-stride table)
// the ten-block, 4-stride build; otherwise LaneMinBlocks with FitStride<K>.
template <int K>
static cudaError_t launch_lane_k(LaneParams& L, LaneParams& R, cudaStream_t stream, int* grid_out) {
    const uint32_t HB = max(kLaneHeapN * 32u * 4u, kLaneHeapW * 32u * 8u);  // main pass heap region
    const uint32_t HBR = kLaneHeapN * 32u * 8u;                          // retry pass: 64-bit keys
    if constexpr (K == 2) {
        lane_layout(L, HB, 4u);
        // blocks per SM that shared memory allows (228 KB, 1 KB reserved per block)
        const uint32_t smem_blocks = 233472u / (L.warp_bytes * kLaneWarpsPerBlock + 1024u);
        if (smem_blocks >= (uint32_t)kLaneHiBlocks2) {
            lane_layout(R, HBR, 4u);
            return launch_pair<K, kLaneHiBlocks2, LaneMinBlocksR<K>::v, 4u>(L, R, stream, grid_out);
        }
        // nine blocks (18 warps) with the 4-stride table (12.2 KB per warp,
        // 96 registers) beat eight with the 2-stride one (13.4 KB): C2
        // 13.65 -> 13.57 ms (profiles/r02_b9_ab.txt)
        if (smem_blocks >= 9u) {
            lane_layout(R, HBR, 4u);
            return launch_pair<K, 9, LaneMinBlocksR<K>::v, 4u>(L, R, stream, grid_out);
        }
    }
    constexpr uint32_t FS = FitStride<K>::v;
    lane_layout(L, HB, FS);
    lane_layout(R, HBR, FS);
    return launch_pair<K, LaneMinBlocks<K>::v, LaneMinBlocksR<K>::v, FS>(L, R, stream, grid_out);
}

cudaError_t launch_sim_lane(const SimParams& p, cudaStream_t stream, int* grid_out) {
    if (p.n_traces > 0xFFFFFFFFull) return cudaErrorInvalidValue;  // 32-bit deferred-trace ids
    LaneParams L;
    L.sp = p;
    const uint32_t N = p.n_pad;
    L.lpt = p.npol * p.ndev;
    // at most 8 traces per warp: the shared slot of a trace is what limits
    // residency, so fewer simulations per trace (npol * ndev < 4) leave lanes
    // idle rather than multiply the warp's shared memory
    L.G = min(32u / L.lpt, 8u);
    L.need_cls = 0;
    for (uint32_t i = 0; i < p.npol; i++) {
        const uint32_t pol = (p.policy_list >> (4 * i)) & 0xFu;
        if (pol >= SG_POLICY_PFIFO) L.need_cls = 1;
    }
    L.need_tbl = N <= 128 ? 1u : 0u;  // all kinds use the fit table (one or two mask words)
    L.cm_per_trace = max(kLaneClassMasks / L.G, 8u);
    sim_layout(L.sp, false, false);
    WorkLease lease;
    cudaError_t err = work_counters(stream, L.sp, p.n_traces, lease);
    if (err == cudaSuccess) {
        LaneParams R = L;
        switch (N / 32) {
            case 1: err = launch_lane_k<1>(L, R, stream, grid_out); break;
            case 2: err = launch_lane_k<2>(L, R, stream, grid_out); break;
            case 4: err = launch_lane_k<4>(L, R, stream, grid_out); break;
            case 8: err = launch_lane_k<8>(L, R, stream, grid_out); break;
            default: err = cudaErrorInvalidValue;
        }
    }
    return work_release(stream, lease, err);
}

cudaError_t lane_warps_per_sm(int* warps) {
    SimParams p;
    memset(&p, 0, sizeof(p));
    p.n_traces = 1u << 20;
    p.apps_per_trace = 64;
    p.n_pad = 64;
    p.npol = 4;
    p.policy_list = 0x3210u;
    p.ndev = 1;
    LaneParams L;
    L.sp = p;
    L.lpt = 4;
    L.G = 8;
    L.need_cls = 1;
    L.need_tbl = 1;
    L.cm_per_trace = max(kLaneClassMasks / L.G, 8u);
    sim_layout(L.sp, false, false);
    const uint32_t HB = max(kLaneHeapN * 32u * 4u, kLaneHeapW * 32u * 8u);
    lane_layout(L, HB, FitStride<2>::v);
    int sms = 0, per_sm = 0;
    const cudaError_t err = kernel_config(
        reinterpret_cast<const void*>(trace_sim_lane_kernel<2, false, LaneMinBlocks<2>::v, FitStride<2>::v>),
        kLaneWarpsPerBlock * 32, (size_t)L.warp_bytes * kLaneWarpsPerBlock, &per_sm, &sms);
    *warps = err == cudaSuccess ? per_sm * kLaneWarpsPerBlock : 0;
    return err;
}

}  // namespace sg
