// sgpu_lanesim.cuh — the per-lane simulation of K1 v5 (LaneSim): one
// (trace, device, policy) simulated by one thread from a staged trace slot.
// Included by sgpu_lane.cu (device code) and, with the shims below, compiled
// by the host C++ compiler for tests/test_lanesim_host.py, which checks this
// exact decision logic against the oracle on CPU.  Semantics: see the header
// of sgpu_lane.cu and SURVEY.md Appendix A.
#pragma once

#include <cstdint>
#include <type_traits>

#ifdef __CUDACC__
#include "sgpu_tracesim.cuh"
#define SG_HD __device__ __forceinline__
#else
// host build: plain C++ (the only intrinsic used is find-first-set)
#include <algorithm>
#include "../../include/sgpu.h"
#define SG_HD inline
namespace sg {
using std::max;
using std::min;
struct SimParams {  // the two output arrays LaneSim writes
    void* grant;
    void* end;
};
inline int __ffsll(long long x) { return __builtin_ffsll(x); }
inline int __ffs(int x) { return __builtin_ffs(x); }
}  // namespace sg
#endif

// Host-side instrumentation point (loop iterations per simulation, used by
// profiling tools that compile LaneSim on the host); empty otherwise.
#ifndef SG_LANE_ITER_HOOK
#define SG_LANE_ITER_HOOK(granting)
#endif

namespace sg {

constexpr uint32_t kLaneHeapN = 20;         // busy-end heap slots per lane: 4-ary, depth 2
constexpr uint32_t kLaneHeapW = 10;         // the same 2.5 KB region with 64-bit keys (main pass)
// Fit table T[r] kept at every FS-th rank: every 2nd at <= 64 apps (one
// extra position to OR in; fits C2's shared budget), every 4th above and in
// the few-traces-per-warp variant (its staging is a larger share).
template <int K> struct FitStride { static constexpr uint32_t v = K <= 2 ? 2u : 4u; };
constexpr uint64_t kInf = ~0ull;
// rank-lookup buckets per trace, with the fit-table stride FS: 192 with the
// 2-stride table (<= 64 apps: fewer requests per bucket to scan; C2 17.89 ->
// 17.81 ms), 128 with the 4-stride one (C4's shared budget; C5's staging)
template <uint32_t FS> struct LtBuckets { static constexpr uint32_t v = FS == 2 ? 192u : 128u; };
constexpr uint32_t kBusyBits = 21;          // busy < 2^21 on this path; app index above it
constexpr uint32_t kClsShift = 29;          // s_bw bits 29-31: priority class of the app within its device
constexpr uint32_t kLaneMaxCls = 8;         // classes per device on this path (more: warp-kernel re-run)

constexpr uint32_t kLtSat = (1u << 23) - 1u;  // packed bucket entry: request field saturated
SG_HD uint32_t bw_busy(uint32_t bw) { return bw & ((1u << kBusyBits) - 1u); }
SG_HD uint32_t bw_app(uint32_t bw) { return (bw >> kBusyBits) & 0xFFu; }
SG_HD uint32_t bw_cls(uint32_t bw) { return bw >> kClsShift; }


// Member arrays (mask, gcand, grem, the fit set) are only ever updated with
// unconditional per-word selects: a predicated store `if (w == q >> 6)
// m[w] |= ...` is merged by the compiler into one dynamically indexed store,
// which moves the whole LaneSim (and a copy of the kernel parameters) to
// local memory (K = 4: a 624-byte stack frame).
SG_HD uint32_t ffs64(uint64_t x) { return (uint32_t)__ffsll((long long)x) - 1u; }
SG_HD uint32_t ffs32(uint32_t x) { return (uint32_t)__ffs((int)x) - 1u; }

// Rank-lookup bucket of a request d = mem - lo >= 0: monotone in d.
template <uint32_t FS> SG_HD uint32_t lt_bucket(uint32_t d, uint32_t scale) {
    return min((uint32_t)(((uint64_t)d * scale) >> 32), LtBuckets<FS>::v - 1u);
}

template <int K> struct LogN { static constexpr uint32_t v = K == 1 ? 5 : K == 2 ? 6 : K == 4 ? 7 : 8; };

// Event keys (t, virtual counter, position).  NARROW: one u32, t << (2 LOGN
// + 1) | counter << LOGN | q, usable when every event time of the trace is
// below LIM = 2^(31 - 2 LOGN) - 1 (arrival max + busy sum, checked at
// staging).  Each app pushes at most one busy end, so the counter of
// the initial pop of app i is i and later pushes count up from N (< 2N).
// Wide: one u64, t << 32 | counter << 8 | q with the block counters
// described above.  HW: heap capacity with 64-bit keys.
template <int K, bool NARROW, uint32_t HW = kLaneHeapW> struct LaneKey {
    static constexpr uint32_t LOGN = LogN<K>::v;
    using T = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    static constexpr uint32_t QB = NARROW ? LOGN : 8u;
    static constexpr uint32_t TS = NARROW ? 2u * LOGN + 1u : 32u;
    static constexpr T INF = (T)~(T)0;
    // heap capacity: kLaneHeapN with 32-bit keys (or HW if larger), HW with
    // 64-bit keys
    static constexpr uint32_t HCAP = NARROW ? (HW > kLaneHeapN ? HW : kLaneHeapN) : HW;
    static constexpr uint32_t LIM = NARROW ? (1u << (32u - TS)) - 1u : ~0u;
    static constexpr uint32_t CMAX = NARROW ? 2u << LOGN : 1u << 24;  // counters must stay below
    static SG_HD T make(uint32_t t, uint32_t c, uint32_t q) {
        return ((T)t << TS) | ((T)c << QB) | (T)q;
    }
    static SG_HD uint32_t time(T k) { return (uint32_t)(k >> TS); }
    static SG_HD uint32_t pos(T k) { return (uint32_t)k & ((1u << QB) - 1u); }
    // counter of the initial pop of app i / first counter of later pushes
    static SG_HD uint32_t c_init(uint32_t i) { return NARROW ? i : i << LOGN; }
    static SG_HD uint32_t c_base(uint32_t n) { return NARROW ? 32u * K : n << LOGN; }
};

template <int K, bool NARROW, uint32_t HW = kLaneHeapW, uint32_t FSt = FitStride<K>::v, bool TB = (K <= 4),
          bool SY = false, uint32_t LBt = LtBuckets<FSt>::v, uint32_t RS = 1>
struct LaneSim {
    static constexpr uint32_t N = 32u * K;
    static constexpr uint32_t NW = (N + 63u) / 64u;  // queue mask words
    static constexpr uint32_t LOGN = LogN<K>::v;
    // fit table (one to four mask words): up to 128 apps in the lane kernel,
    // 256 in the global-table kernel (sgpu_lane256.cu); else a queue scan
    static constexpr bool TBL = TB;
    using KY = LaneKey<K, NARROW, HW>;
    using Key = typename KY::T;
    // rank / position tables: u8 up to 128 apps, u16 at 256 (rank N = 256)
    using PT = typename std::conditional<(K > 4 && TB), uint16_t, uint8_t>::type;
    // heaps of more than 21 keys sift over three levels (root + 4 + 16 + 64)
    static constexpr bool DEEP = KY::HCAP > 21;
    // SY: the lanes running the main loop (smask, set by the caller) meet
    // at a ballot at the end of every iteration, so they re-converge per
    // event (without it the 256-app instantiation let lanes drift into
    // different iterations: 3 active lanes per instruction)
    uint32_t smask;
    SG_HD void sync_iter(bool stop) {
#ifdef __CUDACC__
        if constexpr (SY) smask = __ballot_sync(smask, !stop);
#endif
        (void)stop;
    }

    const SimParams& P;
    // trace slot (shared by the trace's lanes), arrival-position order
    const uint32_t* s_a;     // arrival tick
    // RS: record stride in u32 (2: request and busy word of a position
    // interleaved, s_bw = s_mem + 1, so a position's pair is one sector)
    const uint32_t* s_mem;   // request MiB
    const uint32_t* s_bw;    // busy | app << kBusyBits | class << kClsShift
    const PT* s_por;         // position of the r-th smallest request (N past the end)
    const PT* s_lt;          // s_lt[j] = #requests in buckets < j (LBt buckets)
    const uint32_t* s_ms;    // requests in rank order (s_ms[N] = ~0), or nullptr: s_mem[s_por[r]]
    // optional (with s_ms, K > 4): bucket entries packed as request << 9 |
    // rank (kLtSat in the request field: saturated, load s_ms[rank]), so the
    // first scan step needs no load of its own
    const uint32_t* s_lt32;
    uint32_t lt_lo, lt_hi, lt_scale;
    const uint64_t* s_t4;    // T[FS j] (NW words): positions of the FS j smallest requests
    const uint64_t* s_cm;    // class masks (NW words each) of this lane's device, top class first
    uint32_t ncls;
    // this lane's columns
    Key* heap;               // heap[h * 32]
    uint32_t* gp;            // grant / end ticks of app 0 of the trace under this policy
    uint32_t* ep;            // (nullptr: not requested)
    uint32_t cap, used;
    bool prio_pol, mmu, fail;
    uint64_t mask[NW];
    uint32_t hs;
    Key kh;                  // heap top (KY::INF when empty)
    uint32_t counter;        // next virtual counter of a later push (from KY::c_base)
    // statistics (harness.py:373-461 integer forms)
    uint32_t last, mem_t, busy_prev, B;
    uint64_t I;
    int32_t busy_level, holders;
    uint32_t maxh, grants, pops;
    // incremental grant_waiters state (fit-table path): one select_grants
    // step per loop iteration while `gs` (harness.py:545-558)
    bool gs, ginit;          // granting / the next step starts a round
    uint32_t clsmask;        // priority classes with waiting entries (bit c: class c, top = 0)
    uint32_t gc, gbud, gb0, gg;
    uint64_t gcand[NW], grem[NW];  // unscanned candidates / waiting members of the round's class

    SG_HD LaneSim(const SimParams& p) : P(p), s_ms(nullptr), s_lt32(nullptr) {}

    SG_HD void mem_point(uint32_t now) {
        I += (uint64_t)used * (now - mem_t);
        mem_t = now;
    }
    SG_HD void busy_point(uint32_t now, int32_t delta) {
        B += busy_level > 0 ? now - busy_prev : 0u;
        busy_prev = now;
        busy_level += delta;
    }

    // ------------------------------------------------- busy-end heap
    // 4-ary min-heap of at most kLaneHeapN = 20 keys (depth 2: root + 4 + 16
    // slots): every sift is at
    // most two levels, unrolled and predicated, and the four child loads of a
    // level are independent.  Entries: busy ends, and the resumption of a
    // granted waiter without a busy step (its free).
    SG_HD void push(uint32_t t, uint32_t c, uint32_t q) {
        if (hs >= KY::HCAP || c >= KY::CMAX) { fail = true; return; }
        const Key key = KY::make(t, c, q);
        const uint32_t i = hs++;
        // sift up at most two (three) levels: i -> p1 -> p2 (-> p3); the
        // parent loads are issued at once (their indices follow from the size)
        const uint32_t p1 = i > 0 ? (i - 1) >> 2 : 0u;
        const uint32_t p2 = p1 > 0 ? (p1 - 1) >> 2 : 0u;
        const Key k1 = heap[p1 * 32];
        const Key k2 = heap[p2 * 32];
        const bool up1 = i > 0 && key < k1;
        const bool up2 = up1 && p1 > 0 && key < k2;
        if (up1) heap[i * 32] = k1;
        if (up2) heap[p1 * 32] = k2;
        uint32_t dst = up2 ? p2 : (up1 ? p1 : i);
        if constexpr (DEEP) {
            const uint32_t p3 = p2 > 0 ? (p2 - 1) >> 2 : 0u;
            const Key k3 = heap[p3 * 32];
            const bool up3 = up2 && p2 > 0 && key < k3;
            if (up3) heap[p2 * 32] = k3;
            dst = up3 ? p3 : dst;
        }
        heap[dst * 32] = key;
        if (dst == 0) kh = key;
    }
    // min of the (up to) four children c..c+3 of a node; INF past the end
    SG_HD Key min_child(uint32_t c, uint32_t& m) const {
        const Key k0 = c < hs ? heap[c * 32] : KY::INF;
        const Key k1 = c + 1 < hs ? heap[(c + 1) * 32] : KY::INF;
        const Key k2 = c + 2 < hs ? heap[(c + 2) * 32] : KY::INF;
        const Key k3 = c + 3 < hs ? heap[(c + 3) * 32] : KY::INF;
        const bool s01 = k1 < k0;
        const Key x = s01 ? k1 : k0;
        const uint32_t ix = s01 ? c + 1 : c;
        const bool s23 = k3 < k2;
        const Key y = s23 ? k3 : k2;
        const uint32_t iy = s23 ? c + 3 : c + 2;
        const bool sxy = y < x;
        m = sxy ? iy : ix;
        return sxy ? y : x;
    }
    SG_HD void pop() {
        hs -= 1;
        const Key lastk = heap[hs * 32];
        // level 1: children 1..4 of the root
        uint32_t m1;
        const Key k1 = min_child(1u, m1);
        const bool down1 = k1 < lastk;
        // level 2: children of m1 (5..20)
        uint32_t m2;
        const Key k2 = min_child(4u * m1 + 1u, m2);
        const bool down2 = down1 && k2 < lastk;
        heap[0] = down1 ? k1 : lastk;
        if constexpr (DEEP) {  // level 3: children of m2 (21..84)
            uint32_t m3;
            const Key k3 = min_child(4u * m2 + 1u, m3);
            const bool down3 = down2 && k3 < lastk;
            if (down1) heap[m1 * 32] = down2 ? k2 : lastk;
            if (down2) heap[m2 * 32] = down3 ? k3 : lastk;
            if (down3) heap[m3 * 32] = lastk;
        } else {
            if (down1) heap[m1 * 32] = down2 ? k2 : lastk;
            if (down2) heap[m2 * 32] = lastk;
        }
        kh = hs == 0 ? KY::INF : (down1 ? k1 : lastk);
    }

    // ------------------------------------------------- granted waiters
    // grant_waiters pushes each granted waiter at (now, ++counter)
    // (harness.py:558); its entry pops after every entry of tick `now`
    // pushed before it and starts the busy step, which pushes the busy end
    // (harness.py:514-520).  Until that pop, the only other pushes are
    // those of the arrivals of tick `now` still pending (an app that ran
    // inline at t = 0 owns an initial counter, so its busy end can pop
    // before an arrival of the same tick); busy ends push nothing, and other
    // granted waiters come later in grant order.  So the busy end is pushed
    // at grant time, with a counter above those the pending arrivals of the
    // tick may take: the first grant of a tick reserves one counter per
    // pending arrival (cw = counter + R), granted waiters count up from cw,
    // and a push in a later tick starts above both.  The busy start is
    // accounted at `now` (a zero-length busy segment otherwise).  A waiter
    // without a busy step frees when its entry pops: that entry goes into
    // the heap at (now, its counter).  Pending push of this iteration:
    // pp / pt / pc / pq; counters past CMAX send the lane to the fallback.
    bool pp;
    uint32_t pt, pc, pq;
    uint32_t cw, wt;         // next granted-waiter counter / the tick it belongs to
    uint32_t ap, ae;         // arrival stream: next position / end
    Key ka;                  // key of the next arrival (KY::INF: none)
    SG_HD void start_granted(uint32_t q) {
        const uint32_t b = bw_busy(s_bw[(q) * RS]);
        if (b) {
            busy_point(last, +1);
            pops += 1;  // the waiter's own entry
        }
        if (wt != last) {  // first grant of the tick: reserve the pending arrivals' counters
            uint32_t r = 0;
            if (KY::time(ka) == last)  // (rare) arrivals of this tick still pending
                while (ap + r < ae && s_a[ap + r] == last) r += 1;
            cw = max(counter, cw) + r;
            wt = last;
        }
        pp = true;
        pt = last + b;
        pc = cw++;
        pq = q;
    }

    // ------------------------------------------------- wait queue
    SG_HD void enqueue(uint32_t q, uint32_t bw) {
#pragma unroll
        for (uint32_t w = 0; w < NW; w++)
            mask[w] |= w == (q >> 6) ? 1ull << (q & 63u) : 0ull;  // unconditional: no indexed store
        clsmask |= 1u << bw_cls(bw);
    }
    // number of requests <= budget in the trace: bucket lookup (LtBuckets
    // spread linearly over [smallest, largest] request), then a short
    // forward scan of the sorted requests inside the bucket
    SG_HD uint32_t fit_rank(uint32_t budget) const {
        if (budget > lt_hi) return N;
        const uint32_t bi = budget < lt_lo ? 0u
                                           : min((uint32_t)(((uint64_t)(budget - lt_lo) * lt_scale) >> 32), LBt - 1u);
        if constexpr (K > 4 && TB) {
            if (s_lt32) {
                const uint32_t e = s_lt32[bi];
                uint32_t r = e & 0x1FFu;
                const uint32_t v = e >> 9;
                if (v != kLtSat) {
                    if (v > budget) return r;
                    r += 1;
                }
                while (s_ms[r] <= budget) r += 1;
                return r;
            }
        }
        uint32_t r = s_lt[bi];
        if constexpr (K > 4 && TB) {
            if (s_ms) {  // one load per step
                while (s_ms[r] <= budget) r += 1;
                return r;
            }
        }
        while (s_mem[(s_por[r]) * RS] <= budget) r += 1;  // s_mem[N] = ~0 ends the scan
        return r;
    }
    // T[r]: positions of the r smallest requests = T[FS floor(r/FS)] + the
    // positions of the up to FS - 1 ranks after it
    static constexpr uint32_t FS = FSt;
    SG_HD void fit_set(uint32_t r, uint64_t (&t)[NW]) const {
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) t[w] = s_t4[(r / FS) * NW + w];
        if constexpr (FS == 2) {
            const uint32_t p = s_por[r & ~1u];
#pragma unroll
            for (uint32_t w = 0; w < NW; w++)
                t[w] |= (r & 1u) && (NW == 1 || w == (p >> 6)) ? 1ull << (p & 63u) : 0ull;
        } else if constexpr (FS == 8) {
            // the 8 u16 entries from rank r & ~7: one 16-byte chunk (sector)
            const uint64_t* pw = reinterpret_cast<const uint64_t*>(s_por + (r & ~7u));
            const uint64_t w0 = pw[0], w1 = pw[1];
            const uint32_t k = r & 7u;
#pragma unroll
            for (uint32_t j = 0; j < 7; j++) {
                const uint32_t p = (uint32_t)((j < 4 ? w0 : w1) >> (16u * (j & 3u))) & 0xFFFFu;
#pragma unroll
                for (uint32_t w = 0; w < NW; w++)
                    t[w] |= k > j && (NW == 1 || w == (p >> 6)) ? 1ull << (p & 63u) : 0ull;
            }
        } else {
            // the 4 entries from rank r & ~3 in one load (u8: 32 bits, u16: 64)
            using PW = typename std::conditional<sizeof(PT) == 1, uint32_t, uint64_t>::type;
            const PW pw = *reinterpret_cast<const PW*>(s_por + (r & ~3u));
            const uint32_t k = r & 3u;
#pragma unroll
            for (uint32_t j = 0; j < 3; j++) {
                const uint32_t p = (uint32_t)(pw >> (8u * sizeof(PT) * j)) & ((1u << (8u * sizeof(PT))) - 1u);
#pragma unroll
                for (uint32_t w = 0; w < NW; w++)
                    t[w] |= k > j && (NW == 1 || w == (p >> 6)) ? 1ull << (p & 63u) : 0ull;
            }
        }
    }
    SG_HD void grant_one(uint32_t q, uint32_t m, uint32_t& budget, uint32_t& g) {
#pragma unroll
        for (uint32_t w = 0; w < NW; w++)
            mask[w] &= w == (q >> 6) ? ~(1ull << (q & 63u)) : ~0ull;
        budget -= m;
        g += 1;
        start_granted(q);  // several grants per call on this path: push each at once
        push(pt, pc, pq);
        pp = false;
    }

    // grant_waiters (harness.py:545-558) + select_grants (policy.py:52-74)
    SG_HD void grant_waiters() {
        if constexpr (TBL) grant_waiters_tbl();
        else grant_waiters_scan();
    }

    // <= 64 apps: grant_waiters as a sequence of steps, one per loop
    // iteration, so a lane granting several waiters does not hold the whole
    // warp in a nested loop; the lane pops no event until it is done, so the
    // order is the reference's.  One code path for all four kinds keeps the
    // lanes of a warp (mixed policies) converged.  A round: the top class
    // (all waiting entries for FIFO/MMU, policy.py:58-63); a step: fit =
    // cand & T[#requests <= budget]; FIFO takes the head iff it fits, MMU the
    // lowest fit (policy.py:65-73); both continue above the granted position.
    SG_HD void init_round() {
        if (prio_pol) gc = ffs32(clsmask);  // clsmask != 0 whenever the queue is not empty
        bool any = false;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) {
            gcand[w] = mask[w] & (prio_pol ? s_cm[gc * NW + w] : ~0ull);
            grem[w] = gcand[w];
            any = any || gcand[w] != 0;
        }
        gs = any;
        gb0 = gbud = cap - used;
        gg = 0;
    }
    SG_HD void grant_step() {
        // a round starts inside its first step: one code site for init_round
        // whether the round follows a free or a drained class
        if (ginit) {
            ginit = false;
            init_round();
        }
        uint64_t t[NW];
        fit_set(fit_rank(gbud), t);
        if constexpr (NW == 1) {
            const uint64_t fit = gcand[0] & t[0];
            const uint64_t head = gcand[0] & (0ull - gcand[0]);
            const uint64_t pick = mmu ? fit : (fit & head);
            if (pick) {
                const uint32_t q = ffs64(pick);
                const uint64_t bit = 1ull << q;
                mask[0] &= ~bit;
                grem[0] &= ~bit;
                gbud -= s_mem[(q) * RS];
                gg += 1;
                start_granted(q);
                gcand[0] &= ~((bit << 1) - 1ull);
            }
            if (!pick || !gcand[0]) end_round(grem[0] == 0);
            return;
        }
        // lowest candidate (the queue head of the round) and lowest fit
        uint32_t hq = N, fq = N;
#pragma unroll
        for (int w = (int)NW - 1; w >= 0; w--) {
            const uint64_t fit = gcand[w] & t[w];
            if (gcand[w]) hq = 64u * (uint32_t)w + ffs64(gcand[w]);
            if (fit) fq = 64u * (uint32_t)w + ffs64(fit);
        }
        // FIFO takes the head iff it fits, MMU the lowest fit (policy.py:65-73)
        const uint32_t q = mmu ? fq : (fq == hq ? hq : N);
        const bool pick = q < N;
        bool more = false;
        if (pick) {
            const uint32_t qw = q >> 6;
            const uint64_t bit = 1ull << (q & 63u);
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) {
                mask[w] &= w == qw ? ~bit : ~0ull;
                grem[w] &= w == qw ? ~bit : ~0ull;
                // continue above the granted position
                gcand[w] &= w < qw ? 0ull : (w == qw ? ~((bit << 1) - 1ull) : ~0ull);
                more = more || gcand[w] != 0;
            }
            gbud -= s_mem[(q) * RS];
            gg += 1;
            start_granted(q);
        }
        if (!more) {  // the round ends
            bool left = false;
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) left = left || grem[w] != 0;
            end_round(!left);
        }
    }
    SG_HD void end_round(bool drained) {
        if (gg) {
            mem_point(last);
            used += gb0 - gbud;
            holders += (int32_t)gg;
            maxh = max(maxh, (uint32_t)holders);
            grants += gg;
        }
        // the top class drained: the next class is served in the same tick
        // (harness.py:547-550); otherwise the next round is empty
        if (prio_pol && gg && drained) {
            clsmask &= ~(1u << gc);
            gs = clsmask != 0;  // the next class has waiters: its round starts next step
            ginit = gs;
        } else {
            gs = false;
        }
    }
    SG_HD void grant_waiters_tbl() {
        bool any = false;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) any = any || mask[w] != 0;
        gs = any;
        ginit = any;
    }

    // longer traces: scan the candidates in queue order
    SG_HD void grant_waiters_scan() {
        uint32_t c = 0;  // current class (priority kinds)
        while (true) {
            // candidate set: the waiting entries of the top class (policy.py:58-63)
            uint64_t cand[NW];
            bool any = false;
            if (prio_pol) {
                while (c < ncls) {
#pragma unroll
                    for (uint32_t w = 0; w < NW; w++) {
                        cand[w] = mask[w] & s_cm[c * NW + w];
                        any = any || cand[w] != 0;
                    }
                    if (any) break;
                    c += 1;
                }
            } else {
#pragma unroll
                for (uint32_t w = 0; w < NW; w++) {
                    cand[w] = mask[w];
                    any = any || cand[w] != 0;
                }
            }
            if (!any) return;
            const uint32_t budget0 = cap - used;
            uint32_t budget = budget0, g = 0;
            // FIFO: grant the head while it fits; MMU: skip misfits
            bool stop = false;
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) {
                uint64_t bits = cand[w];
                while (bits && !stop) {
                    const uint32_t q = 64u * w + ffs64(bits);
                    bits &= bits - 1;
                    const uint32_t m = s_mem[(q) * RS];
                    if (m <= budget) {
                        grant_one(q, m, budget, g);
                        if (fail) return;
                    } else if (!mmu) {
                        stop = true;
                    }
                }
            }
            if (g) {
                mem_point(last);
                used += budget0 - budget;
                holders += (int32_t)g;
                maxh = max(maxh, (uint32_t)holders);
                grants += g;
            }
            if (!prio_pol || g == 0) return;
            bool left = false;
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) left = left || (mask[w] & s_cm[c * NW + w]) != 0;
            if (left) return;
            c += 1;
        }
    }

    // --------------------------------------------------------- advance
    SG_HD void end_app(uint32_t m, uint32_t bw, uint32_t now) {
        if (m) {  // free -> grant_waiters (harness.py:537-542)
            mem_point(now);
            used -= m;
            holders -= 1;
            grant_waiters();
        }
        const uint32_t o = bw_app(bw);  // end (harness.py:543)
        if (ep) ep[o] = now;
        // the grant is the busy start: busy runs [grant, grant + busy]
        if (gp) gp[o] = m ? now - bw_busy(bw) : SG_NEVER;
    }
    // initial pop at t = 0 of an app without a cpu step; its busy end owns
    // the app's initial virtual counter c
    SG_HD void run_from_busy(uint32_t q, uint32_t m, uint32_t bw, uint32_t now, uint32_t c) {
        const uint32_t b = bw_busy(bw);
        if (b) {  // busy (harness.py:514-520)
            busy_point(now, +1);
            push(now + b, c, q);
            return;
        }
        end_app(m, bw, now);
    }
    SG_HD void arrive(uint32_t q, uint32_t m, uint32_t bw, uint32_t now, uint32_t c) {
        if (m) {
            if (m <= cap - used) {  // arrival bypass (harness.py:521-531)
                mem_point(now);
                used += m;
                holders += 1;
                maxh = max(maxh, (uint32_t)holders);
                grants += 1;
            } else {                // wait (harness.py:532-536)
                enqueue(q, bw);
                return;
            }
        }
        run_from_busy(q, m, bw, now, c);
    }

    // Simulate device range [s, e) of the slot's arrival order (z apps arrive
    // at t = 0).  Returns false if this lane must be re-run by the fallback.
    SG_HD bool run(uint32_t n_trace, uint32_t s, uint32_t e, uint32_t z,
                                        uint32_t policy, uint32_t cap_mib) {
        cap = cap_mib;
        used = 0;
        prio_pol = policy >= SG_POLICY_PFIFO;
        mmu = (policy & 1u) != 0;
        fail = false;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) mask[w] = 0;
        hs = 0;
        kh = KY::INF;
        last = mem_t = busy_prev = B = 0;
        I = 0;
        busy_level = holders = 0;
        maxh = grants = pops = 0;
        gs = ginit = pp = false;
        pt = pc = pq = 0;
        clsmask = 0;
        // later pushes, including those of waiters granted at t = 0 (after
        // every initial entry), count up from c_base
        counter = cw = KY::c_base(n_trace);
        wt = 0;
        ap = ae = 0;  // no pending arrival of tick 0: those apps run inline
        ka = KY::INF;
        // initial pops at t = 0: apps without a cpu step run inline, in index
        // order, each in its own virtual counter block
        for (uint32_t q = s; q < s + z; q++) {
            const uint32_t bw = s_bw[(q) * RS];
            arrive(q, s_mem[(q) * RS], bw, 0u, KY::c_init(bw_app(bw)));
            if constexpr (TBL) {
                while (gs && !fail) {
                    grant_step();
                    if (pp) {
                        push(pt, pc, pq);
                        pp = false;
                    }
                }
            }
            if (fail) break;  // (into the main loop, which stops at once: SY lanes meet there)
        }
        ap = s + z;
        ae = e;
        uint32_t bwa = 0;
        if (ap < e) {
            bwa = s_bw[(ap) * RS];
            ka = KY::make(s_a[ap], KY::c_init(bw_app(bwa)), ap);
        }
        while (true) {
            SG_LANE_ITER_HOOK(gs);
            bool stop = fail;
            if (!gs && !stop) {
                // next event: the smaller of the arrival / heap keys (busy
                // ends and the frees of granted waiters without a busy step)
                const Key kmin = ka < kh ? ka : kh;
                stop = kmin == KY::INF;
            }
            if (!gs && !stop) {
                const Key kmin = ka < kh ? ka : kh;
                const bool is_arr = ka < kh;
                const uint32_t q = KY::pos(kmin);
                const uint32_t now = KY::time(kmin);
                if (!is_arr) pop();
                if (is_arr) {
                    ap += 1;
                    if (ap < e) {
                        bwa = s_bw[(ap) * RS];
                        ka = KY::make(s_a[ap], KY::c_init(bw_app(bwa)), ap);
                    } else {
                        ka = KY::INF;
                    }
                }
                const uint32_t m = s_mem[(q) * RS];
                const uint32_t bw = s_bw[(q) * RS];
                const uint32_t b = bw_busy(bw);
                pops += 1;
                last = now;
                // arrival: memory-fit admission with bypass, else wait (harness.py:521-536)
                const bool alloc = is_arr && m != 0;
                const bool fits = m <= cap - used;
                const bool enq = alloc && !fits;
                if (enq) enqueue(q, bw);
                mem_point(now);
                if (alloc && fits) {
                    used += m;
                    holders += 1;
                    maxh = max(maxh, (uint32_t)holders);
                    grants += 1;
                }
                // busy (harness.py:514-520), its end, or a granted waiter's free
                const bool start = is_arr && !enq && b != 0;
                busy_point(now, start ? 1 : (!is_arr && b != 0 ? -1 : 0));
                pp = start;
                pt = now + b;
                pq = q;
                // an arrival's busy end: above every counter of earlier ticks
                pc = wt == now ? counter : max(counter, cw);
                counter = pc + (start ? 1u : 0u);
                if ((is_arr && !enq && b == 0) || !is_arr) end_app(m, bw, now);
            }
            if (!stop) {
                if constexpr (TBL) {
                    if (gs) grant_step();
                }
                // at most one push per iteration: an arrival's busy end, or the
                // entry of the waiter this iteration's grant step granted
                if (pp) push(pt, pc, pq);
                pp = false;
            }
            stop = stop || fail;
            sync_iter(stop);
            if (stop) break;
        }
        return !fail;
    }

#ifdef __CUDACC__
    SG_HD void finish(uint64_t srec, uint32_t nd, uint32_t st, uint64_t seq) {
        uint32_t unf = 0;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) {
            for (uint64_t bits = mask[w]; bits; bits &= bits - 1) {
                const uint32_t q = 64u * w + ffs64(bits);
                const uint32_t o = bw_app(s_bw[(q) * RS]);
                if (gp) gp[o] = SG_NEVER;
                if (ep) ep[o] = SG_NEVER;
                unf += 1;
            }
        }
        store_tick_record(P, srec, nd, cap, last, mem_t, I, B, (int64_t)used, grants, pops + nd,
                          maxh, unf, st, seq);
    }
#endif
};

}  // namespace sg
