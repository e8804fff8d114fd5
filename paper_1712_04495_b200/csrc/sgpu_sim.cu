// sgpu_sim.cu — K1 `trace_sim`: one warp simulates one workload trace under
// memshare's memory-fit admission and one of the four wait policies, with the
// reference's exact event order, and emits fused per-trace statistics.
//
// Semantics restated from the reference:
//   event order      (t, push-counter) heap: memshare/harness.py:505-508, 563-565
//   advance          memshare/harness.py:510-543 (inline continuation, arrival
//                    bypass at 521-531, free -> grant_waiters -> continue 537-542)
//   grant_waiters    memshare/harness.py:545-558 (fixpoint of select_grants)
//   select_grants    memshare/policy.py:52-74
//   metrics          memshare/harness.py:373-461 (makespan, memory integral,
//                    busy union, max concurrent holders), fused incrementally
//
// B200 mapping:
//   * warp per trace, all policies of a trace back to back on the staged copy;
//     persistent grid (SMs x resident blocks), grid-stride over traces
//   * the trace's 16 B/app records are staged global->shared by the TMA bulk
//     engine (cp.async.bulk + mbarrier), double-buffered so trace i+1 streams
//     in while trace i is simulated
//   * the heap is a per-app (t, counter) key held in registers (lane l owns
//     apps l, l+32, ...); the next event is a two-step REDUX min (time, then
//     counter) — exact restatement of heapq's tuple order
//   * the wait queue (enqueue order) lives in shared memory; FIFO grants are a
//     warp prefix-sum + ballot, MMU first-fit is a __ballot_sync/__ffs loop,
//     priority classes a REDUX max — no atomics anywhere on event times
#include <cmath>

#include "sgpu_common.cuh"
#include "sgpu_internal.h"

namespace sg {

constexpr uint32_t kBusyFlag = 0x8000u;   // s_pc bit: the pending pop ends a busy step
constexpr uint32_t kSat = 0x7FFFFFFFu;    // MiB saturation for FIFO prefix sums
constexpr uint32_t kAppBits = 10;         // SG_MAX_APPS == 1 << kAppBits
constexpr uint32_t kCounterLimit = 1u << (32 - kAppBits);
constexpr double kMiB = 1048576.0;

// ------------------------------------------------------------ time models

struct TickTM {
    using T = uint32_t;
    using Key = uint32_t;
    using Acc = uint64_t;
    static constexpr bool F64 = false;
    static constexpr Key INFK = 0xFFFFFFFFu;
    static __device__ __forceinline__ Key key(T t) { return t; }
    static __device__ __forceinline__ T time(Key k) { return k; }
    static __device__ __forceinline__ T zero() { return 0u; }
    static __device__ __forceinline__ T never() { return SG_NEVER; }
    static __device__ __forceinline__ bool is_never(T t) { return t == SG_NEVER; }
    static __device__ __forceinline__ T add(T now, uint64_t dur, bool& ovf) {
        uint64_t s = (uint64_t)now + dur;
        if (s > 0xFFFFFFFEull) { ovf = true; s = 0xFFFFFFFEull; }
        return (T)s;
    }
    static __device__ __forceinline__ Key warp_min(Key k) { return __reduce_min_sync(FULL, k); }
    static __device__ __forceinline__ uint64_t bits(T t) { return t; }
};

struct F64TM {
    using T = double;
    using Key = uint64_t;
    using Acc = double;
    static constexpr bool F64 = true;
    static constexpr Key INFK = 0xFFFFFFFFFFFFFFFFull;
    // Event times are non-negative doubles: their IEEE bit patterns order
    // like the values, so the heap key is the raw bits.
    static __device__ __forceinline__ Key key(T t) { return (Key)__double_as_longlong(t); }
    static __device__ __forceinline__ T time(Key k) { return __longlong_as_double((long long)k); }
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T never() { return __longlong_as_double(-1LL); }  // NaN
    static __device__ __forceinline__ bool is_never(T t) { return isnan(t); }
    static __device__ __forceinline__ T add(T now, uint64_t dur, bool&) {
        return __dadd_rn(now, __longlong_as_double((long long)dur));  // harness.py:517,519
    }
    static __device__ __forceinline__ Key warp_min(Key k) { return warp_min_u64(k); }
    static __device__ __forceinline__ uint64_t bits(T t) { return (uint64_t)__double_as_longlong(t); }
};

template <class TM>
struct DevState {
    typename TM::T last;       // time of the latest pop of this device's apps = makespan
    typename TM::T mem_t;      // time of the previous memory point
    typename TM::T busy_prev;  // time of the previous busy point
    typename TM::Acc I;        // memory integral (MiB*ticks, or byte-seconds)
    typename TM::Acc B;        // busy union (ticks, or seconds)
    int64_t used;              // MiB held
    int32_t busy_level;
    int32_t holders;
    uint32_t maxh;
    uint32_t grants;
    uint32_t pops;
};

__device__ __forceinline__ uint32_t q_app(uint64_t e) { return (uint32_t)(e >> 32) & 0xFFFFu; }
__device__ __forceinline__ uint32_t q_prio(uint64_t e) { return (uint32_t)(e >> 48) & 0xFFu; }
__device__ __forceinline__ uint32_t q_dev(uint64_t e) { return (uint32_t)(e >> 56); }
__device__ __forceinline__ uint64_t q_pack(uint32_t app, uint32_t mib, uint32_t prio, uint32_t d) {
    return ((uint64_t)d << 56) | ((uint64_t)(prio & 0xFF) << 48) | ((uint64_t)app << 32) | mib;
}

template <class TM, int K, bool PROG, bool MULTI>
struct TraceSim {
    using T = typename TM::T;
    using Key = typename TM::Key;
    using DS = DevState<TM>;

    const SimParams& P;
    const uint32_t lane;
    // per-warp shared memory
    const uint4* s_app;
    uint64_t* s_q;
    T* s_grant;
    T* s_end;
    uint16_t* s_pc;
    int32_t* s_held;
    // trace / policy
    uint32_t n;
    bool prio_pol, mmu;
    // simulation state (warp-uniform unless noted)
    uint32_t qlen, counter, status;
    Key kt[K];        // per-lane: pending time key of apps lane + 32*j
    uint32_t kc[K];   // per-lane: counter << 10 | app
    Key lt;           // per-lane: local minimum key
    uint32_t lc;
    DS ds[MULTI ? SG_MAX_DEV : 1];
    sg_event* ev;
    uint32_t ev_n;

    __device__ __forceinline__ TraceSim(const SimParams& p, uint32_t lane_, uint8_t* ws,
                                        const uint4* apps_smem)
        : P(p), lane(lane_) {
        s_app = apps_smem;
        s_q = reinterpret_cast<uint64_t*>(ws + p.off_q);
        s_grant = reinterpret_cast<T*>(ws + p.off_grant);
        s_end = reinterpret_cast<T*>(ws + p.off_end);
        s_pc = reinterpret_cast<uint16_t*>(ws + p.off_pc);
        s_held = reinterpret_cast<int32_t*>(ws + p.off_held);
    }

    __device__ __forceinline__ DS& dev(uint32_t d) {
        if constexpr (MULTI) return ds[d];
        else return ds[0];
    }
    __device__ __forceinline__ uint32_t dev_of(uint32_t attr) {
        if constexpr (MULTI) {
            uint32_t d = (attr >> 8) & 0xFF;
            return d < P.ndev ? d : 0;
        } else {
            return 0;
        }
    }

    // ---------------------------------------------------------------- keys
    __device__ __forceinline__ void set_key(uint32_t app, Key k, uint32_t c) {
        const uint32_t owner = app & 31, slot = app >> 5;
#pragma unroll
        for (int j = 0; j < K; j++)
            if (lane == owner && slot == (uint32_t)j) { kt[j] = k; kc[j] = (c << kAppBits) | app; }
    }
    __device__ __forceinline__ void clear_key(uint32_t app) {
        const uint32_t owner = app & 31, slot = app >> 5;
#pragma unroll
        for (int j = 0; j < K; j++)
            if (lane == owner && slot == (uint32_t)j) { kt[j] = TM::INFK; kc[j] = 0xFFFFFFFFu; }
    }
    __device__ __forceinline__ void local_min() {
        lt = kt[0];
        lc = kc[0];
#pragma unroll
        for (int j = 1; j < K; j++)
            if (kt[j] < lt || (kt[j] == lt && kc[j] < lc)) { lt = kt[j]; lc = kc[j]; }
    }
    // harness.py:505-508
    __device__ __forceinline__ void push(uint32_t app, T t) {
        counter += 1;
        if (counter >= kCounterLimit) status |= SG_ST_COUNTER_OVERFLOW;
        set_key(app, TM::key(t), counter);
    }

    // -------------------------------------------------------------- events
    __device__ __forceinline__ void emit(T t, uint32_t app, uint32_t kind, uint32_t d, uint32_t mib) {
        if (ev != nullptr) {
            if (lane == 0 && ev_n < P.ev_cap) {
                sg_event e;
                e.t = TM::bits(t);
                e.app = (uint16_t)app;
                e.kind = (uint8_t)kind;
                e.dev = (uint8_t)d;
                e.mib = mib;
                ev[ev_n] = e;
            }
            ev_n++;
        }
    }

    // ---------------------------------------------------------- statistics
    // Memory point: total += level * (t - prev) (harness.py:414-426).
    __device__ __forceinline__ void mem_point(DS& D, T now, int64_t delta) {
        if constexpr (TM::F64) {
            D.I = __dadd_rn(D.I, __dmul_rn(__ll2double_rn(D.used * 1048576LL), __dsub_rn(now, D.mem_t)));
        } else {
            D.I += (uint64_t)(D.used * (int64_t)(now - D.mem_t));
        }
        D.mem_t = now;
        D.used += delta;
    }
    // Busy point in time order: the sweep of harness.py:429-437.  Points of
    // equal time add zero, so pop order within a tick is immaterial.
    __device__ __forceinline__ void busy_point(DS& D, T now, int32_t delta) {
        if (D.busy_level > 0) {
            if constexpr (TM::F64) D.B = __dadd_rn(D.B, __dsub_rn(now, D.busy_prev));
            else D.B += (uint64_t)(now - D.busy_prev);
        }
        D.busy_prev = now;
        D.busy_level += delta;
    }

    // ------------------------------------------------------- grant_waiters
    // harness.py:545-558 with select_grants (policy.py:52-74) inlined as warp
    // scans over the shared-memory queue (device d's entries only).
    __device__ void grant_waiters(uint32_t d, T now) {
        if (qlen == 0) return;
        DS& D = dev(d);
        const int64_t cap = (int64_t)P.cap[MULTI ? d : 0];
        while (true) {
            int64_t budget = cap - D.used;
            uint32_t top = 0;
            if (prio_pol || MULTI) {
                // top = max priority among device-d waiters (policy.py:58-63)
                uint32_t best = 0;  // priority + 1, 0 = none
                for (uint32_t base = 0; base < qlen; base += 32) {
                    const uint32_t i = base + lane;
                    if (i < qlen) {
                        const uint64_t e = s_q[i];
                        if (!MULTI || q_dev(e) == d) best = max(best, q_prio(e) + 1);
                    }
                }
                best = __reduce_max_sync(FULL, best);
                if (best == 0) return;
                top = best - 1;
            }
            uint32_t removed = 0;
            bool stop = false;
            int64_t carry = 0;
            for (uint32_t base = 0; base < qlen; base += 32) {
                const uint32_t i = base + lane;
                const bool valid = i < qlen;
                const uint64_t e = valid ? s_q[i] : 0ull;
                const uint32_t mib = (uint32_t)e;
                const uint32_t app_l = q_app(e);
                const bool cand = valid && !stop && (!MULTI || q_dev(e) == d) &&
                                  (!prio_pol || q_prio(e) == top);
                uint32_t gm = 0;
                if (__any_sync(FULL, cand)) {
                    if (!mmu) {
                        // FIFO: longest prefix whose running sum fits.
                        uint32_t incl = cand ? min(mib, kSat) : 0u;
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const uint32_t y = __shfl_up_sync(FULL, incl, off);
                            if (lane >= (uint32_t)off) incl = min(incl + y, kSat);
                        }
                        const bool fits = cand && (carry + (int64_t)incl <= budget);
                        gm = __ballot_sync(FULL, fits);
                        if (__ballot_sync(FULL, cand && !fits)) stop = true;
                        carry += (int64_t)__shfl_sync(FULL, incl, 31);
                    } else {
                        // MMU: first fit with a shrinking budget, skip misfits.
                        uint32_t rem = __ballot_sync(FULL, cand);
                        while (rem) {
                            const uint32_t fm = __ballot_sync(FULL, cand && (int64_t)mib <= budget) & rem;
                            if (!fm) break;
                            const uint32_t j = __ffs(fm) - 1;
                            gm |= 1u << j;
                            budget -= (int64_t)__shfl_sync(FULL, mib, j);
                            rem &= (j == 31) ? 0u : (0xFFFFFFFFu << (j + 1));
                        }
                    }
                }
                const bool mine = (gm >> lane) & 1u;
                const uint32_t below = __popc(gm & lanemask_lt());
                if (gm) {
                    // grant in queue order: used += nbytes, grant + alloc events,
                    // pc past the alloc, push (now, ++counter)  (harness.py:551-558)
                    const uint32_t g = __popc(gm);
                    const uint32_t sum = __reduce_add_sync(FULL, mine ? mib : 0u);
                    mem_point(D, now, (int64_t)sum);
                    if constexpr (PROG) {
                        bool inc = false;
                        if (mine) {
                            const int32_t h = s_held[app_l];
                            const int32_t nh = h + (int32_t)mib;
                            s_held[app_l] = nh;
                            inc = h <= 0 && nh > 0;
                            s_pc[app_l] = (uint16_t)(s_pc[app_l] + 1);
                        }
                        D.holders += __popc(__ballot_sync(FULL, inc));
                    } else {
                        D.holders += (int32_t)g;
                        if (mine) s_pc[app_l] = 2;
                    }
                    if (mine && TM::is_never(s_grant[app_l])) s_grant[app_l] = now;
                    D.maxh = max(D.maxh, (uint32_t)max(D.holders, 0));
                    D.grants += g;
                    if (ev != nullptr) {
                        if (mine) {
                            const uint32_t pos = ev_n + 2 * below;
                            sg_event e1;
                            e1.t = TM::bits(now);
                            e1.app = (uint16_t)app_l;
                            e1.dev = (uint8_t)d;
                            e1.mib = mib;
                            e1.kind = SG_EV_GRANT;
                            if (pos < P.ev_cap) ev[pos] = e1;
                            e1.kind = SG_EV_ALLOC;
                            if (pos + 1 < P.ev_cap) ev[pos + 1] = e1;
                        }
                        ev_n += 2 * g;
                    }
                    const uint32_t c0 = counter;
                    counter += g;
                    if (counter >= kCounterLimit) status |= SG_ST_COUNTER_OVERFLOW;
                    uint32_t rem = gm, k = 0;
                    while (rem) {
                        const uint32_t j = __ffs(rem) - 1;
                        rem &= rem - 1;
                        const uint32_t a = __shfl_sync(FULL, app_l, j);
                        set_key(a, TM::key(now), c0 + (++k));
                    }
                }
                // stable compaction of the survivors
                const uint32_t shift = removed + below;
                __syncwarp();
                if (valid && !mine && shift) s_q[i - shift] = e;
                removed += __popc(gm);
                __syncwarp();
            }
            qlen -= removed;
            // FIFO/MMU: a second round is provably empty (every survivor
            // already failed against a budget >= the current one); priority
            // policies drain the top class and may serve the next one in the
            // same tick (fixpoint, harness.py:547-550).
            if (removed == 0 || !prio_pol || qlen == 0) return;
        }
    }

    // -------------------------------------------------------------- advance
    // harness.py:510-543: run app's steps from its pc until it blocks.
    __device__ void advance(uint32_t app, T now, bool counted_pop) {
        const uint4 f = s_app[app];
        uint32_t pc = s_pc[app];
        int32_t held = 0;
        if constexpr (PROG) held = s_held[app];
        __syncwarp();
        const uint32_t d = dev_of(f.w);
        DS& D = dev(d);
        const int64_t cap = (int64_t)P.cap[MULTI ? d : 0];
        D.last = now;
        if (counted_pop) D.pops += 1;
        if (pc & kBusyFlag) {
            busy_point(D, now, -1);
            pc &= ~kBusyFlag;
        }
        while (true) {
            uint32_t op = 0, mib = 0;
            uint64_t dur = 0;
            bool done = false;
            if constexpr (PROG) {
                if (pc >= f.y) {
                    done = true;
                } else {
                    const uint4 st = __ldg(reinterpret_cast<const uint4*>(P.steps) + f.x + pc);
                    op = st.x;
                    mib = st.y;
                    dur = ((uint64_t)st.w << 32) | st.z;
                }
            } else {
                // T0: cpu(arrival) -> alloc(mem) -> busy(busy) -> free(mem),
                // zero fields skipped (harness.py:482-489)
                if (pc == 0) {
                    if (f.x) { op = SG_OP_CPU; dur = f.x; } else { pc = 1; continue; }
                } else if (pc == 1) {
                    if (f.y) { op = SG_OP_ALLOC; mib = f.y; } else { pc = 2; continue; }
                } else if (pc == 2) {
                    if (f.z) { op = SG_OP_BUSY; dur = f.z; } else { pc = 3; continue; }
                } else if (pc == 3) {
                    if (f.y) { op = SG_OP_FREE; mib = f.y; } else { pc = 4; continue; }
                } else {
                    done = true;
                }
            }
            if (done) {  // harness.py:543
                s_end[app] = now;
                s_pc[app] = (uint16_t)pc;
                emit(now, app, SG_EV_END, d, 0);
                return;
            }
            if (op == SG_OP_CPU || op == SG_OP_BUSY) {  // harness.py:514-520
                bool ovf = false;
                const T t2 = TM::add(now, dur, ovf);
                if (ovf) status |= SG_ST_TICK_OVERFLOW;
                if (op == SG_OP_BUSY) {
                    busy_point(D, now, +1);
                    emit(now, app, SG_EV_BUSY_START, d, 0);
                    emit(t2, app, SG_EV_BUSY_END, d, 0);
                }
                pc += 1;
                s_pc[app] = (uint16_t)(pc | (op == SG_OP_BUSY ? kBusyFlag : 0u));
                if constexpr (PROG) s_held[app] = held;
                push(app, t2);
                return;
            }
            if (op == SG_OP_ALLOC) {  // harness.py:521-536
                emit(now, app, SG_EV_REQUEST, d, mib);
                if (D.used + (int64_t)mib <= cap) {  // arrival bypass: fits => granted
                    mem_point(D, now, (int64_t)mib);
                    if constexpr (PROG) {
                        if (held <= 0 && held + (int32_t)mib > 0) D.holders += 1;
                        held += (int32_t)mib;
                    } else {
                        D.holders += 1;
                    }
                    D.maxh = max(D.maxh, (uint32_t)max(D.holders, 0));
                    D.grants += 1;
                    if (TM::is_never(s_grant[app])) s_grant[app] = now;
                    emit(now, app, SG_EV_GRANT, d, mib);
                    emit(now, app, SG_EV_ALLOC, d, mib);
                    pc += 1;
                    continue;
                }
                s_q[qlen] = q_pack(app, min(mib, kSat), f.w & 0xFF, d);
                qlen += 1;
                s_pc[app] = (uint16_t)pc;
                if constexpr (PROG) s_held[app] = held;
                return;
            }
            // SG_OP_FREE: harness.py:537-542
            mem_point(D, now, -(int64_t)mib);
            if constexpr (PROG) {
                if (held > 0 && held - (int32_t)mib <= 0) D.holders -= 1;
                held -= (int32_t)mib;
            } else {
                D.holders -= 1;
            }
            pc += 1;
            s_pc[app] = (uint16_t)pc;
            if constexpr (PROG) s_held[app] = held;
            emit(now, app, SG_EV_FREE, d, mib);
            __syncwarp();
            grant_waiters(d, now);
        }
    }

    // first step of app i is a cpu step (initial pop only pushes)?
    __device__ __forceinline__ bool first_is_cpu(uint32_t i, uint64_t& dur) {
        const uint4 f = s_app[i];
        if constexpr (PROG) {
            if (f.y == 0) return false;
            const uint4 st = __ldg(reinterpret_cast<const uint4*>(P.steps) + f.x);
            dur = ((uint64_t)st.w << 32) | st.z;
            return st.x == SG_OP_CPU;
        } else {
            dur = f.x;
            return f.x != 0;
        }
    }

    // ------------------------------------------------------------------ run
    __device__ void run(uint32_t n_apps, uint32_t policy, sg_event* ev_slice) {
        n = n_apps;
        prio_pol = policy >= SG_POLICY_PFIFO;
        mmu = (policy & 1u) != 0;
        qlen = 0;
        counter = n;  // initial pushes took counters 1..n (harness.py:560-562)
        status = 0;
        ev = ev_slice;
        ev_n = 0;
#pragma unroll
        for (int j = 0; j < K; j++) { kt[j] = TM::INFK; kc[j] = 0xFFFFFFFFu; }
#pragma unroll
        for (int d = 0; d < (MULTI ? SG_MAX_DEV : 1); d++) {
            ds[d].last = TM::zero();
            ds[d].mem_t = TM::zero();
            ds[d].busy_prev = TM::zero();
            ds[d].I = 0;
            ds[d].B = 0;
            ds[d].used = 0;
            ds[d].busy_level = 0;
            ds[d].holders = 0;
            ds[d].maxh = 0;
            ds[d].grants = 0;
            ds[d].pops = 0;
        }
        for (uint32_t i = lane; i < n; i += 32) {
            s_pc[i] = 0;
            s_grant[i] = TM::never();
            s_end[i] = TM::never();
            if constexpr (PROG) s_held[i] = 0;
            if (ev != nullptr && i < P.ev_cap) {  // start events (harness.py:561)
                sg_event e;
                e.t = TM::bits(TM::zero());
                e.app = (uint16_t)i;
                e.kind = SG_EV_START;
                e.dev = (uint8_t)dev_of(s_app[i].w);
                e.mib = 0;
                ev[i] = e;
            }
        }
        if (ev != nullptr) ev_n = n;
        __syncwarp();

        uint32_t next_init = 0;
        local_min();
        while (true) {
            uint32_t app;
            T now;
            bool counted = true;
            if (next_init < n) {
                // Initial pops run in index order at t = 0 before anything else
                // (their counters 1..n precede every later push).  A run of apps
                // whose first step is cpu only pushes (t = d, ++counter): do the
                // whole run at once; any other app is advanced individually.
                const uint32_t c = next_init >> 5;
                const uint32_t i = (c << 5) + lane;
                const bool valid = i < n && i >= next_init;
                uint64_t dur = 0;
                const bool simple = valid && first_is_cpu(i, dur);
                const uint32_t vm = __ballot_sync(FULL, valid);
                const uint32_t sm = __ballot_sync(FULL, simple);
                const uint32_t nonsimple = vm & ~sm;
                const uint32_t run = nonsimple ? (sm & ((1u << (__ffs(nonsimple) - 1)) - 1u)) : sm;
                if (run) {
                    const bool in = (run >> lane) & 1u;
                    bool ovf = false;
                    const T t2 = TM::add(TM::zero(), dur, ovf);
                    if (__any_sync(FULL, in && ovf)) status |= SG_ST_TICK_OVERFLOW;
                    const uint32_t cval = counter + __popc(run & lanemask_lt()) + 1;
#pragma unroll
                    for (int j = 0; j < K; j++)
                        if (in && c == (uint32_t)j) { kt[j] = TM::key(t2); kc[j] = (cval << kAppBits) | i; }
                    if (in) s_pc[i] = 1;
                    counter += __popc(run);
                    if (counter >= kCounterLimit) status |= SG_ST_COUNTER_OVERFLOW;
                }
                if (!nonsimple) {
                    next_init = min(n, (c + 1) << 5);
                    continue;
                }
                app = (c << 5) + __ffs(nonsimple) - 1;
                next_init = app + 1;
                now = TM::zero();
                counted = false;
                __syncwarp();
            } else {
                local_min();
                const Key kmin = TM::warp_min(lt);
                if (kmin == TM::INFK) break;
                const uint32_t cm = __reduce_min_sync(FULL, lt == kmin ? lc : 0xFFFFFFFFu);
                app = cm & (SG_MAX_APPS - 1);
                now = TM::time(kmin);
                clear_key(app);
            }
            __syncwarp();
            advance(app, now, counted);
        }
    }

    // --------------------------------------------------------------- output
    __device__ void finish(uint64_t rec_base, uint64_t app_out_base, uint32_t* ev_count_out) {
        __syncwarp();
        const uint32_t nd = MULTI ? P.ndev : 1;
        uint32_t napps[MULTI ? SG_MAX_DEV : 1];
        uint32_t unf[MULTI ? SG_MAX_DEV : 1];
#pragma unroll
        for (int d = 0; d < (MULTI ? SG_MAX_DEV : 1); d++) { napps[d] = 0; unf[d] = 0; }
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            const bool valid = i < n;
            T gv = TM::never(), evv = TM::never();
            uint32_t dd = 0;
            if (valid) {
                gv = s_grant[i];
                evv = s_end[i];
                dd = dev_of(s_app[i].w);
                if (P.grant) reinterpret_cast<T*>(P.grant)[app_out_base + i] = gv;
                if (P.end) reinterpret_cast<T*>(P.end)[app_out_base + i] = evv;
            }
#pragma unroll
            for (int d = 0; d < (MULTI ? SG_MAX_DEV : 1); d++) {
                napps[d] += __popc(__ballot_sync(FULL, valid && dd == (uint32_t)d));
                unf[d] += __popc(__ballot_sync(FULL, valid && dd == (uint32_t)d && TM::is_never(evv)));
            }
        }
        if (ev_count_out != nullptr && lane == 0) *ev_count_out = ev_n;
        const double scale = ldexp(1.0, -P.tick_log2);
#pragma unroll
        for (int d = 0; d < (MULTI ? SG_MAX_DEV : 1); d++) {
            if ((uint32_t)d >= nd) break;
            if (lane != (uint32_t)d) continue;
            DS& D = ds[d];
            uint32_t st = status;
            double mem_pct, dev_pct;
            const double cap_bytes = (double)P.cap[d] * kMiB;
            if constexpr (TM::F64) {
                // makespan_s = max(t_end - t0, 1e-9), final integral term (harness.py:378, 425)
                const double span = D.last >= 1e-9 ? D.last : 1e-9;
                D.I = __dadd_rn(D.I, __dmul_rn(__ll2double_rn(D.used * 1048576LL), __dsub_rn(span, D.mem_t)));
                mem_pct = __ddiv_rn(__dmul_rn(100.0, D.I), __dmul_rn(cap_bytes, span));
                dev_pct = __ddiv_rn(__dmul_rn(100.0, D.B), span);
                sg_trace_stats_f64 r;
                r.makespan_s = D.last;
                r.mem_integral = D.I;
                r.busy_s = D.B;
                r.grants = D.grants;
                r.pops = D.pops + napps[d];
                r.max_holders = (uint16_t)D.maxh;
                r.unfinished = (uint16_t)unf[d];
                r.status = st;
                reinterpret_cast<sg_trace_stats_f64*>(P.stats)[rec_base + d] = r;
            } else {
                uint64_t I = D.I;
                double integral;
                if (D.last == 0 && D.used != 0) {
                    // span = 1e-9 s is not on the tick grid: report the level
                    st |= SG_ST_ZERO_SPAN_LEVEL;
                    I = (uint64_t)D.used;
                    integral = __dmul_rn(__ll2double_rn(D.used * 1048576LL), 1e-9);
                } else {
                    I += (uint64_t)(D.used * (int64_t)(D.last - D.mem_t));
                    integral = __dmul_rn((double)I, kMiB * scale);
                }
                const double span = D.last > 0 ? __dmul_rn((double)D.last, scale) : 1e-9;
                mem_pct = __ddiv_rn(__dmul_rn(100.0, integral), __dmul_rn(cap_bytes, span));
                dev_pct = __ddiv_rn(__dmul_rn(100.0, __dmul_rn((double)D.B, scale)), span);
                sg_trace_stats r;
                r.makespan = D.last;
                r.busy = (uint32_t)D.B;
                r.mem_integral = I;
                r.grants = D.grants;
                r.pops = D.pops + napps[d];
                r.max_holders = (uint16_t)D.maxh;
                r.unfinished = (uint16_t)unf[d];
                r.status = st;
                reinterpret_cast<sg_trace_stats*>(P.stats)[rec_base + d] = r;
            }
            if (napps[d] == 0) { mem_pct = 0.0; dev_pct = 0.0; }  // empty event list (harness.py:374-375)
            if (P.mem_pct) P.mem_pct[rec_base + d] = mem_pct;
            if (P.dev_pct) P.dev_pct[rec_base + d] = dev_pct;
        }
        __syncwarp();
    }
};

// ------------------------------------------------------------------ kernel

template <class TM, int K, bool PROG, bool MULTI>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32)
trace_sim_kernel(const SimParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * P.warp_bytes;
    uint4* app_buf[2] = {reinterpret_cast<uint4*>(ws + P.off_app),
                         reinterpret_cast<uint4*>(ws + P.off_app + (size_t)P.n_pad * 16)};
    uint64_t* bar = reinterpret_cast<uint64_t*>(ws + P.off_bar);

    const uint64_t gw = (uint64_t)blockIdx.x * kSimWarpsPerBlock + warp;
    const uint64_t stride = (uint64_t)gridDim.x * kSimWarpsPerBlock;

    auto trace_range = [&](uint64_t t, uint64_t& a0, uint32_t& na) {
        if (P.trace_offsets) {
            const uint64_t o0 = P.trace_offsets[0];
            a0 = P.trace_offsets[t] - o0;
            na = (uint32_t)(P.trace_offsets[t + 1] - P.trace_offsets[t]);
        } else {
            a0 = t * P.apps_per_trace;
            na = P.apps_per_trace;
        }
    };
    // T0 mode: stage the trace's 16 B/app records with the bulk-copy engine.
    auto stage = [&](uint64_t t, int b) {
        uint64_t a0;
        uint32_t na;
        trace_range(t, a0, na);
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[b], na * 16u);
            if (na) bulk_g2s(app_buf[b], P.apps + a0, na * 16u, &bar[b]);
        }
    };

    if constexpr (!PROG) {
        if (lane == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            fence_mbar_init();
        }
        __syncwarp();
        if (gw < P.n_traces) stage(gw, 0);
    }

    uint32_t iter = 0;
    for (uint64_t t = gw; t < P.n_traces; t += stride, iter++) {
        uint64_t a0;
        uint32_t na;
        trace_range(t, a0, na);
        const int b = PROG ? 0 : (int)(iter & 1u);
        if constexpr (!PROG) {
            mbar_wait(&bar[b], (iter >> 1) & 1u);
            __syncwarp();
            if (t + stride < P.n_traces) stage(t + stride, b ^ 1);
        } else {
            const uint32_t s0 = P.step_offsets[0];
            for (uint32_t i = lane; i < na; i += 32) {
                const uint32_t sb = P.step_offsets[a0 + i] - s0;
                const uint32_t se = P.step_offsets[a0 + i + 1] - s0;
                app_buf[0][i] = make_uint4(sb, se - sb, 0u, P.apps[a0 + i].attr);
            }
            __syncwarp();
        }
        for (uint32_t p = 0; p < P.npol; p++) {
            TraceSim<TM, K, PROG, MULTI> sim(P, lane, ws, app_buf[b]);
            const uint64_t slot = (uint64_t)p * P.n_traces + t;
            sg_event* evs = P.events ? P.events + slot * P.ev_cap : nullptr;
            sim.run(na, P.policies[p], evs);
            sim.finish(slot * P.ndev, (uint64_t)p * P.n_apps_total + a0,
                       P.event_counts ? P.event_counts + slot : nullptr);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ launch

static inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

void sim_layout(SimParams& p, bool program_mode, bool f64) {
    const uint32_t N = p.n_pad;
    const uint32_t tsz = f64 ? 8u : 4u;
    uint32_t o = 0;
    p.off_app = o;
    o = align16(o + N * 16u * (program_mode ? 1u : 2u));
    p.off_q = o;
    o = align16(o + N * 8u);
    p.off_grant = o;
    o = align16(o + N * tsz);
    p.off_end = o;
    o = align16(o + N * tsz);
    p.off_pc = o;
    o = align16(o + N * 2u);
    p.off_held = o;
    o = align16(o + (program_mode ? N * 4u : 0u));
    p.off_bar = o;
    o = align16(o + 16u);
    p.warp_bytes = o;
}

template <class TM, int K, bool PROG, bool MULTI>
static cudaError_t launch_t(const SimParams& p, cudaStream_t stream, int* grid_out) {
    auto kern = trace_sim_kernel<TM, K, PROG, MULTI>;
    const size_t smem = (size_t)p.warp_bytes * kSimWarpsPerBlock;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSimWarpsPerBlock * 32, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t need = (p.n_traces + kSimWarpsPerBlock - 1) / kSimWarpsPerBlock;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (need < grid) grid = need;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    kern<<<(unsigned)grid, kSimWarpsPerBlock * 32, smem, stream>>>(p);
    return cudaGetLastError();
}

template <class TM, bool PROG, bool MULTI>
static cudaError_t launch_k(const SimParams& p, cudaStream_t s, int* g) {
    const uint32_t k = p.n_pad / 32;
    if (k <= 1) return launch_t<TM, 1, PROG, MULTI>(p, s, g);
    if (k <= 2) return launch_t<TM, 2, PROG, MULTI>(p, s, g);
    if (k <= 4) return launch_t<TM, 4, PROG, MULTI>(p, s, g);
    if (k <= 8) return launch_t<TM, 8, PROG, MULTI>(p, s, g);
    return launch_t<TM, 32, PROG, MULTI>(p, s, g);
}

cudaError_t launch_sim(const SimParams& p, bool program_mode, bool f64, bool multi,
                       cudaStream_t stream, int* grid_out) {
    if (f64) {
        if (!program_mode) return cudaErrorInvalidValue;
        return multi ? launch_k<F64TM, true, true>(p, stream, grid_out)
                     : launch_k<F64TM, true, false>(p, stream, grid_out);
    }
    if (program_mode)
        return multi ? launch_k<TickTM, true, true>(p, stream, grid_out)
                     : launch_k<TickTM, true, false>(p, stream, grid_out);
    return multi ? launch_k<TickTM, false, true>(p, stream, grid_out)
                 : launch_k<TickTM, false, false>(p, stream, grid_out);
}

}  // namespace sg
