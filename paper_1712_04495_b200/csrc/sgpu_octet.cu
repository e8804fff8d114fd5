// sgpu_octet.cu — K1 v8 `trace_sim_octet`: one OCTET (8 lanes of a warp)
// simulates one (trace, policy) of a T0 (burst) batch of 129..256-app
// single-device traces; four simulations per warp, two trace slots staged
// per warp at two policies (one at three or four).
//
// Same semantics as LaneSim (sgpu_lanesim.cuh; every restatement argued
// there, memshare/harness.py:475-572 + policy.py:52-74), with the per-
// simulation state that scales with the trace length spread over the
// octet instead of held by one lane:
//
//  * Wait queue.  Positions are arrival positions (an app enqueues at most
//    once); octet lane j holds the presence word of positions 32j..32j+31,
//    so select_grants' candidate / fit / head sets are one word per lane
//    and "lowest set position" is a ballot + find-first-set (policy.py:52-74).
//  * Fit table.  T[r] (positions of the r smallest requests) is a 256-bit
//    row of eight words, kept at every 4th rank, read one word per lane.
//  * Busy set.  The pending busy ends (and frees of granted waiters
//    without a busy step) are at most 32 keys: four 64-bit registers per
//    lane; the next one is the octet minimum (two REDUX.MIN).  A 33rd
//    concurrent entry fails the simulation over to the exact warp-per-trace
//    TraceSim, run by the whole warp in the same kernel.
//  * Arrival stream, virtual counters, granted waiters pushed at grant
//    time with reserved counters: as LaneSim, with 64-bit keys
//    t << 32 | counter << 8 | position.
//
// Octet-uniform values are held by all eight lanes; every branch on them is
// octet-uniform, so the octet's lanes stay converged and octet collectives
// (__ballot_sync / __shfl_sync / __reduce_min_sync on the octet mask) are
// legal while the four octets of a warp diverge.
#include <cstring>

#include "sgpu_lanesim.cuh"
#include "sgpu_stage256.cuh"
#include "sgpu_warpsort.cuh"

namespace sg {

constexpr uint32_t kOctN = 256;       // positions per trace (n_pad)
constexpr uint32_t kOctFS = kStage256FS;  // fit-table stride (ranks)
constexpr uint32_t kOctLB = 256;      // rank-lookup buckets
constexpr uint32_t kOctSlots = 4;     // busy-set keys per lane (32 per simulation)
constexpr uint32_t kOctMaxCls = kStage256MaxCls;  // priority classes per trace on this path
constexpr int kOctWarpsPerBlock = 2;
constexpr int kOctMinBlocks = 8;      // 16 warps/SM: <= 128 registers

struct OctParams {
    SimParams sp;          // inputs/outputs + the fallback TraceSim layout (single app buffer)
    uint32_t T;            // trace slots per warp (4 / npol, >= 1)
    uint32_t need_cls;     // a priority policy is requested: build class masks
    // per-warp shared-memory layout (bytes); slot strides in OctSlot
    uint32_t off_a, off_mem, off_bw, off_por, off_lt, off_tbl, off_cm, off_meta, off_scr, warp_bytes;
};

// Per-slot strides (elements) of the shared arrays.
struct OctSlot {
    static constexpr uint32_t S32 = kOctN + 1;             // u32 records + the s_mem[N] sentinel
    static constexpr uint32_t POR = kOctN + 4;             // rank -> position (u16) + sentinels
    static constexpr uint32_t LTB = kOctLB + 8;            // u16 buckets, then lo / hi / scale (u32)
    static constexpr uint32_t TBL = (kOctN / kOctFS + 1) * 8;  // fit rows, 8 u32 words each
    static constexpr uint32_t CM = kOctMaxCls * 8;         // class masks, 8 u32 words each
    static constexpr uint32_t META = 8;                    // u32 (sgpu_stage256.cuh)
};

// ------------------------------------------------------------ octet ops
struct Oct {
    uint32_t mask;  // the octet's lanes
    uint32_t base;  // its first lane
    uint32_t j;     // this lane's index in the octet
};
__device__ __forceinline__ uint32_t oballot(const Oct& o, bool p) {
    return (__ballot_sync(o.mask, p) >> o.base) & 0xFFu;
}
__device__ __forceinline__ uint32_t obcast(const Oct& o, uint32_t v, uint32_t src) {
    return __shfl_sync(o.mask, v, (int)(o.base + src));
}
__device__ __forceinline__ uint64_t omin64(const Oct& o, uint64_t v) {
    const uint32_t hi = __reduce_min_sync(o.mask, (uint32_t)(v >> 32));
    const uint32_t lo = __reduce_min_sync(o.mask, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0xFFFFFFFFu);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t osum(const Oct& o, uint32_t v) { return __reduce_add_sync(o.mask, v); }

// --------------------------------------------------------- the simulator
struct OctSim {
    using KY = LaneKey<8, false, kOctSlots * 8u>;  // 64-bit keys, N = 256 counters
    using Key = uint64_t;
    static constexpr uint32_t N = kOctN;
    static constexpr uint32_t FS = kOctFS;

    Oct o;
    // trace slot
    const uint32_t* s_a;
    const uint32_t* s_mem;
    const uint32_t* s_bw;
    const uint16_t* s_por;
    const uint16_t* s_lt;
    uint32_t lt_lo, lt_hi, lt_scale;
    const uint32_t* s_tbl;
    const uint32_t* s_cm;
    uint32_t* gp;            // grant / end ticks of app 0 of the trace under this policy
    uint32_t* ep;
    uint32_t cap, used;
    bool prio_pol, mmu, fail;
    // lane-distributed: queue word (positions 32j..32j+31), round candidates / class members
    uint32_t qw, gcw, grw;
    Key bk[kOctSlots];       // busy set (KY::INF = free slot)
    Key kh;                  // its minimum (octet-uniform)
    uint32_t counter, cw, wt, ap, ae;
    Key ka;
    uint32_t last, mem_t, busy_prev, B;
    uint64_t I;
    int32_t busy_level, holders;
    uint32_t maxh, grants, pops;
    bool gs, ginit;
    uint32_t clsmask, gc, gbud, gb0, gg;
    bool pp;
    uint32_t pt, pc, pq;

    __device__ __forceinline__ void mem_point(uint32_t now) {
        I += (uint64_t)used * (now - mem_t);
        mem_t = now;
    }
    __device__ __forceinline__ void busy_point(uint32_t now, int32_t delta) {
        B += busy_level > 0 ? now - busy_prev : 0u;
        busy_prev = now;
        busy_level += delta;
    }

    // ---------------------------------------------------------- busy set
    __device__ __forceinline__ void refresh_kh() {
        Key m = bk[0];
#pragma unroll
        for (uint32_t s = 1; s < kOctSlots; s++) m = bk[s] < m ? bk[s] : m;
        kh = omin64(o, m);
    }
    __device__ __forceinline__ void push(uint32_t t, uint32_t c, uint32_t q) {
        uint32_t fs = kOctSlots;  // this lane's first free slot
#pragma unroll
        for (int s = (int)kOctSlots - 1; s >= 0; s--) fs = bk[s] == KY::INF ? (uint32_t)s : fs;
        const uint32_t hb = oballot(o, fs < kOctSlots);
        if (hb == 0 || c >= KY::CMAX) {
            fail = true;
            return;
        }
        const Key key = KY::make(t, c, q);
        const bool mine = o.j == (uint32_t)(__ffs(hb) - 1);
#pragma unroll
        for (uint32_t s = 0; s < kOctSlots; s++) bk[s] = mine && s == fs ? key : bk[s];
        kh = key < kh ? key : kh;
    }
    __device__ __forceinline__ void pop() {  // the entry kh (keys are unique: they hold the position)
#pragma unroll
        for (uint32_t s = 0; s < kOctSlots; s++) bk[s] = bk[s] == kh ? KY::INF : bk[s];
        refresh_kh();
    }

    // ------------------------------------------------------- wait queue
    __device__ __forceinline__ void enqueue(uint32_t q, uint32_t bw) {
        qw |= o.j == (q >> 5) ? 1u << (q & 31u) : 0u;
        clsmask |= 1u << bw_cls(bw);
    }
    // number of requests <= budget (LaneSim::fit_rank with u16 tables)
    __device__ __forceinline__ uint32_t fit_rank(uint32_t budget) const {
        if (budget > lt_hi) return N;
        const uint32_t bi = budget < lt_lo ? 0u
                                           : min((uint32_t)(((uint64_t)(budget - lt_lo) * lt_scale) >> 32), kOctLB - 1u);
        uint32_t r = s_lt[bi];
        while (s_mem[s_por[r]] <= budget) r += 1;  // s_por[N] = N, s_mem[N] = ~0 ends the scan
        return r;
    }
    // this lane's word of T[r]: row T[FS floor(r/FS)] + the positions of the
    // up to FS - 1 ranks after it
    __device__ __forceinline__ uint32_t fit_word(uint32_t r) const {
        uint32_t w = s_tbl[(r / FS) * 8u + o.j];
        const uint32_t r0 = r & ~(FS - 1u), k = r & (FS - 1u);
#pragma unroll
        for (uint32_t i = 0; i + 1 < FS; i++) {
            const uint32_t p = s_por[r0 + i];
            w |= i < k && (p >> 5) == o.j ? 1u << (p & 31u) : 0u;
        }
        return w;
    }

    // ------------------------------------------------- granted waiters
    // (LaneSim::start_granted: busy end pushed at grant time with a
    // counter above the ones the tick's pending arrivals may take)
    __device__ __forceinline__ void start_granted(uint32_t q) {
        const uint32_t b = bw_busy(s_bw[q]);
        if (b) {
            busy_point(last, +1);
            pops += 1;  // the waiter's own entry
        }
        if (wt != last) {  // first grant of the tick: reserve the pending arrivals' counters
            uint32_t r = 0;
            if (KY::time(ka) == last)
                while (ap + r < ae && s_a[ap + r] == last) r += 1;
            cw = max(counter, cw) + r;
            wt = last;
        }
        pp = true;
        pt = last + b;
        pc = cw++;
        pq = q;
    }

    // one select_grants step (harness.py:545-558, policy.py:52-74): the
    // round's candidates are the waiting entries of the top class; FIFO takes
    // the head iff it fits, MMU the lowest fit; both continue above it
    __device__ __forceinline__ void grant_step() {
        if (ginit) {  // a round starts inside its first step
            ginit = false;
            if (prio_pol) gc = __ffs(clsmask) - 1;  // clsmask != 0 whenever the queue is not empty
            gcw = qw & (prio_pol ? s_cm[gc * 8u + o.j] : ~0u);
            grw = gcw;
            gs = oballot(o, gcw != 0) != 0;
            gb0 = gbud = cap - used;
            gg = 0;
        }
        const uint32_t fw = gcw & fit_word(fit_rank(gbud));
        // lowest candidate (the round's head) and lowest fit
        const uint32_t hb = oballot(o, gcw != 0), fb = oballot(o, fw != 0);
        uint32_t q = N;
        if (mmu) {
            if (fb) {
                const uint32_t l = __ffs(fb) - 1;
                q = 32u * l + (uint32_t)(__ffs(obcast(o, fw, l)) - 1);
            }
        } else if (hb) {
            const uint32_t l = __ffs(hb) - 1;
            const uint32_t hq = 32u * l + (uint32_t)(__ffs(obcast(o, gcw, l)) - 1);
            q = (obcast(o, fw, l) >> (hq & 31u)) & 1u ? hq : N;
        }
        bool more = false;
        if (q < N) {
            const uint32_t ql = q >> 5, bit = 1u << (q & 31u);
            if (o.j == ql) {
                qw &= ~bit;
                grw &= ~bit;
            }
            // continue above the granted position
            gcw &= o.j < ql ? 0u : (o.j == ql ? ~((bit << 1) - 1u) : ~0u);
            more = oballot(o, gcw != 0) != 0;
            gbud -= s_mem[q];
            gg += 1;
            start_granted(q);
        }
        if (!more) end_round(oballot(o, grw != 0) == 0);
    }
    __device__ __forceinline__ void end_round(bool drained) {
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
            gs = clsmask != 0;
            ginit = gs;
        } else {
            gs = false;
        }
    }

    // --------------------------------------------------------- advance
    __device__ __forceinline__ void end_app(uint32_t m, uint32_t bw, uint32_t now) {
        if (m) {  // free -> grant_waiters (harness.py:537-542)
            mem_point(now);
            used -= m;
            holders -= 1;
            gs = oballot(o, qw != 0) != 0;
            ginit = gs;
        }
        if (o.j == 0) {  // end (harness.py:543); the grant is the busy start
            const uint32_t a = bw_app(bw);
            if (ep) ep[a] = now;
            if (gp) gp[a] = m ? now - bw_busy(bw) : SG_NEVER;
        }
    }
    // initial pop at t = 0 of an app without a cpu step (its busy end owns
    // the app's initial counter c)
    __device__ __forceinline__ void arrive0(uint32_t q, uint32_t m, uint32_t bw, uint32_t c) {
        if (m) {
            if (m <= cap - used) {  // arrival bypass (harness.py:521-531)
                mem_point(0u);
                used += m;
                holders += 1;
                maxh = max(maxh, (uint32_t)holders);
                grants += 1;
            } else {                // wait (harness.py:532-536)
                enqueue(q, bw);
                return;
            }
        }
        const uint32_t b = bw_busy(bw);
        if (b) {  // busy (harness.py:514-520)
            busy_point(0u, +1);
            push(b, c, q);
            return;
        }
        end_app(m, bw, 0u);
    }

    // Positions [0, n) of the slot, z of them arriving at t = 0.  Returns
    // false if the simulation must be re-run by the fallback.
    __device__ __forceinline__ bool run(uint32_t n, uint32_t z, uint32_t policy, uint32_t cap_mib) {
        cap = cap_mib;
        used = 0;
        prio_pol = policy >= SG_POLICY_PFIFO;
        mmu = (policy & 1u) != 0;
        fail = false;
        qw = gcw = grw = 0;
#pragma unroll
        for (uint32_t s = 0; s < kOctSlots; s++) bk[s] = KY::INF;
        kh = KY::INF;
        last = mem_t = busy_prev = B = 0;
        I = 0;
        busy_level = holders = 0;
        maxh = grants = pops = 0;
        gs = ginit = pp = false;
        pt = pc = pq = 0;
        clsmask = gc = gbud = gb0 = gg = 0;
        counter = cw = KY::c_base(n);
        wt = 0;
        ap = ae = 0;
        ka = KY::INF;
        // initial pops at t = 0, in index order (positions [0, z) are the
        // t = 0 arrivals in index order)
        for (uint32_t q = 0; q < z; q++) {
            const uint32_t bw = s_bw[q];
            arrive0(q, s_mem[q], bw, KY::c_init(bw_app(bw)));
            while (gs && !fail) {
                grant_step();
                if (pp) {
                    push(pt, pc, pq);
                    pp = false;
                }
            }
            if (fail) return false;
        }
        ap = z;
        ae = n;
        if (ap < ae) ka = KY::make(s_a[ap], KY::c_init(bw_app(s_bw[ap])), ap);
        while (true) {
            if (!gs) {
                // next event: the smaller of the arrival / busy-set keys
                const Key kmin = ka < kh ? ka : kh;
                if (kmin == KY::INF) break;
                const bool is_arr = ka < kh;
                const uint32_t q = KY::pos(kmin);
                const uint32_t now = KY::time(kmin);
                if (is_arr) {
                    ap += 1;
                    ka = ap < ae ? KY::make(s_a[ap], KY::c_init(bw_app(s_bw[ap])), ap) : KY::INF;
                } else {
                    pop();
                }
                const uint32_t m = s_mem[q];
                const uint32_t bw = s_bw[q];
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
                pc = wt == now ? counter : max(counter, cw);
                counter = pc + (start ? 1u : 0u);
                if ((is_arr && !enq && b == 0) || !is_arr) end_app(m, bw, now);
            }
            if (gs) grant_step();
            if (pp) push(pt, pc, pq);
            pp = false;
            if (fail) return false;
        }
        return !fail;
    }

    // unfinished waiters (never granted): NEVER ticks; returns their count
    __device__ __forceinline__ uint32_t finish_waiters() {
        for (uint32_t bits = qw; bits; bits &= bits - 1) {
            const uint32_t q = 32u * o.j + (uint32_t)(__ffs(bits) - 1);
            const uint32_t a = bw_app(s_bw[q]);
            if (gp) gp[a] = SG_NEVER;
            if (ep) ep[a] = SG_NEVER;
        }
        return osum(o, (uint32_t)__popc(qw));
    }
};

// ------------------------------------------------------------ staging
// Stage trace t into slot g (sgpu_stage256.cuh, in this warp's shared memory).
__device__ __forceinline__ void oct_stage(const OctParams& L, uint8_t* ws, uint32_t g, uint64_t t, uint32_t lane) {
    Slot256 S;
    S.s_a = reinterpret_cast<uint32_t*>(ws + L.off_a) + g * OctSlot::S32;
    S.s_mem = reinterpret_cast<uint32_t*>(ws + L.off_mem) + g * OctSlot::S32;
    S.s_bw = reinterpret_cast<uint32_t*>(ws + L.off_bw) + g * OctSlot::S32;
    S.s_por = reinterpret_cast<uint16_t*>(ws + L.off_por) + g * OctSlot::POR;
    S.s_lt = reinterpret_cast<uint16_t*>(ws + L.off_lt) + g * OctSlot::LTB;
    S.s_tbl = reinterpret_cast<uint32_t*>(ws + L.off_tbl) + g * OctSlot::TBL;
    S.s_cm = reinterpret_cast<uint32_t*>(ws + L.off_cm) + g * OctSlot::CM;
    S.meta = reinterpret_cast<uint32_t*>(ws + L.off_meta) + g * OctSlot::META;
    S.s_rank = reinterpret_cast<uint16_t*>(ws + L.off_scr);
    S.s_lt32 = nullptr;
    S.rs = 1;
    S.s_ms = nullptr;
    stage256<kOctLB>(L.sp, L.need_cls != 0, S, t, lane);
}

// ------------------------------------------------------------ kernel
// Groups of L.T traces are handed out by one atomic counter per stream
// (work_fetch / work_done, as the lane kernel).  Octet o simulates slot
// o / npol under policy slot o % npol; failed simulations are re-run by the
// whole warp with the exact TraceSim once the group's octets are done.
template <int MB>
__global__ void __launch_bounds__(kOctWarpsPerBlock * 32, MB) trace_sim_octet_kernel(const OctParams L) {
    const SimParams& P = L.sp;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * L.warp_bytes;
    const uint64_t n_groups = (P.n_traces + L.T - 1) / L.T;
    const uint32_t oi = lane >> 3;
    Oct o;
    o.base = oi * 8u;
    o.mask = 0xFFu << o.base;
    o.j = lane & 7u;
    const uint32_t g = oi / P.npol;
    const uint32_t pslot = oi - g * P.npol;
    const uint32_t policy = (P.policy_list >> (4 * pslot)) & 0xFu;

    uint64_t grp = work_fetch(P.work, lane);
    while (grp < n_groups) {
        const uint64_t next = work_fetch(P.work, lane);
        const uint64_t t0 = grp * L.T;
        const uint32_t gcount = (uint32_t)min((uint64_t)L.T, P.n_traces - t0);
        for (uint32_t s = 0; s < gcount; s++) oct_stage(L, ws, s, t0 + s, lane);
        bool fail = false;
        if (g < gcount) {
            const uint32_t* meta = reinterpret_cast<const uint32_t*>(ws + L.off_meta) + g * OctSlot::META;
            const uint64_t t = t0 + g;
            if (meta[1]) {
                fail = true;
            } else {
                OctSim sim;
                sim.o = o;
                sim.s_a = reinterpret_cast<const uint32_t*>(ws + L.off_a) + g * OctSlot::S32;
                sim.s_mem = reinterpret_cast<const uint32_t*>(ws + L.off_mem) + g * OctSlot::S32;
                sim.s_bw = reinterpret_cast<const uint32_t*>(ws + L.off_bw) + g * OctSlot::S32;
                sim.s_por = reinterpret_cast<const uint16_t*>(ws + L.off_por) + g * OctSlot::POR;
                sim.s_lt = reinterpret_cast<const uint16_t*>(ws + L.off_lt) + g * OctSlot::LTB;
                const uint32_t* prm = reinterpret_cast<const uint32_t*>(sim.s_lt + kOctLB);
                sim.lt_lo = prm[0];
                sim.lt_hi = prm[1];
                sim.lt_scale = prm[2];
                sim.s_tbl = reinterpret_cast<const uint32_t*>(ws + L.off_tbl) + g * OctSlot::TBL;
                sim.s_cm = reinterpret_cast<const uint32_t*>(ws + L.off_cm) + g * OctSlot::CM;
                uint64_t a0 = t * P.apps_per_trace;
                if (P.trace_offsets) a0 = P.trace_offsets[t] - P.trace_offsets[0];
                const uint64_t ob = (uint64_t)pslot * P.n_apps_total + a0;
                sim.gp = P.grant ? reinterpret_cast<uint32_t*>(P.grant) + ob : nullptr;
                sim.ep = P.end ? reinterpret_cast<uint32_t*>(P.end) + ob : nullptr;
                const uint32_t n = meta[0];
                if (sim.run(n, meta[2], policy, P.cap[0])) {
                    const uint32_t unf = sim.finish_waiters();
                    if (o.j == 0) {
                        const uint64_t seq = P.speedup ? ((uint64_t)meta[5] << 32 | meta[4]) : 0ull;
                        store_tick_record(P, (uint64_t)pslot * P.n_traces + t, n, sim.cap, sim.last, sim.mem_t,
                                          sim.I, sim.B, (int64_t)sim.used, sim.grants, sim.pops + n, sim.maxh,
                                          unf, 0u, seq);
                    }
                } else {
                    fail = true;
                }
            }
        }
        __syncwarp();
        // exact fallback: the whole warp re-simulates each failed (trace, policy)
        for (uint32_t fm = __ballot_sync(FULL, fail && (lane & 7u) == 0); fm; fm &= fm - 1) {
            const uint32_t fo = (uint32_t)(__ffs(fm) - 1) >> 3;
            const uint32_t fg = fo / P.npol, fp = fo - fg * P.npol;
            const uint64_t t = t0 + fg;
            uint64_t a0;
            uint32_t na;
            if (P.trace_offsets) {
                a0 = P.trace_offsets[t] - P.trace_offsets[0];
                na = (uint32_t)(P.trace_offsets[t + 1] - P.trace_offsets[t]);
            } else {
                a0 = t * P.apps_per_trace;
                na = P.apps_per_trace;
            }
            uint8_t* fb = ws;  // the whole warp region: the group's octets are done
            uint4* apps_s = reinterpret_cast<uint4*>(fb + P.off_app);
            for (uint32_t i = lane; i < na; i += 32) apps_s[i] = __ldg(reinterpret_cast<const uint4*>(P.apps + a0) + i);
            __syncwarp();
            TraceSim<TickTM, 8, false, false> sim(P, lane, fb, apps_s);
            sim.run(na, (P.policy_list >> (4 * fp)) & 0xFu, P.cap[0], nullptr);
            sim.finish((uint64_t)fp * P.n_traces + t, (uint64_t)fp * P.n_apps_total + a0, nullptr, nullptr);
            __syncwarp();
        }
        __syncwarp();
        grp = next;
    }
    work_done(P.work, lane);
}

static inline uint32_t align16o(uint32_t x) { return (x + 15u) & ~15u; }

// Octet path eligibility: T0 ticks mode, no event log, one device, traces of
// 129..256 apps (n_pad 256), < 2^32 traces.
bool octet_eligible(const SimParams& p, bool program_mode, bool f64) {
    if (program_mode || f64 || p.events != nullptr || p.ndev != 1 || p.npol > 4) return false;
    if (p.n_traces > 0xFFFFFFFFull) return false;
    return p.n_pad == kOctN;
}

cudaError_t launch_sim_octet(const SimParams& p, cudaStream_t stream, int* grid_out) {
    OctParams L;
    memset(&L, 0, sizeof(L));
    L.sp = p;
    sim_layout(L.sp, false, false, true);  // the fallback TraceSim, one app buffer
    L.T = p.npol >= 4 ? 1u : 4u / p.npol;
    L.need_cls = 0;
    for (uint32_t i = 0; i < p.npol; i++)
        if (((p.policy_list >> (4 * i)) & 0xFu) >= SG_POLICY_PFIFO) L.need_cls = 1;
    uint32_t off = 0;
    L.off_a = off;
    off = align16o(off + L.T * OctSlot::S32 * 4u);
    L.off_mem = off;
    off = align16o(off + L.T * OctSlot::S32 * 4u);
    L.off_bw = off;
    off = align16o(off + L.T * OctSlot::S32 * 4u);
    L.off_por = off;
    off = align16o(off + L.T * OctSlot::POR * 2u);
    L.off_lt = off;
    off = align16o(off + L.T * OctSlot::LTB * 2u);
    L.off_tbl = off;
    off = align16o(off + L.T * OctSlot::TBL * 4u);
    L.off_cm = off;
    off = align16o(off + L.T * OctSlot::CM * 4u);
    L.off_meta = off;
    off = align16o(off + L.T * OctSlot::META * 4u);
    L.off_scr = off;
    off = align16o(off + kOctN * 2u);
    L.warp_bytes = max(off, align16o(L.sp.warp_bytes));
    const size_t smem = (size_t)L.warp_bytes * kOctWarpsPerBlock;
    int sms = 0, per_sm = 0;
    cudaError_t err = kernel_config(reinterpret_cast<const void*>(trace_sim_octet_kernel<kOctMinBlocks>),
                                    kOctWarpsPerBlock * 32, smem, &per_sm, &sms);
    if (err != cudaSuccess) return err;
    const uint64_t groups = (p.n_traces + L.T - 1) / L.T;
    const uint64_t need = (groups + kOctWarpsPerBlock - 1) / kOctWarpsPerBlock;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (need < grid) grid = need;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    WorkLease lease;
    err = work_counters(stream, L.sp, 0, lease);
    if (err == cudaSuccess) {
        trace_sim_octet_kernel<kOctMinBlocks><<<(unsigned)grid, kOctWarpsPerBlock * 32, smem, stream>>>(L);
        err = cudaGetLastError();
    }
    return work_release(stream, lease, err);
}

}  // namespace sg
