// sgpu_lane.cu — K1 v4 `trace_sim_lane`: one LANE simulates one (trace,
// device, policy) of a T0 (burst) batch, 32 simulations per warp in SIMT.
//
// Same semantics as trace_sim_kernel (sgpu_sim.cu),
// restated for a single thread.  The T0 shape (cpu(arrival) -> alloc ->
// busy -> free, memshare/harness.py:478-490) makes three reductions exact:
//
//  * Arrival stream.  The initial pops run in index order at t = 0
//    (harness.py:560-562); an app with arrival a > 0 only pushes (a, c), with
//    c increasing in the app index, so arrivals pop in (a, index) order: a
//    per-trace sort, shared by every lane of the trace, replaces those heap
//    entries.  Heap counters are restated as order-preserving virtual
//    counters: the initial pop of app i owns the counter block [i << LOGN,
//    (i + 1) << LOGN) (its arrival push, or the pushes its inline run at t = 0
//    makes), and every later push counts up from n << LOGN.  Comparing
//    (t, virtual counter) is therefore the reference's (t, counter) order
//    (harness.py:505-508, 563-565).
//  * Wait queue.  An app enqueues at most once, at its arrival pop, so its
//    queue position is its rank in the arrival order (FIFO/MMU), or its rank
//    in (priority desc, arrival order) for the priority policies (the class
//    order of policy.py:58-63).  The queue is a presence bitmask over those
//    static positions, in registers; select_grants (policy.py:52-74) is a
//    scan over set bits: FIFO stops at the first misfit, MMU skips it, the
//    priority kinds scan only the top class [first waiting position, class
//    end) and loop to the next class when it drained (harness.py:545-558).
//  * Heap.  Only busy-end and wake-up entries remain: a per-lane binary heap
//    in shared memory, laid out [slot][lane] so every access of a warp is
//    bank-conflict free whatever slot each lane touches.
//
// Lanes that cannot take this path (heap capacity exceeded, or a trace
// whose times could leave the 32-bit tick range) are re-simulated by the
// whole warp with the exact warp-per-trace TraceSim (sgpu_tracesim.cuh)
// right after, in the same kernel: no host round trip, no extra buffers.
#include "sgpu_tracesim.cuh"

namespace sg {

constexpr uint32_t kLaneHeap = 32;          // heap slots per lane
constexpr uint32_t kKindWake = 0, kKindBusyEnd = 1, kKindArrival = 2;
constexpr uint64_t kInf = ~0ull;

struct LaneParams {
    SimParams sp;          // inputs/outputs + the fallback TraceSim layout (off_* relative to off_fb)
    uint32_t G;            // traces per block group (32 / ndev)
    uint32_t need_cls;     // some policy is priority-aware: build the class order
    uint32_t off_rec, off_cls, off_meta;  // block-shared staging (G trace slots)
    uint32_t off_fb, fb_bytes;            // per-warp region: heap / scratch / fallback
    uint32_t block_bytes;
};

// meta per trace slot (u16): [0] n, [1] big, [2..10] device bounds, [11..18] a==0 counts
constexpr uint32_t kMetaU16 = 32;

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
    const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m);
    const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m);
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

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int K>
struct LaneSim {
    static constexpr uint32_t N = 32u * K;
    static constexpr uint32_t NW = (N + 63u) / 64u;  // queue mask words
    static constexpr uint32_t LOGN = K == 1 ? 5 : K == 2 ? 6 : K == 4 ? 7 : 8;

    const SimParams& P;
    const uint4* rec;      // trace slot records, arrival order
    const uint32_t* cls;   // class position -> apos | class_end << 16
    uint64_t* heap;        // this lane's column: heap[h * 32]
    uint64_t out_base;     // grant/end index of app 0 of the trace under this policy
    uint32_t cap, used;
    bool prio_pol, mmu, fail;
    uint64_t mask[NW];
    uint32_t hs;
    uint64_t kh;           // heap top (kInf when empty)
    uint32_t counter;
    // statistics (harness.py:373-461 integer forms)
    uint32_t last, mem_t, busy_prev, B;
    uint64_t I;
    int32_t busy_level, holders;
    uint32_t maxh, grants, pops;

    __device__ __forceinline__ LaneSim(const SimParams& p) : P(p) {}

    __device__ __forceinline__ void mem_point(uint32_t now) {
        I += (uint64_t)used * (now - mem_t);
        mem_t = now;
    }
    __device__ __forceinline__ void busy_point(uint32_t now, int32_t delta) {
        B += busy_level > 0 ? now - busy_prev : 0u;
        busy_prev = now;
        busy_level += delta;
    }

    // ------------------------------------------------------------ heap
    __device__ __forceinline__ void push(uint32_t t, uint32_t kind, uint32_t q) {
        if (hs >= kLaneHeap) { fail = true; return; }
        const uint64_t key = ((uint64_t)t << 32) | (counter << 10) | (kind << 8) | q;
        counter += 1;
        uint32_t i = hs++;
        while (i > 0) {
            const uint32_t par = (i - 1) >> 1;
            const uint64_t pk = heap[par * 32];
            if (pk < key) break;
            heap[i * 32] = pk;
            i = par;
        }
        heap[i * 32] = key;
        if (i == 0) kh = key;
    }
    __device__ __forceinline__ void pop() {
        hs -= 1;
        if (hs == 0) { kh = kInf; return; }
        const uint64_t lastk = heap[hs * 32];
        uint32_t i = 0;
        uint64_t top = lastk;
        bool first = true;
        while (true) {
            uint32_t c = 2 * i + 1;
            if (c >= hs) break;
            uint64_t ck = heap[c * 32];
            if (c + 1 < hs) {
                const uint64_t c2 = heap[(c + 1) * 32];
                if (c2 < ck) { ck = c2; c += 1; }
            }
            if (lastk < ck) break;
            heap[i * 32] = ck;
            if (first) top = ck;
            first = false;
            i = c;
        }
        heap[i * 32] = lastk;
        kh = top;
    }

    // ------------------------------------------------------- wait queue
    __device__ __forceinline__ void enqueue(uint32_t q) {
#pragma unroll
        for (uint32_t w = 0; w < NW; w++)
            if (w == (q >> 6)) mask[w] |= 1ull << (q & 63u);
    }
    __device__ __forceinline__ uint32_t q_apos(uint32_t q) const {
        return prio_pol ? (cls[q] & 0xFFFFu) : q;
    }

    // grant_waiters (harness.py:545-558) + select_grants (policy.py:52-74)
    __device__ __forceinline__ void grant_waiters(uint32_t now) {
        while (true) {
            // first waiting position
            uint32_t q0 = N;
#pragma unroll
            for (int w = NW - 1; w >= 0; w--)
                if (mask[w]) q0 = 64u * w + (__ffsll((long long)mask[w]) - 1);
            if (q0 == N) return;
            const uint32_t qend = prio_pol ? (cls[q0] >> 16) : N;
            const uint32_t budget0 = cap - used;
            uint32_t budget = budget0, g = 0;
            bool left = false, stop = false;
#pragma unroll
            for (uint32_t w = 0; w < NW; w++) {
                uint64_t bits = mask[w];
                while (bits && !stop) {
                    const uint32_t q = 64u * w + (__ffsll((long long)bits) - 1);
                    bits &= bits - 1;
                    if (q >= qend) { stop = true; break; }
                    const uint32_t apos = q_apos(q);
                    const uint32_t m = rec[apos].y;
                    if (m <= budget) {
                        budget -= m;
                        g += 1;
                        mask[w] &= ~(1ull << (q & 63u));
                        push(now, kKindWake, apos);
                        if (fail) return;
                    } else {
                        left = true;
                        if (!mmu) stop = true;
                    }
                }
            }
            if (g) {
                mem_point(now);
                used += budget0 - budget;
                holders += (int32_t)g;
                maxh = max(maxh, (uint32_t)holders);
                grants += g;
            }
            if (!prio_pol || g == 0 || left) return;
        }
    }

    // --------------------------------------------------------- advance
    __device__ __forceinline__ void end_app(const uint4& r, uint32_t now) {
        if (r.y) {  // free -> grant_waiters (harness.py:537-542)
            mem_point(now);
            used -= r.y;
            holders -= 1;
            grant_waiters(now);
        }
        const uint64_t o = out_base + (r.w & kAppMask);  // end (harness.py:543)
        if (P.end) reinterpret_cast<uint32_t*>(P.end)[o] = now;
        // the grant is the busy start: busy runs [grant, grant + busy]
        if (P.grant) reinterpret_cast<uint32_t*>(P.grant)[o] = r.y ? now - r.z : SG_NEVER;
    }
    __device__ __forceinline__ void run_from_busy(uint32_t q, const uint4& r, uint32_t now) {
        if (r.z) {  // busy (harness.py:514-520)
            busy_point(now, +1);
            push(now + r.z, kKindBusyEnd, q);
            return;
        }
        end_app(r, now);
    }
    __device__ __forceinline__ void arrive(uint32_t q, const uint4& r, uint32_t now) {
        if (r.y) {
            if (r.y <= cap - used) {  // arrival bypass (harness.py:521-531)
                mem_point(now);
                used += r.y;
                holders += 1;
                maxh = max(maxh, (uint32_t)holders);
                grants += 1;
            } else {                  // wait (harness.py:532-536)
                enqueue(prio_pol ? ((r.w >> 10) & 0x3FFu) : q);
                return;
            }
        }
        run_from_busy(q, r, now);
    }

    // Simulate device range [s, e) of the slot's arrival order (z apps arrive
    // at t = 0).  Returns false if this lane must be re-run by the fallback.
    __device__ __forceinline__ bool run(uint32_t n_trace, uint32_t s, uint32_t e, uint32_t z,
                                        uint32_t policy, uint32_t cap_mib) {
        cap = cap_mib;
        used = 0;
        prio_pol = policy >= SG_POLICY_PFIFO;
        mmu = (policy & 1u) != 0;
        fail = false;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) mask[w] = 0;
        hs = 0;
        kh = kInf;
        last = mem_t = busy_prev = B = 0;
        I = 0;
        busy_level = holders = 0;
        maxh = grants = pops = 0;
        // initial pops at t = 0: apps without a cpu step run inline, in index
        // order, each in its own virtual counter block
        for (uint32_t q = s; q < s + z; q++) {
            const uint4 r = rec[q];
            counter = (r.w & kAppMask) << LOGN;
            arrive(q, r, 0u);
            if (fail) return false;
        }
        counter = n_trace << LOGN;
        uint32_t ap = s + z;
        uint4 ra = make_uint4(0, 0, 0, 0);
        uint64_t ka = kInf;
        if (ap < e) {
            ra = rec[ap];
            ka = ((uint64_t)ra.x << 32) | (((ra.w & kAppMask) << LOGN) << 10) | (kKindArrival << 8) | ap;
        }
        while (true) {
            if (ka < kh) {
                const uint32_t q = ap;
                const uint4 r = ra;
                const uint32_t now = ra.x;
                ap += 1;
                if (ap < e) {
                    ra = rec[ap];
                    ka = ((uint64_t)ra.x << 32) | (((ra.w & kAppMask) << LOGN) << 10) | (kKindArrival << 8) | ap;
                } else {
                    ka = kInf;
                }
                pops += 1;
                last = now;
                arrive(q, r, now);
            } else if (kh != kInf) {
                const uint64_t key = kh;
                pop();
                const uint32_t q = (uint32_t)key & 0xFFu;
                const uint32_t now = (uint32_t)(key >> 32);
                const uint4 r = rec[q];
                pops += 1;
                last = now;
                if (((uint32_t)key >> 8) & 1u) {  // busy end
                    busy_point(now, -1);
                    end_app(r, now);
                } else {                          // granted waiter resumes
                    run_from_busy(q, r, now);
                }
            } else {
                break;
            }
            if (fail) return false;
        }
        return true;
    }

    __device__ __forceinline__ void finish(uint64_t srec, uint32_t nd) {
        uint32_t unf = 0;
#pragma unroll
        for (uint32_t w = 0; w < NW; w++) {
            for (uint64_t bits = mask[w]; bits; bits &= bits - 1) {
                const uint32_t q = 64u * w + (__ffsll((long long)bits) - 1);
                const uint64_t o = out_base + (rec[q_apos(q)].w & kAppMask);
                if (P.grant) reinterpret_cast<uint32_t*>(P.grant)[o] = SG_NEVER;
                if (P.end) reinterpret_cast<uint32_t*>(P.end)[o] = SG_NEVER;
                unf += 1;
            }
        }
        store_tick_record(P, srec, nd, cap, last, mem_t, I, B, (int64_t)used, grants, pops + nd,
                          maxh, unf, 0u);
    }
};

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

// Stage trace t into slot g (scratch: the calling warp's fb region): records in (device, arrival, index) order, the
// class order for the priority policies, device bounds.  Warp-collective.
template <int K>
__device__ __forceinline__ void stage_trace(const LaneParams& L, uint8_t* ws, uint8_t* fb, uint32_t g,
                                            uint64_t t, uint32_t lane) {
    const SimParams& P = L.sp;
    constexpr uint32_t N = 32u * K;
    uint64_t a0;
    uint32_t na;
    lane_trace_range(P, t, a0, na);
    uint4* raw = reinterpret_cast<uint4*>(fb);
    uint16_t* cpos = reinterpret_cast<uint16_t*>(fb + N * 16u);
    uint4* rec = reinterpret_cast<uint4*>(ws + L.off_rec) + g * N;
    uint32_t* cls = reinterpret_cast<uint32_t*>(ws + L.off_cls) + g * N;
    uint16_t* meta = reinterpret_cast<uint16_t*>(ws + L.off_meta) + g * kMetaU16;
    const uint32_t ndev = P.ndev;

    uint64_t key[K];
    bool big = false;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        key[k] = kInf;
        if (i < na) {
            const uint4 f = __ldg(reinterpret_cast<const uint4*>(P.apps + a0) + i);
            raw[i] = f;
            uint32_t dv = ndev > 1 ? (f.w >> 8) & 0xFFu : 0u;
            if (dv >= ndev) dv = 0;
            key[k] = ((uint64_t)dv << 42) | ((uint64_t)f.x << 10) | i;
            big = big || f.x >= (1u << 31) || f.z >= (1u << 21);
        }
    }
    big = __any_sync(FULL, big);
    warp_bitonic_sort<K>(key, lane);
    __syncwarp();
    // device bounds and arrivals at t = 0, per device
    uint32_t cnt_d = 0, z_d = 0;  // lane d < ndev holds device d's counts
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
    if (L.need_cls) {
        // class order: (device, priority desc, arrival position)
        uint32_t ck[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const uint32_t e = (uint32_t)k * 32u + lane;
            ck[k] = ~0u;
            if (key[k] != kInf) {
                const uint32_t i = (uint32_t)key[k] & kAppMask;
                const uint32_t prio = raw[i].w & 0xFFu;
                ck[k] = ((uint32_t)(key[k] >> 42) << 18) | ((255u - prio) << 10) | e;
            }
        }
        warp_bitonic_sort<K>(ck, lane);
        // class boundaries as a bitmask over positions
        uint32_t bw[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            uint32_t prev = __shfl_up_sync(FULL, ck[k], 1);
            const uint32_t pk = k > 0 ? __shfl_sync(FULL, ck[k > 0 ? k - 1 : 0], 31) : ~0u;
            if (lane == 0) prev = pk;
            const bool valid = ck[k] != ~0u;
            bw[k] = __ballot_sync(FULL, valid && (prev == ~0u || (prev >> 10) != (ck[k] >> 10)));
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            if (ck[k] != ~0u) {
                const uint32_t c = (uint32_t)k * 32u + lane;
                uint32_t cend = na;
                bool found = false;
                const uint32_t above = lane == 31 ? 0u : (bw[k] & ~((2u << lane) - 1u));
                if (above) { cend = (uint32_t)k * 32u + __ffs(above) - 1; found = true; }
#pragma unroll
                for (int k2 = k + 1; k2 < K; k2++)
                    if (!found && bw[k2]) { cend = (uint32_t)k2 * 32u + __ffs(bw[k2]) - 1; found = true; }
                const uint32_t apos = ck[k] & 0x3FFu;
                cls[c] = apos | (cend << 16);
                cpos[apos] = (uint16_t)c;
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t e = (uint32_t)k * 32u + lane;
        if (key[k] != kInf) {
            const uint32_t i = (uint32_t)key[k] & kAppMask;
            const uint4 f = raw[i];
            const uint32_t cp = L.need_cls ? cpos[e] : 0u;
            rec[e] = make_uint4(f.x, f.y, f.z, i | (cp << 10) | ((f.w & 0xFFu) << 20));
        }
    }
    // meta: exclusive scan of the device counts
    uint32_t incl = cnt_d;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    if (lane < ndev) {
        meta[3 + lane] = (uint16_t)incl;
        meta[11 + lane] = (uint16_t)z_d;
    }
    if (lane == 0) {
        meta[0] = (uint16_t)na;
        meta[1] = big ? 1 : 0;
        meta[2] = 0;
    }
    __syncwarp();
}

// Block = one warp per requested policy; the block stages G = 32 / ndev
// traces at a time into shared memory (the warps split the traces), then
// warp w simulates policy w of all of them, lane = (trace slot, device).
// Every lane of a warp runs the same policy, so their control flow differs
// only by the trace data.
template <int K>
__global__ void __launch_bounds__(128) trace_sim_lane_kernel(const LaneParams L) {
    const SimParams& P = L.sp;
    constexpr uint32_t N = 32u * K;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t npol = P.npol;
    const uint32_t ndev = P.ndev;
    uint8_t* fb = smem + L.off_fb + (size_t)warp * L.fb_bytes;
    const uint64_t n_groups = (P.n_traces + L.G - 1) / L.G;

    // lane -> (slot, device); warp -> policy slot
    const uint32_t g = lane / ndev;
    const uint32_t d = lane - g * ndev;
    const uint32_t pslot = warp;
    const uint32_t policy = (P.policy_list >> (4 * pslot)) & 0xFu;
    uint32_t cap_d = P.cap[0];
#pragma unroll
    for (uint32_t j = 1; j < SG_MAX_DEV; j++)
        if (d == j) cap_d = P.cap[j];

    for (uint64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
        const uint64_t t0 = grp * L.G;
        const uint32_t gcount = (uint32_t)min((uint64_t)L.G, P.n_traces - t0);
        for (uint32_t s = warp; s < gcount; s += npol) stage_trace<K>(L, smem, fb, s, t0 + s, lane);
        // warm L2 with the next group's records while this one simulates
        if (warp == 0 && grp + gridDim.x < n_groups && !P.trace_offsets) {
            const uint64_t nt0 = (grp + gridDim.x) * L.G;
            const uint64_t nb = min((uint64_t)L.G, P.n_traces - nt0) * P.apps_per_trace * 16u;
            const uint8_t* base = reinterpret_cast<const uint8_t*>(P.apps + nt0 * P.apps_per_trace);
            for (uint64_t off = (uint64_t)lane * 128u; off < nb; off += 32u * 128u) prefetch_l2(base + off);
        }
        __syncthreads();

        bool fail = false;
        if (g < gcount) {
            const uint64_t t = t0 + g;
            const uint16_t* meta = reinterpret_cast<const uint16_t*>(smem + L.off_meta) + g * kMetaU16;
            const uint32_t na = meta[0];
            if (meta[1]) {
                fail = true;
            } else {
                const uint32_t s0 = meta[2 + d], s1 = meta[3 + d], z = meta[11 + d];
                uint64_t a0;
                uint32_t na_unused;
                lane_trace_range(P, t, a0, na_unused);
                LaneSim<K> sim(P);
                sim.rec = reinterpret_cast<const uint4*>(smem + L.off_rec) + g * N;
                sim.cls = reinterpret_cast<const uint32_t*>(smem + L.off_cls) + g * N;
                sim.heap = reinterpret_cast<uint64_t*>(fb) + lane;
                sim.out_base = (uint64_t)pslot * P.n_apps_total + a0;
                if (sim.run(na, s0, s1, z, policy, cap_d))
                    sim.finish(((uint64_t)pslot * P.n_traces + t) * ndev + d, s1 - s0);
                else
                    fail = true;
            }
        }
        __syncwarp();
        // exact fallback: the whole warp re-simulates each failed lane
        for (uint32_t fm = __ballot_sync(FULL, fail); fm; fm &= fm - 1) {
            const uint32_t fl = __ffs(fm) - 1;
            const uint32_t fg = fl / ndev;
            const uint32_t fd = fl - fg * ndev;
            const uint64_t t = t0 + fg;
            uint64_t a0;
            uint32_t na;
            lane_trace_range(P, t, a0, na);
            uint4* apps_s = reinterpret_cast<uint4*>(fb + P.off_app);
            for (uint32_t i = lane; i < na; i += 32)
                apps_s[i] = __ldg(reinterpret_cast<const uint4*>(P.apps + a0) + i);
            __syncwarp();
            const uint4* sub = apps_s;
            const uint16_t* idx = nullptr;
            uint32_t nd = na;
            if (ndev > 1) {
                uint4* s_sub = reinterpret_cast<uint4*>(fb + P.off_sub);
                uint16_t* s_idx = reinterpret_cast<uint16_t*>(fb + P.off_idx);
                nd = build_subtrace(apps_s, na, fd, ndev, s_sub, s_idx, lane);
                sub = s_sub;
                idx = s_idx;
            }
            uint32_t fcap = P.cap[0];
#pragma unroll
            for (uint32_t j = 1; j < SG_MAX_DEV; j++)
                if (fd == j) fcap = P.cap[j];
            TraceSim<TickTM, K, false> sim(P, lane, fb, sub);
            sim.run(nd, policy, fcap, nullptr);
            sim.finish(((uint64_t)pslot * P.n_traces + t) * ndev + fd,
                       (uint64_t)pslot * P.n_apps_total + a0, idx, nullptr);
        }
        __syncthreads();
    }
}

static inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Lane path eligibility: T0 ticks mode, no event log, <= 256 apps per trace.
bool lane_eligible(const SimParams& p, bool program_mode, bool f64) {
    return !program_mode && !f64 && p.events == nullptr && p.n_pad <= 256 && p.npol <= 4 &&
           p.ndev <= 32;
}

template <int K>
static cudaError_t launch_lane_t(LaneParams& L, cudaStream_t stream, int* grid_out) {
    auto kern = trace_sim_lane_kernel<K>;
    const uint32_t threads = 32u * L.sp.npol;
    const size_t smem = L.block_bytes;
    if (smem > 227u * 1024u) return cudaErrorInvalidConfiguration;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t groups = (L.sp.n_traces + L.G - 1) / L.G;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (groups < grid) grid = groups;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    kern<<<(unsigned)grid, threads, smem, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_sim_lane(const SimParams& p, cudaStream_t stream, int* grid_out) {
    LaneParams L;
    L.sp = p;
    const uint32_t N = p.n_pad;
    L.G = 32u / p.ndev;
    L.need_cls = 0;
    for (uint32_t i = 0; i < p.npol; i++)
        if (((p.policy_list >> (4 * i)) & 0xFu) >= SG_POLICY_PFIFO) L.need_cls = 1;
    // per-warp region: heap / staging scratch / fallback TraceSim layout (relative to it)
    sim_layout(L.sp, false, false);
    uint32_t fb = L.sp.warp_bytes;
    fb = max(fb, kLaneHeap * 32u * 8u);
    fb = max(fb, N * 16u + N * 2u);
    L.fb_bytes = align16(fb);
    uint32_t o = 0;
    L.off_rec = o;
    o = align16(o + L.G * N * 16u);
    L.off_cls = o;
    o = align16(o + (L.need_cls ? L.G * N * 4u : 0u));
    L.off_meta = o;
    o = align16(o + L.G * kMetaU16 * 2u);
    L.off_fb = o;
    o += L.fb_bytes * p.npol;
    L.block_bytes = o;
    switch (N / 32) {
        case 1: return launch_lane_t<1>(L, stream, grid_out);
        case 2: return launch_lane_t<2>(L, stream, grid_out);
        case 4: return launch_lane_t<4>(L, stream, grid_out);
        case 8: return launch_lane_t<8>(L, stream, grid_out);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sg
