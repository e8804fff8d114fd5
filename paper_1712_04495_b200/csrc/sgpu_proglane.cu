// sgpu_proglane.cu — K1 v6 `trace_prog_lane`: step-program batches (the
// reference's multi-phase AppProfiles, memshare/harness.py:39-83, flattened
// at 478-490) with one LANE per (trace, policy) simulation, 32 simulations
// per warp in SIMT.  The per-lane simulator is ProgLaneSim
// (sgpu_proglanesim.cuh); this file stages trace slots and launches.
//
// Eligible batches: step-program mode, integer ticks, no event log, one
// simulated device, at most 32 apps per trace.  A warp owns G = 32 / npol
// (at most 8) trace slots; each slot holds the trace's steps packed to 8 B
// (op << 62 | value), the first-step index and priority rank of every app.
// The heaps, program counters, held bytes and wait queues live in
// [slot][lane] columns (bank-conflict free whatever entry each lane
// touches).  Traces with more steps than a slot holds, and lanes whose times
// or push counters leave the key range, are re-simulated by the whole warp
// with the exact warp-per-trace TraceSim (program mode) once the group's
// lanes are done, in the same kernel.  Results are identical to the warp
// kernel's (tests/test_gpu_parity.py, both engines; tests/test_proglanesim_host.py
// checks ProgLaneSim against the oracle on CPU).
#include <cstring>

#include "sgpu_proglanesim.cuh"

namespace sg {

constexpr int kPLWarpsPerBlock = 2;
// steps per trace slot: the 12-app builtin workload (4 ara + 4 mummer + 4
// blast, 136 steps) fits either variant
template <int NA> struct ProgSlot { static constexpr uint32_t SCAP = NA <= 16 ? 192u : 256u; };

struct ProgLaneParams {
    SimParams sp;          // inputs/outputs + the fallback TraceSim layout
    uint32_t G;            // trace slots per warp
    uint32_t lpt;          // lanes per trace = npol
    // per-warp shared-memory layout (bytes)
    uint32_t off_st, off_first, off_prio, off_meta, off_heap, off_pc, off_held, off_q, warp_bytes;
};

struct ProgMeta {          // per slot
    uint32_t n, fail;
    uint64_t seq;          // cpu + busy ticks of the trace (speed-up vs sequential)
};

__device__ __forceinline__ void prog_trace_range(const SimParams& P, uint64_t t, uint64_t& a0, uint32_t& na) {
    if (P.trace_offsets) {
        const uint64_t o0 = P.trace_offsets[0];
        a0 = P.trace_offsets[t] - o0;
        na = (uint32_t)(P.trace_offsets[t + 1] - P.trace_offsets[t]);
    } else {
        a0 = t * P.apps_per_trace;
        na = P.apps_per_trace;
    }
}

// Stage trace t into slot g.  Warp-collective.
template <int NA>
__device__ __forceinline__ void prog_stage(const ProgLaneParams& L, uint8_t* ws, uint32_t g, uint64_t t,
                                           uint32_t lane) {
    const SimParams& P = L.sp;
    constexpr uint32_t SCAP = ProgSlot<NA>::SCAP;
    uint64_t a0;
    uint32_t na;
    prog_trace_range(P, t, a0, na);
    const uint32_t s0 = P.step_offsets[0];
    const uint32_t t0s = P.step_offsets[a0] - s0;
    const uint32_t ns = P.step_offsets[a0 + na] - s0 - t0s;
    ProgMeta* meta = reinterpret_cast<ProgMeta*>(ws + L.off_meta) + g;
    const bool fail = na > (uint32_t)NA || ns > SCAP;
    uint64_t seq = 0;
    if (!fail) {
        uint64_t* st = reinterpret_cast<uint64_t*>(ws + L.off_st) + g * SCAP;
        uint16_t* first = reinterpret_cast<uint16_t*>(ws + L.off_first) + g * (NA + 1);
        uint8_t* prio = ws + L.off_prio + g * NA;
        const uint4* src = reinterpret_cast<const uint4*>(P.steps) + t0s;
        for (uint32_t j = lane; j < ns; j += 32) {
            const uint4 v = __ldg(src + j);
            const uint64_t dur = ((uint64_t)v.w << 32) | v.z;
            st[j] = pack_step(v.x, v.y, dur);
            if (v.x == SG_OP_CPU || v.x == SG_OP_BUSY) seq += dur;
        }
        for (uint32_t i = lane; i <= na; i += 32) first[i] = (uint16_t)(P.step_offsets[a0 + i] - s0 - t0s);
        for (uint32_t i = lane; i < na; i += 32) prio[i] = (uint8_t)(P.apps[a0 + i].attr & 0xFFu);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) seq += __shfl_xor_sync(FULL, seq, o);
    if (lane == 0) *meta = ProgMeta{na, fail ? 1u : 0u, seq};
    __syncwarp();
}

template <int NA, int MB>
__global__ void __launch_bounds__(kPLWarpsPerBlock * 32, MB) trace_prog_lane_kernel(const ProgLaneParams L) {
    const SimParams& P = L.sp;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * L.warp_bytes;
    constexpr uint32_t SCAP = ProgSlot<NA>::SCAP;
    const uint64_t n_groups = (P.n_traces + L.G - 1) / L.G;
    const uint32_t g = lane / L.lpt;
    const uint32_t pslot = lane - g * L.lpt;
    const uint32_t policy = (P.policy_list >> (4 * pslot)) & 0xFu;
    const uint32_t cap = P.cap[0];

    uint64_t grp = work_fetch(P.work, lane);
    while (grp < n_groups) {
        const uint64_t next = work_fetch(P.work, lane);
        const uint64_t t0 = grp * L.G;
        const uint32_t gcount = (uint32_t)min((uint64_t)L.G, P.n_traces - t0);
        for (uint32_t s = 0; s < gcount; s++) prog_stage<NA>(L, ws, s, t0 + s, lane);
        bool fail = false;
        if (g < gcount) {
            const ProgMeta* meta = reinterpret_cast<const ProgMeta*>(ws + L.off_meta) + g;
            const uint64_t t = t0 + g;
            if (meta->fail) {
                fail = true;
            } else {
                uint64_t a0;
                uint32_t na;
                prog_trace_range(P, t, a0, na);
                ProgLaneSim<NA> sim(P);
                sim.st = reinterpret_cast<const uint64_t*>(ws + L.off_st) + g * SCAP;
                sim.first = reinterpret_cast<const uint16_t*>(ws + L.off_first) + g * (NA + 1);
                sim.prio = ws + L.off_prio + g * NA;
                sim.heap = reinterpret_cast<uint64_t*>(ws + L.off_heap) + lane;
                sim.pc = reinterpret_cast<uint16_t*>(ws + L.off_pc) + lane;
                sim.held = reinterpret_cast<int32_t*>(ws + L.off_held) + lane;
                sim.q = ws + L.off_q + lane;
                sim.out_base = (uint64_t)pslot * P.n_apps_total + a0;
                if (sim.run(na, policy, cap))
                    sim.finish((uint64_t)pslot * P.n_traces + t, meta->seq);
                else
                    fail = true;
            }
        }
        __syncwarp();
        // exact fallback: the whole warp re-simulates each failed lane with
        // the warp engine's program mode (steps read from global memory)
        for (uint32_t fm = __ballot_sync(FULL, fail); fm; fm &= fm - 1) {
            const uint32_t fl = __ffs(fm) - 1;
            const uint32_t fg = fl / L.lpt;
            const uint32_t fp = fl - fg * L.lpt;
            const uint64_t t = t0 + fg;
            uint64_t a0;
            uint32_t na;
            prog_trace_range(P, t, a0, na);
            uint8_t* fb = ws;  // the whole warp region: the group's lanes are done
            uint4* apps_s = reinterpret_cast<uint4*>(fb + P.off_app);
            const uint32_t s0 = P.step_offsets[0];
            __syncwarp();
            for (uint32_t i = lane; i < na; i += 32) {
                const uint32_t sb = P.step_offsets[a0 + i] - s0;
                const uint32_t se = P.step_offsets[a0 + i + 1] - s0;
                apps_s[i] = make_uint4(sb, se - sb, 0u, P.apps[a0 + i].attr);
            }
            __syncwarp();
            TraceSim<TickTM, 1, true> sim(P, lane, fb, apps_s);
            sim.run(na, (P.policy_list >> (4 * fp)) & 0xFu, cap, nullptr);
            sim.finish((uint64_t)fp * P.n_traces + t, (uint64_t)fp * P.n_apps_total + a0, nullptr, nullptr);
            __syncwarp();
            // restage the group's slots the fallback overlaid (later failed lanes
            // read nothing from them; the next group restages anyway)
        }
        __syncwarp();
        grp = next;
    }
    work_done(P.work, lane);
}

static inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

bool prog_lane_eligible(const SimParams& p, bool program_mode, bool f64, bool forced) {
    (void)forced;
    if (!program_mode || f64 || p.events != nullptr || p.ndev != 1) return false;
    return p.n_pad <= 32u && p.max_apps <= 32u;
}

template <int NA>
static void prog_layout(ProgLaneParams& L) {
    constexpr uint32_t SCAP = ProgSlot<NA>::SCAP;
    uint32_t o = 0;
    L.off_st = o;
    o = align16(o + L.G * SCAP * 8u);
    L.off_first = o;
    o = align16(o + L.G * (NA + 1u) * 2u);
    L.off_prio = o;
    o = align16(o + L.G * NA);
    L.off_meta = o;
    o = align16(o + L.G * (uint32_t)sizeof(ProgMeta));
    L.off_heap = o;
    o = align16(o + NA * 32u * 8u);
    L.off_pc = o;
    o = align16(o + NA * 32u * 2u);
    L.off_held = o;
    o = align16(o + NA * 32u * 4u);
    L.off_q = o;
    o = align16(o + NA * 32u);
    // the fallback TraceSim overlays the whole region
    L.warp_bytes = max(o, align16(L.sp.warp_bytes));
}

template <int NA, int MB>
static cudaError_t launch_prog_t(ProgLaneParams& L, cudaStream_t stream, int* grid_out) {
    prog_layout<NA>(L);
    auto kern = trace_prog_lane_kernel<NA, MB>;
    const uint32_t wpb = kPLWarpsPerBlock;
    const size_t smem = (size_t)L.warp_bytes * wpb;
    int sms = 0, per_sm = 0;
    cudaError_t err = kernel_config(reinterpret_cast<const void*>(kern), wpb * 32, smem, &per_sm, &sms);
    if (err != cudaSuccess) return err;
    const uint64_t groups = (L.sp.n_traces + L.G - 1) / L.G;
    const uint64_t need = (groups + wpb - 1) / wpb;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (need < grid) grid = need;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    kern<<<(unsigned)grid, wpb * 32, smem, stream>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_sim_prog_lane(const SimParams& p, cudaStream_t stream, int* grid_out) {
    ProgLaneParams L;
    L.sp = p;
    L.lpt = p.npol;
    L.G = min(32u / L.lpt, 8u);
    L.sp.n_pad = 32;
    sim_layout(L.sp, true, false);  // the fallback's layout (K = 1, program mode)
    WorkLease lease;
    cudaError_t err = work_counters(stream, L.sp, 0, lease);
    if (err == cudaSuccess) {
        if (p.max_apps <= 16) err = launch_prog_t<16, 8>(L, stream, grid_out);
        else err = launch_prog_t<32, 6>(L, stream, grid_out);
    }
    return work_release(stream, lease, err);
}

}  // namespace sg
