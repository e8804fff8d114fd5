// sgpu_lane256.cu — K1 v9 `trace_sim_lane256`: one LANE simulates one
// (trace, policy) of a T0 batch of 129..256-app single-device traces, 32
// simulations per warp, with the staged trace tables in GLOBAL memory.
//
// A 256-app trace's staged state (records in arrival order, a fit table of
// 256-bit rows, u16 rank tables, class masks: ~6.6 KB) is too large for a
// lane-per-simulation kernel to keep 16 of them per warp in shared memory
// (the octet kernel, v8, keeps two and spreads each simulation over eight
// lanes instead, which serialises the four octets of a warp).  Here the
// warp stages its traces into a per-warp slot of a global scratch buffer
// (sgpu_stage256.cuh, the octet kernel's staging with LaneSim's bucket
// count) and each lane runs LaneSim<8> (sgpu_lanesim.cuh, the lane kernel's
// simulator with four-word masks, u16 rank tables and a 32-key three-level
// heap — checked on the host against the oracle by
// tests/test_lanesim_host.py) reading its trace from there: the random
// per-event reads of the trace are L1 / L2 hits, and only the heaps
// (32 keys per lane) live in shared memory.  Event order, virtual counters,
// grant-time pushes: LaneSim's (memshare/harness.py:475-572, policy.py:52-74).
// A lane that cannot take this path (a 33rd concurrent busy end, counters
// past the key field, > 8 priority classes, priorities >= 32, times near the
// 32-bit range) is re-simulated by the whole warp with the exact TraceSim
// in shared memory, in the same kernel.
#include <cstring>

#include "sgpu_lanesim.cuh"
#include "sgpu_stage256.cuh"

namespace sg {

constexpr uint32_t kL256N = 256;
constexpr uint32_t kL256Heap = 32;     // heap keys per lane (4-ary, three levels)
constexpr uint32_t kL256FS = 8;     // fit-table stride: 8 (1 KB less per slot than 4; C3 165.9 -> 162.9 ms)  // fit-table stride (the table lives in global memory)
constexpr uint32_t kL256LB = 256;     // rank-lookup buckets (about one request each)
constexpr bool kL256Sorted = true;    // requests in rank order: one load per rank-lookup step
constexpr int kL256WarpsPerBlock = 2;
constexpr int kL256MinBlocks = 6;      // 12 warps/SM (register cap 168)

// Per-slot layout of the global scratch (bytes, 16-aligned offsets).
struct L256Slot {
    static constexpr uint32_t S32 = (kL256N + 1) * 4;
    static constexpr uint32_t A = 0;
    static constexpr uint32_t MEM = (A + S32 + 15) & ~15u;   // (request, busy word) pairs, N + 1 of them
    static constexpr uint32_t BW = MEM + 4;
    static constexpr uint32_t POR = (MEM + 2 * S32 + 15) & ~15u;
    static constexpr uint32_t LT = (POR + (kL256N + 8) * 2 + 15) & ~15u;
    static constexpr uint32_t TBL = (LT + kL256LB * 4 + 12 + 15) & ~15u;  // packed u32 bucket entries + 3 u32
    static constexpr uint32_t CM = (TBL + (kL256N / kL256FS + 1) * 32 + 15) & ~15u;
    static constexpr uint32_t META = (CM + kStage256MaxCls * 32 + 15) & ~15u;
    static constexpr uint32_t MS = (META + 32 + 15) & ~15u;
    static constexpr uint32_t BYTES = (MS + (kL256N + 4) * 4 + 127) & ~127u;  // staging rank scratch: shared
};

struct L256Params {
    SimParams sp;          // inputs/outputs + the fallback TraceSim layout (single app buffer, shared memory)
    uint8_t* scratch;      // global: per warp, G slots of L256Slot::BYTES
    uint32_t G;            // traces per warp (32 / npol, at most 16)
    uint32_t need_cls;
    uint32_t warp_bytes;   // shared memory per warp: max(heaps, fallback TraceSim)
};

__device__ __forceinline__ Slot256 l256_slot(uint8_t* base) {
    Slot256 S;
    S.s_a = reinterpret_cast<uint32_t*>(base + L256Slot::A);
    S.s_mem = reinterpret_cast<uint32_t*>(base + L256Slot::MEM);
    S.s_bw = reinterpret_cast<uint32_t*>(base + L256Slot::BW);
    S.s_por = reinterpret_cast<uint16_t*>(base + L256Slot::POR);
    S.s_lt = reinterpret_cast<uint16_t*>(base + L256Slot::LT);
    S.s_tbl = reinterpret_cast<uint32_t*>(base + L256Slot::TBL);
    S.s_cm = reinterpret_cast<uint32_t*>(base + L256Slot::CM);
    S.meta = reinterpret_cast<uint32_t*>(base + L256Slot::META);
    S.s_rank = nullptr;  // set by the caller (the warp's shared region while staging)
    S.s_lt32 = reinterpret_cast<uint32_t*>(base + L256Slot::LT);
    S.rs = 2;
    S.s_ms = kL256Sorted ? reinterpret_cast<uint32_t*>(base + L256Slot::MS) : nullptr;
    return S;
}

// One lane's simulation of (trace t, policy) from staged slot S.
template <bool NARROW>
__device__ __forceinline__ bool l256_run(const SimParams& P, const Slot256& S, uint8_t* ws, uint32_t pslot,
                                         uint32_t policy, uint64_t t, uint32_t lane, uint32_t runmask) {
    using Sim = LaneSim<8, NARROW, kL256Heap, kL256FS, true, true, kL256LB, 2>;
    const uint32_t na = S.meta[0], z = S.meta[2];
    Sim sim(P);
    sim.smask = runmask;  // the lanes of this warp in the main loop: they re-converge per iteration
    sim.s_a = S.s_a;
    sim.s_mem = S.s_mem;
    sim.s_bw = S.s_bw;
    sim.s_por = S.s_por;
    sim.s_lt = S.s_lt;
    sim.s_ms = S.s_ms;
    sim.s_lt32 = S.s_lt32;
    const uint32_t* prm = S.s_lt32 + kL256LB;
    sim.lt_lo = prm[0];
    sim.lt_hi = prm[1];
    sim.lt_scale = prm[2];
    sim.s_t4 = reinterpret_cast<const uint64_t*>(S.s_tbl);
    sim.s_cm = reinterpret_cast<const uint64_t*>(S.s_cm);
    sim.ncls = S.meta[3];
    sim.heap = reinterpret_cast<typename Sim::Key*>(ws) + lane;
    uint64_t a0 = t * P.apps_per_trace;
    if (P.trace_offsets) a0 = P.trace_offsets[t] - P.trace_offsets[0];
    const uint64_t ob = (uint64_t)pslot * P.n_apps_total + a0;
    sim.gp = P.grant ? reinterpret_cast<uint32_t*>(P.grant) + ob : nullptr;
    sim.ep = P.end ? reinterpret_cast<uint32_t*>(P.end) + ob : nullptr;
    if (!sim.run(na, 0u, na, z, policy, P.cap[0])) return false;
    const uint64_t seq = P.speedup ? ((uint64_t)S.meta[5] << 32 | S.meta[4]) : 0ull;
    sim.finish((uint64_t)pslot * P.n_traces + t, na, 0u, seq);
    return true;
}

// Groups of G traces are handed out by one atomic counter per stream
// (work_fetch / work_done).  Lane l simulates slot l / npol under policy
// slot l % npol.
template <int MB>
__global__ void __launch_bounds__(kL256WarpsPerBlock * 32, MB) trace_sim_lane256_kernel(const L256Params L) {
    const SimParams& P = L.sp;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * L.warp_bytes;
    uint8_t* scr = L.scratch + ((size_t)blockIdx.x * kL256WarpsPerBlock + warp) * L.G * L256Slot::BYTES;
    const uint64_t n_groups = (P.n_traces + L.G - 1) / L.G;
    const uint32_t g = lane / P.npol;
    const uint32_t pslot = lane - g * P.npol;
    const uint32_t policy = (P.policy_list >> (4 * pslot)) & 0xFu;

    uint64_t grp = work_fetch(P.work, lane);
    while (grp < n_groups) {
        const uint64_t next = work_fetch(P.work, lane);
        const uint64_t t0 = grp * L.G;
        const uint32_t gcount = (uint32_t)min((uint64_t)L.G, P.n_traces - t0);
        for (uint32_t s = 0; s < gcount; s++) {
            Slot256 S = l256_slot(scr + (size_t)s * L256Slot::BYTES);
            S.s_rank = reinterpret_cast<uint16_t*>(ws);  // the heaps are not in use yet
            stage256<kL256LB, kL256FS>(P, L.need_cls != 0, S, t0 + s, lane);
        }
        // 32-bit lane keys when every trace of the group allows them (warp-uniform)
        const uint32_t gi = min(g, gcount - 1);
        const Slot256 S = l256_slot(scr + (size_t)gi * L256Slot::BYTES);
        const bool narrow = __all_sync(FULL, g >= gcount || S.meta[6] == 1);
        bool fail = false;
        const uint32_t runmask = __ballot_sync(FULL, g < gcount && !S.meta[1]);
        if (g < gcount) {
            if (S.meta[1])
                fail = true;
            else if (narrow)
                fail = !l256_run<true>(P, S, ws, pslot, policy, t0 + g, lane, runmask);
            else
                fail = !l256_run<false>(P, S, ws, pslot, policy, t0 + g, lane, runmask);
        }
        __syncwarp();
        // exact fallback: the whole warp re-simulates each failed lane in its
        // shared-memory region (the group's heaps are done with)
        for (uint32_t fm = __ballot_sync(FULL, fail); fm; fm &= fm - 1) {
            const uint32_t fl = __ffs(fm) - 1;
            const uint32_t fg = fl / P.npol, fp = fl - fg * P.npol;
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
            uint4* apps_s = reinterpret_cast<uint4*>(ws + P.off_app);
            for (uint32_t i = lane; i < na; i += 32) apps_s[i] = __ldg(reinterpret_cast<const uint4*>(P.apps + a0) + i);
            __syncwarp();
            TraceSim<TickTM, 8, false, false> sim(P, lane, ws, apps_s);
            sim.run(na, (P.policy_list >> (4 * fp)) & 0xFu, P.cap[0], nullptr);
            sim.finish((uint64_t)fp * P.n_traces + t, (uint64_t)fp * P.n_apps_total + a0, nullptr, nullptr);
            __syncwarp();
        }
        __syncwarp();
        grp = next;
    }
    work_done(P.work, lane);
}

static inline uint32_t align16l(uint32_t x) { return (x + 15u) & ~15u; }

// Eligibility: as the octet kernel (T0 ticks, no event log, one device,
// n_pad 256).
bool lane256_eligible(const SimParams& p, bool program_mode, bool f64) {
    if (program_mode || f64 || p.events != nullptr || p.ndev != 1 || p.npol > 4) return false;
    if (p.n_traces > 0xFFFFFFFFull) return false;
    return p.n_pad == kL256N;
}

cudaError_t launch_sim_lane256(const SimParams& p, cudaStream_t stream, int* grid_out) {
    L256Params L;
    memset(&L, 0, sizeof(L));
    L.sp = p;
    sim_layout(L.sp, false, false, true);  // the fallback TraceSim, one app buffer
    L.G = min(32u / p.npol, 16u);
    L.need_cls = 0;
    for (uint32_t i = 0; i < p.npol; i++)
        if (((p.policy_list >> (4 * i)) & 0xFu) >= SG_POLICY_PFIFO) L.need_cls = 1;
    const uint32_t heap_b = kL256Heap * 32u * 8u;  // 64-bit keys (32-bit keys use half)
    L.warp_bytes = max(align16l(heap_b), align16l(L.sp.warp_bytes));
    const size_t smem = (size_t)L.warp_bytes * kL256WarpsPerBlock;
    int sms = 0, per_sm = 0;
    cudaError_t err = kernel_config(reinterpret_cast<const void*>(trace_sim_lane256_kernel<kL256MinBlocks>),
                                    kL256WarpsPerBlock * 32, smem, &per_sm, &sms);
    if (err != cudaSuccess) return err;
    const uint64_t groups = (p.n_traces + L.G - 1) / L.G;
    const uint64_t need = (groups + kL256WarpsPerBlock - 1) / kL256WarpsPerBlock;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (need < grid) grid = need;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    // global staging scratch: one slot per trace of every resident warp
    const size_t scr_b = (size_t)grid * kL256WarpsPerBlock * L.G * L256Slot::BYTES;
    keep_pool_memory();
    err = cudaMallocAsync(reinterpret_cast<void**>(&L.scratch), scr_b, stream);
    if (err != cudaSuccess) return err;
    WorkLease lease;
    err = work_counters(stream, L.sp, 0, lease);
    if (err == cudaSuccess) {
        trace_sim_lane256_kernel<kL256MinBlocks><<<(unsigned)grid, kL256WarpsPerBlock * 32, smem, stream>>>(L);
        err = cudaGetLastError();
    }
    err = work_release(stream, lease, err);
    const cudaError_t e2 = cudaFreeAsync(L.scratch, stream);
    return err != cudaSuccess ? err : e2;
}

}  // namespace sg
