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
//   * warp per trace, all requested policies of a trace back to back on one
//     staged copy; persistent grid (SMs x resident blocks), grid-stride
//   * the trace's 16 B/app records are staged global->shared by the TMA bulk
//     engine (cp.async.bulk + mbarrier), double-buffered so trace i+1 streams
//     in while trace i is simulated
//   * the heap is a per-app packed (t, counter, app) key in shared memory; lane
//     l owns apps l, l+32, ...; each pop is one lane-local min over its slots
//     plus a two-step REDUX min (time, then counter) — the exact tuple order of
//     heapq; grants write their keys lane-parallel
//   * the wait queue lives in shared memory in enqueue order.  T0 apps enqueue
//     at most once, so the queue is position-stable with a presence bitmask per
//     32 entries (no compaction); FIFO and MMU selection are __ballot_sync/__ffs
//     loops, the priority class a REDUX max — no atomics on event times
//   * all control flow is warp-uniform: every lane holds the same scalar state
//     (ledger, counters, statistics) in registers
//   * traces with several simulated devices run as per-device sub-traces: the
//     devices share only the global push counter, whose interleaving cannot
//     reorder events of one device (pinned by tests/golden/ref_multidev.npz)
#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>
#include <thread>
#include <vector>

#include "sgpu_tracesim.cuh"

namespace sg {

// ------------------------------------------------------------------ kernel

// SG_SIM_MIN_BLOCKS (build-time A/B knob): minimum resident blocks per SM
// requested from ptxas, i.e. a register cap of 64K / (128 * min_blocks).
#ifdef SG_SIM_MIN_BLOCKS
#define SG_SIM_BOUNDS __launch_bounds__(kSimWarpsPerBlock * 32, SG_SIM_MIN_BLOCKS)
#else
#define SG_SIM_BOUNDS __launch_bounds__(kSimWarpsPerBlock * 32)
#endif

template <class TM, int K, bool PROG>
__global__ void SG_SIM_BOUNDS trace_sim_kernel(const SimParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint8_t* ws = smem + (size_t)warp * P.warp_bytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(ws + P.off_bar);
    const uint32_t buf_bytes = P.n_pad * 16u;

    // traces are handed out by one atomic counter (sgpu_internal.h
    // work_reserve); each warp makes exactly one fetch past the end
    auto fetch = [&]() -> uint64_t { return work_fetch(P.work, lane); };

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
    auto stage = [&](uint64_t t, uint32_t b) {
        uint64_t a0;
        uint32_t na;
        trace_range(t, a0, na);
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[b], na * 16u);
            if (na) bulk_g2s(ws + P.off_app + b * buf_bytes, P.apps + a0, na * 16u, &bar[b]);
        }
    };

    uint64_t t = fetch();
    if constexpr (!PROG) {
        if (lane == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            fence_mbar_init();
        }
        __syncwarp();
        if (t < P.n_traces) stage(t, 0);
    }

    uint32_t iter = 0;
    while (t < P.n_traces) {
        const uint64_t next = fetch();
        uint64_t a0;
        uint32_t na;
        trace_range(t, a0, na);
        const uint32_t b = PROG ? 0u : (iter & 1u);
        bool steps_cached = false;
        if constexpr (!PROG) {
            mbar_wait(&bar[b], (iter >> 1) & 1u);
            __syncwarp();
            if (next < P.n_traces) stage(next, b ^ 1u);
        } else {
            uint4* dst = reinterpret_cast<uint4*>(ws + P.off_app);
            const uint32_t s0 = P.step_offsets[0];
            // the trace's steps go to shared memory when they fit: the step
            // fetch is on every event's critical path
            const uint32_t t0s = P.step_offsets[a0] - s0, t1s = P.step_offsets[a0 + na] - s0;
            steps_cached = t1s - t0s <= P.steps_cap;
            const uint32_t rel = steps_cached ? t0s : 0u;
            for (uint32_t i = lane; i < na; i += 32) {
                const uint32_t sb = P.step_offsets[a0 + i] - s0;
                const uint32_t se = P.step_offsets[a0 + i + 1] - s0;
                dst[i] = make_uint4(sb - rel, se - sb, 0u, P.apps[a0 + i].attr);
            }
            if (steps_cached) {
                uint4* s_steps = reinterpret_cast<uint4*>(ws + P.off_steps);
                for (uint32_t j = lane; j < t1s - t0s; j += 32)
                    s_steps[j] = __ldg(reinterpret_cast<const uint4*>(P.steps) + t0s + j);
            }
            __syncwarp();
        }
        const uint4* apps_smem = reinterpret_cast<const uint4*>(ws + P.off_app + b * buf_bytes);
        for (uint32_t d = 0; d < P.ndev; d++) {
            // (no dynamic indexing into the kernel parameters: it would force a
            // local-memory copy of SimParams)
            uint32_t cap_d = P.cap[0];
#pragma unroll
            for (uint32_t j = 1; j < SG_MAX_DEV; j++)
                if (d == j) cap_d = P.cap[j];
            // device d's sub-trace (all apps when ndev == 1), in index order
            const uint4* sub = apps_smem;
            const uint16_t* idx = nullptr;
            uint32_t nd = na;
            bool bad_dev = false;
            if (P.ndev > 1) {
                uint4* s_sub = reinterpret_cast<uint4*>(ws + P.off_sub);
                uint16_t* s_idx = reinterpret_cast<uint16_t*>(ws + P.off_idx);
                nd = build_subtrace(apps_smem, na, d, P.ndev, s_sub, s_idx, lane, bad_dev);
                sub = s_sub;
                idx = s_idx;
            }
            for (uint32_t p = 0; p < P.npol; p++) {
                TraceSim<TM, K, PROG> sim(P, lane, ws, sub);
                if (PROG && steps_cached) sim.s_steps = reinterpret_cast<const uint4*>(ws + P.off_steps);
                const uint64_t slot = (uint64_t)p * P.n_traces + t;
                sg_event* evs = P.events ? P.events + slot * P.ev_cap : nullptr;
                sim.run(nd, (P.policy_list >> (4 * p)) & 0xFu, cap_d, evs);
                if (bad_dev) sim.status |= SG_ST_BAD_DEVICE;
                sim.finish(slot * P.ndev + d, (uint64_t)p * P.n_apps_total + a0, idx,
                           P.event_counts ? P.event_counts + slot : nullptr);
            }
        }
        __syncwarp();
        t = next;
        iter++;
    }
    work_done(P.work, lane);
}

// ------------------------------------------------------------------ launch

// Work counters for dynamic scheduling, one set per (device, stream): the
// kernels reset them at the end of every launch (sgpu_common.cuh
// work_done), and launches on one stream are ordered, so a stream's set is
// always zero when its next launch starts.  A pool per device; new streams
// take slots round robin, and the per-thread default stream is keyed by
// thread.  A recycled slot may still be in use by work its previous stream
// has queued: the new owner's stream first waits on the slot's last-use
// event (recorded by every lease's release), so the two never overlap.
namespace {
constexpr int kWorkSlots = 512;
constexpr int kWorkWords = 4;  // u64 counters per slot
struct WorkPool {
    unsigned long long* ctr = nullptr;
    std::map<std::pair<cudaStream_t, std::thread::id>, int> slot;
    int next = 0;
    std::vector<std::pair<uint32_t*, uint64_t>> retry = std::vector<std::pair<uint32_t*, uint64_t>>(kWorkSlots);
    std::vector<cudaEvent_t> last_use = std::vector<cudaEvent_t>(kWorkSlots, nullptr);
};
std::mutex g_work_mu;
std::map<int, WorkPool> g_work;
}  // namespace

cudaError_t work_counters(cudaStream_t stream, SimParams& p, uint64_t retry_cap, WorkLease& lease) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(stream, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) {
        // inside a capture: counters and list are graph allocations (zeroed
        // by a memset node at every replay), so a replay never shares them
        // with the capturing stream's later work or with another replay
        void* b = nullptr;
        e = cudaMallocAsync(&b, kWorkWords * sizeof(unsigned long long) + retry_cap * 4u, stream);
        if (e != cudaSuccess) return e;
        lease.owned = b;
        e = cudaMemsetAsync(b, 0, kWorkWords * sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return e;
        p.work = static_cast<unsigned long long*>(b);
        p.retry = retry_cap ? reinterpret_cast<uint32_t*>(p.work + kWorkWords) : nullptr;
        return cudaSuccess;
    }
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    lease.lk = std::unique_lock<std::mutex>(g_work_mu);
    WorkPool& w = g_work[dev];
    if (!w.ctr) {
        e = cudaMalloc(&w.ctr, kWorkWords * kWorkSlots * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemset(w.ctr, 0, kWorkWords * kWorkSlots * sizeof(unsigned long long));
        if (e != cudaSuccess) { w.ctr = nullptr; return e; }
    }
    const auto key = std::make_pair(stream, stream == cudaStreamPerThread ? std::this_thread::get_id()
                                                                           : std::thread::id());
    auto it = w.slot.find(key);
    int s;
    if (it == w.slot.end()) {
        s = w.next;
        w.next = (w.next + 1) % kWorkSlots;
        for (auto i = w.slot.begin(); i != w.slot.end();) i = i->second == s ? w.slot.erase(i) : std::next(i);
        w.slot[key] = s;
        // the slot's previous owner may still have launches queued
        if (w.last_use[s]) {
            e = cudaStreamWaitEvent(stream, w.last_use[s], 0);
            if (e != cudaSuccess) return e;
        }
    } else {
        s = it->second;
    }
    if (!w.last_use[s]) {
        e = cudaEventCreateWithFlags(&w.last_use[s], cudaEventDisableTiming);
        if (e != cudaSuccess) { w.last_use[s] = nullptr; return e; }
    }
    lease.last_use = w.last_use[s];
    p.work = w.ctr + kWorkWords * s;
    p.retry = nullptr;
    if (retry_cap == 0) return cudaSuccess;
    auto& rb = w.retry[s];
    if (rb.second < retry_cap) {
        // grow: the old list is freed in stream order, after every queued
        // launch of this slot (this stream's, and the previous owner's,
        // which this stream already waits on)
        if (rb.first) {
            e = cudaFreeAsync(rb.first, stream);
            rb = {nullptr, 0};
            if (e != cudaSuccess) return e;
        }
        const uint64_t c = std::max<uint64_t>(retry_cap, 1u << 16);
        e = cudaMallocAsync(reinterpret_cast<void**>(&rb.first), c * 4u, stream);
        if (e != cudaSuccess) { rb = {nullptr, 0}; return e; }
        rb.second = c;
    }
    p.retry = rb.first;
    return cudaSuccess;
}

cudaError_t work_release(cudaStream_t stream, WorkLease& lease, cudaError_t err) {
    if (lease.owned) {
        const cudaError_t e = cudaFreeAsync(lease.owned, stream);
        lease.owned = nullptr;
        if (err == cudaSuccess) err = e;
    }
    if (lease.last_use) {
        const cudaError_t e = cudaEventRecord(lease.last_use, stream);
        lease.last_use = nullptr;
        if (err == cudaSuccess) err = e;
    }
    if (lease.lk.owns_lock()) lease.lk.unlock();
    return err;
}

namespace {
struct KernelCfg {
    int per_sm, sms;
};
std::mutex g_cfg_mu;
std::map<std::tuple<const void*, int, int, size_t>, KernelCfg> g_cfg;
// the dynamic shared-memory limit set on each (kernel, device): only ever
// raised, so a configuration cached at a larger size stays launchable
std::map<std::pair<const void*, int>, size_t> g_smem_max;
}  // namespace

void keep_pool_memory() {
    static std::mutex mu;
    static bool kept[64] = {false};
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    if (kept[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    kept[dev] = true;
}

cudaError_t kernel_config(const void* kern, int threads, size_t smem, int* per_sm, int* sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const auto key = std::make_tuple(kern, dev, threads, smem);
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    auto it = g_cfg.find(key);
    if (it == g_cfg.end()) {
        if (smem > 227u * 1024u) return cudaErrorInvalidConfiguration;
        size_t& lim = g_smem_max[std::make_pair(kern, dev)];
        if (smem > lim) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            lim = smem;
        }
        // all of the unified L1/shared array as shared memory: the occupancy
        // the grid is sized for must not depend on the driver's carveout choice
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        KernelCfg c{0, 0};
        e = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.per_sm, kern, threads, smem);
        if (e != cudaSuccess) return e;
        it = g_cfg.emplace(key, c).first;
    }
    *per_sm = it->second.per_sm;
    *sms = it->second.sms;
    return *per_sm < 1 ? cudaErrorInvalidConfiguration : cudaSuccess;
}

static inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

void sim_layout(SimParams& p, bool program_mode, bool f64, bool single_app_buf) {
    const uint32_t N = p.n_pad;
    const uint32_t tsz = f64 ? 8u : 4u;
    const bool multi = p.ndev > 1;
    uint32_t o = 0;
    p.off_app = o;
    o = align16(o + N * 16u * (program_mode || single_app_buf ? 1u : 2u));
    p.off_sub = o;
    o = align16(o + (multi ? N * 16u : 0u));
    p.off_idx = o;
    o = align16(o + (multi ? N * 2u : 0u));
    p.off_key = o;
    o = align16(o + N * 8u);
    p.off_kc = o;
    o = align16(o + (f64 ? N * 4u : 0u));
    p.off_q = o;
    o = align16(o + N * 8u);
    p.off_grant = o;
    o = align16(o + N * tsz);
    p.off_end = o;
    o = align16(o + N * tsz);
    p.off_st = o;
    o = align16(o + N * 2u);
    p.off_held = o;
    o = align16(o + (program_mode ? N * 4u : 0u));
    p.off_pc = o;  // T0: waiting entries per priority (256 x u16) + their queue chunks (256 x u32)
    o = align16(o + (program_mode ? 0u : 512u + 1024u));
    p.off_steps = o;  // program mode: the trace's steps, when they fit (8 per app slot)
    p.steps_cap = program_mode ? 8u * N : 0u;
    o = align16(o + p.steps_cap * 16u);
    p.off_bar = o;
    o = align16(o + 16u);
    p.warp_bytes = o;
}

template <class TM, int K, bool PROG>
static cudaError_t launch_t(const SimParams& p, cudaStream_t stream, int* grid_out) {
    auto kern = trace_sim_kernel<TM, K, PROG>;
    // warps per block: as many as fit (<= kSimWarpsPerBlock) in 227 KB
    uint32_t wpb = kSimWarpsPerBlock;
    while (wpb > 1 && (size_t)p.warp_bytes * wpb > 227u * 1024u) wpb--;
    const size_t smem = (size_t)p.warp_bytes * wpb;
    int sms = 0, per_sm = 0;
    cudaError_t err = kernel_config(reinterpret_cast<const void*>(kern), wpb * 32, smem, &per_sm, &sms);
    if (err != cudaSuccess) return err;
    const uint64_t need = (p.n_traces + wpb - 1) / wpb;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (need < grid) grid = need;
    if (grid == 0) grid = 1;
    if (grid_out) *grid_out = (int)grid;
    SimParams q = p;
    WorkLease lease;
    err = work_counters(stream, q, 0, lease);
    if (err == cudaSuccess) {
        kern<<<(unsigned)grid, wpb * 32, smem, stream>>>(q);
        err = cudaGetLastError();
    }
    return work_release(stream, lease, err);
}

template <class TM, bool PROG>
static cudaError_t launch_k(const SimParams& p, cudaStream_t s, int* g) {
    switch (p.n_pad / 32) {
        case 1: return launch_t<TM, 1, PROG>(p, s, g);
        case 2: return launch_t<TM, 2, PROG>(p, s, g);
        case 4: return launch_t<TM, 4, PROG>(p, s, g);
        case 8: return launch_t<TM, 8, PROG>(p, s, g);
        case 16: return launch_t<TM, 16, PROG>(p, s, g);
        case 32: return launch_t<TM, 32, PROG>(p, s, g);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_sim(const SimParams& p, bool program_mode, bool f64, cudaStream_t stream,
                       int* grid_out) {
    if (f64) {
        if (!program_mode) return cudaErrorInvalidValue;
        return launch_k<F64TM, true>(p, stream, grid_out);
    }
    if (program_mode) return launch_k<TickTM, true>(p, stream, grid_out);
    return launch_k<TickTM, false>(p, stream, grid_out);
}

}  // namespace sg
