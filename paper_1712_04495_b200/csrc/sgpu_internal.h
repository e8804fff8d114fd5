// sgpu_internal.h — launch parameters shared by the ABI layer and kernels.
#pragma once

#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#include "../../include/sgpu.h"

namespace sg {

constexpr int kSimWarpsPerBlock = 4;

struct SimParams {
    uint64_t n_traces;
    const uint64_t* trace_offsets;  // optional CSR
    uint32_t apps_per_trace;
    uint32_t max_apps;              // upper bound of apps per trace
    uint32_t n_pad;                 // per-warp app capacity (multiple of 32)
    const sg_app* apps;
    const sg_step* steps;           // program mode
    const uint32_t* step_offsets;
    uint32_t policy_list;           // policy codes, 4 bits each, in output order
    uint32_t npol;
    uint32_t ndev;
    uint32_t cap[SG_MAX_DEV];
    int32_t tick_log2;
    uint32_t ev_cap;
    uint64_t n_apps_total;          // per-policy stride of grant/end
    void* grant;
    void* end;
    void* stats;
    double* mem_pct;
    double* dev_pct;
    double* speedup;                // optional: per-record speed-up vs sequential (ticks mode)
    sg_event* events;
    uint32_t* event_counts;
    // per-warp shared-memory layout (bytes)
    uint32_t off_app, off_sub, off_idx, off_key, off_kc, off_q, off_grant, off_end, off_st, off_held,
        off_pc, off_steps, off_bar, warp_bytes;
    uint32_t steps_cap;             // program mode: steps of one trace kept in shared memory
    // dynamic scheduling: work[0] hands out work items, work[1] counts the
    // warps that are done; the last warp of a launch resets both.  work[2]
    // counts the entries of `retry` (lane kernel: traces deferred to the
    // 64-bit-key pass), reset by the last warp of that pass.
    unsigned long long* work;
    uint32_t* retry;
};

// A lease on one stream's work counters (and deferred-trace list), from
// work_counters() until work_release(), which the caller invokes after its
// last launch using them.  Outside a capture the pool lock is held for the
// whole lease, so no other host thread can grow the list or reassign the
// slot between the lookup and the launches; the release records the slot's
// last-use event, which a later owner of a recycled slot waits on.  Inside a
// capture counters and list are one graph allocation, freed on the stream
// by the release.
struct WorkLease {
    std::unique_lock<std::mutex> lk;
    cudaEvent_t last_use = nullptr;
    void* owned = nullptr;
};

// The work counters of `stream` on the current device (sets p.work) and,
// when retry_cap > 0, a deferred-trace list of that many entries that stays
// valid for work on `stream` (sets p.retry).
cudaError_t work_counters(cudaStream_t stream, SimParams& p, uint64_t retry_cap, WorkLease& lease);
// End the lease after the launches; returns `err` or the first release error.
cudaError_t work_release(cudaStream_t stream, WorkLease& lease, cudaError_t err);

// Kernel attributes (dynamic shared memory, max-shared carveout) set once per
// (kernel, device, smem) and the resulting resident blocks per SM, cached:
// launches pay no attribute call or occupancy query.
cudaError_t kernel_config(const void* kern, int threads, size_t smem, int* per_sm, int* sms);
// Once per device: the current device's default memory pool keeps freed
// memory (release threshold = max), so the per-launch cudaMallocAsync
// scratch of the lane kernels is recycled instead of unmapped at each
// synchronisation and mapped again by the next launch.
void keep_pool_memory();

// Shared-memory layout for one warp simulating traces of up to n_pad apps
// (single_app_buf: one staged trace instead of the T0 double buffer, for the
// in-kernel fallbacks of the lane / octet kernels).
void sim_layout(SimParams& p, bool program_mode, bool f64, bool single_app_buf = false);

// Launch K1 (trace simulation).  Returns a cudaError_t.
cudaError_t launch_sim(const SimParams& p, bool program_mode, bool f64, cudaStream_t stream,
                       int* grid_out);

// K1 v5: lane-per-(trace, device, policy) kernel for T0 tick-mode batches
// (sgpu_lane.cu), with an in-kernel exact fallback to TraceSim.
bool lane_eligible(const SimParams& p, bool program_mode, bool f64, bool forced);
cudaError_t launch_sim_lane(const SimParams& p, cudaStream_t stream, int* grid_out);
// K1 v8: octet-per-(trace, policy) kernel for T0 tick-mode batches of
// 129..256-app single-device traces (sgpu_octet.cu), with an in-kernel exact
// fallback to TraceSim.
bool octet_eligible(const SimParams& p, bool program_mode, bool f64);
cudaError_t launch_sim_octet(const SimParams& p, cudaStream_t stream, int* grid_out);
// K1 v9: lane-per-(trace, policy) kernel for the same batches as v8, its
// staged trace tables in global memory (sgpu_lane256.cu), with an in-kernel
// exact fallback to TraceSim.
bool lane256_eligible(const SimParams& p, bool program_mode, bool f64);
cudaError_t launch_sim_lane256(const SimParams& p, cudaStream_t stream, int* grid_out);
// K1 v6: lane-per-(trace, policy) kernel for step-program tick-mode batches
// (sgpu_proglane.cu), with an in-kernel exact fallback to TraceSim.
bool prog_lane_eligible(const SimParams& p, bool program_mode, bool f64, bool forced);
cudaError_t launch_sim_prog_lane(const SimParams& p, cudaStream_t stream, int* grid_out);
// Resident warps per SM of the lane kernel for a C2-shaped batch (64 apps, 4
// policies, 1 device) on the current device (sg_device_info).
cudaError_t lane_warps_per_sm(int* warps);

cudaError_t launch_reduce(const sg_trace_stats* stats, uint64_t count, sg_aggr* out,
                          cudaStream_t stream);
cudaError_t launch_generate(const sg_gen_params& p, uint64_t trace_begin, uint64_t n_traces,
                            sg_app* out, cudaStream_t stream);
cudaError_t launch_select(uint64_t n_queues, const uint64_t* qoff, const int64_t* nbytes,
                          const int32_t* prio, const int64_t* free_bytes, const uint32_t* kind,
                          uint8_t* granted, cudaStream_t stream);
// K5: host-pipeline transfer format of a simulated chunk: b16[i] = busy of
// app i as u16 (0xFFFF = no memory request), e16[p * na + i] = end tick
// end[p * stride + i] as u16 (0xFFFF = SG_NEVER); *overflow = 1 if that is
// not exact.
cudaError_t launch_pack16(const sg_app* apps, const uint32_t* end, uint64_t na, uint64_t stride, uint32_t npol,
                          uint16_t* b16, uint16_t* e16, uint32_t* overflow, cudaStream_t stream);

}  // namespace sg
