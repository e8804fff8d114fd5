/*
 * sgpu.h — C ABI of libsgpu.so, the B200 (sm_100a) trace-simulation engine
 * for schedGPU's memory-safe co-scheduling hot path (arXiv 1712.04495).
 *
 * The reference ("memshare", /root/reference/pkg) has no FFI: its hot path
 * is a set of pure Python callables.  Each entry point below replaces one of
 * them; the Python package `paper_1712_04495_b200` binds this header through
 * ctypes and re-exposes the reference's own names.
 *
 *   sg_simulate_batch        replaces memshare/harness.py:475-572  simulate(spec)
 *                            (+ memshare/harness.py:373-461 _metrics_from_events,
 *                               fused as per-trace integer statistics)
 *                            batched: one warp per (trace, policy)
 *   sg_simulate_batch_host   same, host buffers, chunked H2D/compute/D2H pipeline
 *   sg_simulate_small_host   same, host buffers, a few traces at the lowest
 *                            latency (one H2D, one launch, one D2H): the
 *                            drop-in simulate(spec) of one workload
 *   sg_select_grants_batch   replaces memshare/policy.py:52-74 select_grants
 *   sg_reduce_stats          new: aggregate statistics over traces (no reference
 *                            counterpart; feeds the single cross-GPU collective)
 *   sg_generate_traces       new: counter-based synthetic trace generator,
 *                            bit-identical to paper_1712_04495_b200/tracegen.py
 *
 * Conventions
 *   - Return 0 on success, a negative SG_E* code otherwise; sg_last_error()
 *     returns a thread-local diagnostic string.  No exception crosses the ABI.
 *   - The caller owns every buffer; the library never frees caller memory.
 *   - Device entry points are asynchronous on the given cudaStream_t (passed
 *     as void*; NULL = legacy default stream).
 *   - Times are integer ticks of 2^-tick_log2 seconds (default 2^-10 s: the
 *     reference run at time_scale = 1000/1024 makes every event time exactly
 *     ticks/1024 s, SURVEY.md §8 "Ticks"), or IEEE-754 float64 seconds in
 *     SG_TIME_F64 mode, which reproduces the reference's own float arithmetic
 *     for non-dyadic time scales.
 *   - Memory sizes are MiB (the reference allocates whole MiB:
 *     memshare/harness.py:485,489 `alloc_mib * MIB`).
 */
#ifndef SGPU_H
#define SGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 2

/* Largest trace (apps per trace) one warp simulates. */
#define SG_MAX_APPS 1024
/* Largest number of simulated devices per trace (config 5). */
#define SG_MAX_DEV 8

/* Policy codes: memshare/policy.py:47-48 (docs/format.md:35). */
enum sg_policy {
    SG_POLICY_FIFO = 0,  /* head blocks                              */
    SG_POLICY_MMU = 1,   /* first-fit greedy, skip misfits           */
    SG_POLICY_PFIFO = 2, /* max-priority class, then FIFO            */
    SG_POLICY_PMMU = 3   /* max-priority class, then MMU             */
};

/* Step opcodes of the general step-program mode (memshare/harness.py:478-490). */
enum sg_op { SG_OP_CPU = 0, SG_OP_ALLOC = 1, SG_OP_BUSY = 2, SG_OP_FREE = 3 };

enum sg_time_mode { SG_TIME_TICKS = 0, SG_TIME_F64 = 1 };

/* Event kinds of the optional event log (memshare/harness.py:501-503, 514-543). */
enum sg_event_kind {
    SG_EV_START = 0, SG_EV_REQUEST = 1, SG_EV_GRANT = 2, SG_EV_ALLOC = 3,
    SG_EV_BUSY_START = 4, SG_EV_BUSY_END = 5, SG_EV_FREE = 6, SG_EV_END = 7
};

/* Per-trace status bits (sg_trace_stats.status). */
#define SG_ST_TICK_OVERFLOW   0x1u  /* an event time exceeded 2^32-2 ticks   */
#define SG_ST_COUNTER_OVERFLOW 0x2u /* more than 2^22 heap pushes            */
#define SG_ST_BAD_DEVICE      0x4u  /* ndev > 1 and an app of the trace has a
                                       device index >= ndev (it is simulated
                                       on device 0); set on every record of
                                       the trace                           */
#define SG_ST_EVENT_OVERFLOW  0x8u  /* event log capacity exceeded           */
#define SG_ST_ZERO_SPAN_LEVEL 0x10u /* T == 0 with memory still held: the
                                       reference integrates level * 1e-9 s;
                                       mem_integral then holds the level MiB */

/*
 * T0 trace encoding, 16 B per app (SURVEY.md §8 "T0"): the reference profile
 *   AppProfile(name, [Phase(cpu_ms=arrival),
 *                     Phase(alloc_mib=mem_mib, busy_ms=busy, free_mib=mem_mib)],
 *              priority=prio)
 * which flattens (zero fields skipped) to cpu -> alloc -> busy -> free.
 * attr = prio (8 bits) | device (8 bits) << 8.  In step-program mode only
 * attr is read.
 */
typedef struct sg_app {
    uint32_t arrival;
    uint32_t mem_mib;
    uint32_t busy;
    uint32_t attr;
} sg_app;

/* One step of the general step-program mode; dur = ticks, or the bits of a
 * float64 seconds value in SG_TIME_F64 mode. */
typedef struct sg_step {
    uint32_t op;
    uint32_t mib;
    uint64_t dur;
} sg_step;

typedef struct sg_batch {
    uint64_t n_traces;
    /* Optional CSR app offsets (n_traces + 1 entries, device memory for
     * sg_simulate_batch).  Trace t owns apps [off[t]-off[0], off[t+1]-off[0]).
     * NULL => every trace has apps_per_trace apps. */
    const uint64_t* trace_offsets;
    uint32_t apps_per_trace;
    uint32_t max_apps;          /* upper bound of apps/trace (<= SG_MAX_APPS) */
    const sg_app* apps;
    /* Step-program mode when non-NULL: app a runs steps
     * [step_offsets[a]-step_offsets[0], step_offsets[a+1]-step_offsets[0]). */
    const sg_step* steps;
    const uint32_t* step_offsets;
    uint32_t policy_mask;       /* bit p => simulate policy p; outputs are laid
                                   out policy-major in increasing p          */
    uint32_t ndev;              /* simulated devices per trace, 1..8         */
    uint32_t cap_mib[SG_MAX_DEV];
    uint32_t time_mode;         /* sg_time_mode (F64 requires steps)         */
    int32_t tick_log2;          /* seconds per tick = 2^-tick_log2           */
    /* With trace_offsets: the per-policy stride of grant/end, at least
     * trace_offsets[n_traces] - trace_offsets[0] (the batch's app count).
     * Passed by the caller so the call never reads device memory on the
     * host: it stays asynchronous and graph-capturable.  Ignored without
     * trace_offsets (the stride is then n_traces * apps_per_trace). */
    uint64_t apps_total;
} sg_batch;

/* Per-(policy, trace, device) statistics, ticks mode, 32 B. */
typedef struct sg_trace_stats {
    uint32_t makespan;      /* T: max event tick                              */
    uint32_t busy;          /* B: ticks with >= 1 busy interval               */
    uint64_t mem_integral;  /* I: sum(level_mib * dticks) over [0, T]         */
    uint32_t grants;        /* admission decisions (grant events)             */
    uint32_t pops;          /* event-queue pops (heappop count)               */
    uint16_t max_holders;   /* max concurrent holders                         */
    uint16_t unfinished;    /* apps that never emitted `end`                  */
    uint32_t status;        /* SG_ST_* bits                                   */
} sg_trace_stats;

/* Per-(policy, trace, device) statistics, F64 mode, 40 B. */
typedef struct sg_trace_stats_f64 {
    double makespan_s;      /* max event time, seconds                        */
    double mem_integral;    /* byte-seconds, reference accumulation order     */
    double busy_s;          /* seconds with >= 1 busy interval                */
    uint32_t grants;
    uint32_t pops;
    uint16_t max_holders;
    uint16_t unfinished;
    uint32_t status;
} sg_trace_stats_f64;

/* Event-log record, 16 B; t = ticks or float64 seconds bits. */
typedef struct sg_event {
    uint64_t t;
    uint16_t app;
    uint8_t kind;
    uint8_t dev;
    uint32_t mib;
} sg_event;

typedef struct sg_out {
    /* Per (policy, app): first grant time and end time; SG_NEVER if none.
     * uint32_t ticks, or double seconds in F64 mode (NaN = never). May be NULL. */
    void* grant;
    void* end;
    /* Per (policy, trace, device): sg_trace_stats or sg_trace_stats_f64. */
    void* stats;
    /* Optional per (policy, trace, device) utilisation percentages, computed
     * with the reference's float operation order (harness.py:427,437). */
    double* mem_pct;
    double* dev_pct;
    /* Optional event log: (policy, trace) slice of events_per_trace records,
     * in reference emission order; event_counts per (policy, trace). */
    sg_event* events;
    uint32_t* event_counts;
    uint32_t events_per_trace;
    uint32_t reserved;
    /* Optional per (policy, trace, device) speed-up vs sequential execution
     * (ticks mode; NaN in F64 mode and for an empty sub-trace):
     *   sum over apps of (cpu + busy) * time_scale / makespan_ms
     * in the reference's float order (AppProfile.total_ms(),
     * memshare/harness.py:61-62; pkg/tests/test_harness.py:119-126), i.e.
     * (S * 1000 * 2^-tick_log2) / (max(T * 2^-tick_log2, 1e-9) * 1000) with
     * S = sum of the sub-trace's cpu and busy ticks and T its makespan. */
    double* speedup;
} sg_out;

#define SG_NEVER 0xFFFFFFFFu

/* Aggregate statistics over many trace records (sg_reduce_stats).  Fields
 * [0, SG_AGGR_NSUM) are sums, [SG_AGGR_NSUM, 16) maxima: a cross-GPU
 * reduction is one SUM all-reduce plus one MAX all-reduce. */
#define SG_AGGR_NSUM 12
typedef struct sg_aggr {
    uint64_t records;
    uint64_t sum_makespan;
    uint64_t sum_busy;
    uint64_t sum_mem_integral;
    uint64_t sum_grants;
    uint64_t sum_pops;
    uint64_t sum_unfinished;
    uint64_t sum_max_holders;
    uint64_t stuck_records;     /* records with unfinished > 0 */
    uint64_t error_records;     /* records with status != 0    */
    uint64_t reserved_sum0;
    uint64_t reserved_sum1;
    uint64_t max_makespan;
    uint64_t max_holders;
    uint64_t status_or;
    uint64_t reserved_max0;
} sg_aggr;

/* Synthetic trace generator parameters. */
enum sg_arrival_kind { SG_ARR_UNIFORM = 0, SG_ARR_CUBIC = 1 };
enum sg_prio_kind { SG_PRIO_UNIFORM = 0, SG_PRIO_SKEWED = 1 };
typedef struct sg_gen_params {
    uint64_t seed;
    uint32_t apps_per_trace;
    uint32_t arrival_kind;  /* UNIFORM: U[arr_lo, arr_hi]; CUBIC: arr_lo +
                               (c * (arr_hi - arr_lo + 1)) >> 24 with
                               c = ((u*u >> 24) * u) >> 24, u 24-bit       */
    uint32_t arr_lo, arr_hi;
    uint32_t mem_lo, mem_hi;
    uint32_t busy_lo, busy_hi;
    uint32_t prio_kind;     /* UNIFORM: U{0..levels-1}; SKEWED: weights
                               2^(levels-1-k) for level k                  */
    uint32_t prio_levels;   /* 1..8 */
    uint32_t ndev;          /* device = app index mod ndev                  */
} sg_gen_params;

int sg_abi_version(void);
const char* sg_last_error(void);

/* Number of SMs, and resident warps per SM of the default K1 engine for a
 * C2-shaped batch (64-app T0 traces, four policies, one device). */
int sg_device_info(int cuda_device, int* sm_count, int* warps_per_sm);

/* Device-pointer batch simulation (async on stream). */
int sg_simulate_batch(const sg_batch* in, const sg_out* out, void* stream);

/* Host-pointer batch simulation: copies inputs to `cuda_device` in chunks of
 * chunk_traces traces (0 = automatic), simulates, copies outputs back,
 * overlapping the three with streams.  Synchronous.  Event logs unsupported.
 * With both tick arrays requested, a chunk whose ticks all fit 16 bits
 * crosses PCIe as u16 end and busy ticks and host threads write both u32
 * arrays (grant = end - busy); other chunks cross as u32 end ticks. */
int sg_simulate_batch_host(const sg_batch* in, const sg_out* out, int cuda_device,
                           uint64_t chunk_traces);

/* Bytes the calling thread's last sg_simulate_batch_host call copied host ->
 * device and device -> host (either pointer may be NULL). */
void sg_last_host_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* Host-buffer simulation of a few traces with the lowest latency (the
 * drop-in simulate(spec) path, memshare/harness.py:475-572): any mode the
 * device call supports (step programs, float64 time, event logs), fixed
 * apps_per_trace (no trace_offsets).  Inputs are packed into one pinned
 * staging buffer and copied in one H2D, simulated, and every requested
 * output comes back in one D2H; staging, device buffers and the stream are
 * kept per calling thread and device.  Synchronous.  Event slots past a
 * trace's count are zero. */
int sg_simulate_small_host(const sg_batch* in, const sg_out* out, int cuda_device);

/* Reduce `count` sg_trace_stats records into *out (device pointer, overwritten). */
int sg_reduce_stats(const sg_trace_stats* stats, uint64_t count, sg_aggr* out,
                    void* stream);

/* Generate apps for traces [trace_begin, trace_begin + n_traces) into
 * out (n_traces * apps_per_trace records, device memory). */
int sg_generate_traces(const sg_gen_params* p, uint64_t trace_begin, uint64_t n_traces,
                       sg_app* out, void* stream);

/* Batched select_grants: queue q holds entries [qoff[q]-qoff[0], qoff[q+1]-qoff[0])
 * in enqueue order; granted[e] = 1 iff the entry is granted (policy.py:52-74).
 * kind[q] and free_bytes[q] per queue.  Device pointers. */
int sg_select_grants_batch(uint64_t n_queues, const uint64_t* qoff, const int64_t* nbytes,
                           const int32_t* prio, const int64_t* free_bytes,
                           const uint32_t* kind, uint8_t* granted, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGPU_H */
