// sgpu_abi.cu — extern "C" entry points of libsgpu.so (include/sgpu.h):
// argument validation, kernel dispatch, and the host-buffer pipeline.
#include <algorithm>
#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <map>
#include <memory>
#include <vector>

#include "sgpu_common.cuh"
#include "sgpu_internal.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

constexpr int E_ARG = -1;
constexpr int E_CUDA = -2;
constexpr int E_RANGE = -3;

int cuda_fail(cudaError_t e, const char* what) {
    return fail(E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct Shape {
    uint32_t npol = 0;
    uint32_t policies[4] = {0, 0, 0, 0};
    bool program = false, f64 = false, multi = false;
    uint32_t n_pad = 0;
};

int validate(const sg_batch* in, Shape& s) {
    if (!in) return fail(E_ARG, "null batch");
    if (in->policy_mask == 0 || (in->policy_mask & ~0xFu))
        return fail(E_ARG, "policy_mask must be a non-empty subset of 0xF (got 0x%x)", in->policy_mask);
    for (uint32_t p = 0; p < 4; p++)
        if (in->policy_mask & (1u << p)) s.policies[s.npol++] = p;
    if (in->ndev < 1 || in->ndev > SG_MAX_DEV) return fail(E_ARG, "ndev must be 1..%d", SG_MAX_DEV);
    for (uint32_t d = 0; d < in->ndev; d++)
        if (in->cap_mib[d] == 0 || in->cap_mib[d] >= 0x7FFFFFFFu)
            return fail(E_RANGE, "cap_mib[%u] must be in [1, 2^31-1)", d);
    if (in->time_mode != SG_TIME_TICKS && in->time_mode != SG_TIME_F64)
        return fail(E_ARG, "unknown time_mode %u", in->time_mode);
    s.program = in->steps != nullptr;
    if (s.program && !in->step_offsets) return fail(E_ARG, "steps given without step_offsets");
    s.f64 = in->time_mode == SG_TIME_F64;
    if (s.f64 && !s.program) return fail(E_ARG, "SG_TIME_F64 requires step-program mode");
    if (in->tick_log2 < -64 || in->tick_log2 > 64) return fail(E_RANGE, "tick_log2 out of range");
    s.multi = in->ndev > 1;
    const uint32_t maxn = in->trace_offsets ? in->max_apps : in->apps_per_trace;
    if (maxn > SG_MAX_APPS) return fail(E_RANGE, "traces longer than %d apps are not supported", SG_MAX_APPS);
    if (in->n_traces && maxn && !in->apps) return fail(E_ARG, "null apps");
    if (reinterpret_cast<uintptr_t>(in->apps) & 15u) return fail(E_ARG, "apps must be 16-byte aligned");
    // apps per lane K in {1, 2, 4, 8, 16, 32}: the kernel instantiation buckets
    const uint32_t chunks = (maxn + 31u) / 32u;
    const uint32_t k = chunks <= 1 ? 1 : chunks <= 2 ? 2 : chunks <= 4 ? 4 : chunks <= 8 ? 8
                       : chunks <= 16 ? 16 : 32;
    s.n_pad = 32u * k;
    return 0;
}

}  // namespace

extern "C" {

int sg_abi_version(void) { return SG_ABI_VERSION; }

const char* sg_last_error(void) { return g_err; }

int sg_device_info(int cuda_device, int* sm_count, int* warps_per_sm) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (sm_count) *sm_count = sms;
    if (warps_per_sm) {
        int cur = 0;
        e = cudaGetDevice(&cur);
        if (e == cudaSuccess && cur != cuda_device) e = cudaSetDevice(cuda_device);
        if (e == cudaSuccess) e = sg::lane_warps_per_sm(warps_per_sm);
        if (cur != cuda_device) cudaSetDevice(cur);
        if (e != cudaSuccess) return cuda_fail(e, "lane kernel occupancy");
    }
    return 0;
}

static int simulate_device(const sg_batch* in, const sg_out* out, cudaStream_t stream,
                           uint64_t n_apps_total) {
    Shape s;
    int rc = validate(in, s);
    if (rc) return rc;
    if (!out || !out->stats) return fail(E_ARG, "sg_out.stats is required");
    if (out->events && out->events_per_trace == 0) return fail(E_ARG, "events_per_trace must be > 0");
    if (out->events && !s.program) return fail(E_ARG, "event logs require step-program mode");
    if (out->events && s.multi) return fail(E_ARG, "event logs require ndev == 1");
    if (in->n_traces == 0) return 0;
    sg::SimParams p;
    memset(&p, 0, sizeof(p));
    p.n_traces = in->n_traces;
    p.trace_offsets = in->trace_offsets;
    p.apps_per_trace = in->apps_per_trace;
    p.max_apps = in->trace_offsets ? in->max_apps : in->apps_per_trace;
    p.n_pad = s.n_pad;
    p.apps = in->apps;
    p.steps = in->steps;
    p.step_offsets = in->step_offsets;
    for (uint32_t i = 0; i < s.npol; i++) p.policy_list |= s.policies[i] << (4 * i);
    p.npol = s.npol;
    p.ndev = in->ndev;
    for (uint32_t d = 0; d < SG_MAX_DEV; d++) p.cap[d] = d < in->ndev ? in->cap_mib[d] : 1;
    p.tick_log2 = in->tick_log2;
    p.ev_cap = out->events_per_trace;
    p.n_apps_total = n_apps_total;
    p.grant = out->grant;
    p.end = out->end;
    p.stats = out->stats;
    p.mem_pct = out->mem_pct;
    p.dev_pct = out->dev_pct;
    p.speedup = out->speedup;
    p.events = out->events;
    p.event_counts = out->event_counts;
    sg::sim_layout(p, s.program, s.f64);
    if (p.warp_bytes > 227u * 1024u)
        return fail(E_RANGE, "shared memory per warp exceeds 227 KB (n_pad=%u)", s.n_pad);
    // K1 engine: the lane kernel (v5) where eligible, else the warp kernel
    // (v3).  SGPU_K1=warp|lane overrides (A/B runs and parity tests).
    const char* eng = getenv("SGPU_K1");
    const bool want_warp = eng && strcmp(eng, "warp") == 0;
    const bool want_lane = eng && strcmp(eng, "lane") == 0;
    const bool want_octet = eng && strcmp(eng, "octet") == 0;
    const bool want_l256 = eng && strcmp(eng, "lane256") == 0;
    const bool lane_ok = sg::lane_eligible(p, s.program, s.f64, want_lane);
    const bool prog_ok = sg::prog_lane_eligible(p, s.program, s.f64, want_lane);
    const bool oct_ok = want_octet && sg::octet_eligible(p, s.program, s.f64);
    if (want_lane && !lane_ok && !prog_ok) return fail(E_ARG, "SGPU_K1=lane: batch not eligible for a lane kernel");
    if (want_octet && !oct_ok) return fail(E_ARG, "SGPU_K1=octet: batch not eligible for the octet kernel");
    // 129..256-app single-device T0 traces: the lane256 kernel (v9) by
    // default, the octet kernel (v8) when asked for
    const bool l256_ok = !want_octet && !want_lane && !want_warp && sg::lane256_eligible(p, s.program, s.f64);
    if (want_l256 && !l256_ok) return fail(E_ARG, "SGPU_K1=lane256: batch not eligible for the lane256 kernel");
    cudaError_t e;
    if (prog_ok && !want_warp) {
        e = sg::launch_sim_prog_lane(p, stream, nullptr);
        if (e != cudaSuccess) return cuda_fail(e, "trace_prog_lane launch");
    } else if (l256_ok) {
        e = sg::launch_sim_lane256(p, stream, nullptr);
        if (e != cudaSuccess) return cuda_fail(e, "trace_sim_lane256 launch");
    } else if (oct_ok && !want_warp) {
        e = sg::launch_sim_octet(p, stream, nullptr);
        if (e != cudaSuccess) return cuda_fail(e, "trace_sim_octet launch");
    } else if (lane_ok && !want_warp) {
        e = sg::launch_sim_lane(p, stream, nullptr);
        if (e != cudaSuccess) return cuda_fail(e, "trace_sim_lane launch");
    } else {
        e = sg::launch_sim(p, s.program, s.f64, stream, nullptr);
        if (e != cudaSuccess) return cuda_fail(e, "trace_sim launch");
    }
    return 0;
}

int sg_simulate_batch(const sg_batch* in, const sg_out* out, void* stream) {
    if (!in) return fail(E_ARG, "null batch");
    // the per-policy stride of grant/end: given by the caller for CSR
    // batches (no device read on the host: the call stays asynchronous)
    const uint64_t n_apps_total = in->trace_offsets ? in->apps_total
                                                    : in->n_traces * (uint64_t)in->apps_per_trace;
    return simulate_device(in, out, static_cast<cudaStream_t>(stream), n_apps_total);
}

// Host-buffer pipeline: chunks of traces cycle through NBUF device buffer
// sets on NBUF streams; each chunk is H2D -> trace_sim -> K5 pack16 -> D2H
// on its stream, so the copies of one chunk overlap the simulation of the
// next.
//
// The per-app grant ticks are not copied back: for T0 traces the grant is
// the start of the busy step, so grant = end - busy for apps that request
// memory and end, NEVER otherwise (memshare/harness.py:514-531).  With both
// tick arrays requested, K5 packs a chunk's end ticks and its per-app busy
// ticks as u16 (10 B per app at four policies instead of 16 B of u32 end
// ticks) into pinned staging, and host threads write the caller's grant and
// end arrays from it (streaming stores) while later chunks are still on the
// GPU: the pipeline is bound by host memory bandwidth ("End to
// end").  A chunk whose ticks do not fit 16 bits is copied as u32 end rows
// (the batch's end ticks stay on the device for the call) and its grants
// derived from the input records; when most chunks of a call did not fit,
// the next call of that shape copies u32 end ticks from the start.  Traces
// whose record reports a tick overflow (where grant = end - busy does not
// hold) are re-simulated with device grants afterwards.
namespace {

thread_local uint64_t t_h2d = 0, t_d2h = 0;  // sg_last_host_transfer

struct HostChunk {
    uint64_t t0, nt;
    cudaEvent_t done;
    uint32_t idx;  // chunk index (pack16 overflow flag)
};

constexpr int kPipeBufs = 8;  // at most; SGPU_PIPE_BUFS picks (default 4)
struct PipeStreams {
    std::mutex mu;
    cudaStream_t st[kPipeBufs] = {};
    // pinned: the batch's pack16 staging (end ticks, then busy ticks, u16)
    // and per-chunk overflow flags, grown on demand and kept
    uint16_t* stage = nullptr;
    size_t stage_cap = 0;
    uint32_t* flags = nullptr;
    size_t flags_cap = 0;
    // per (apps per trace, policies, devices): the last call found most
    // chunks beyond 16-bit ticks, so the next one copies u32 end ticks
    std::map<uint64_t, bool> prefer_u32;
};
// The CPUs local to a GPU (its PCI device's NUMA node, from sysfs): the host
// pipeline's threads run there, next to the memory the GPU's DMA uses.
// Returns the number of CPUs in `set` (0: unknown, leave affinity alone).
int gpu_local_cpus(int dev, cpu_set_t* set) {
    CPU_ZERO(set);
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return 0;
    for (char* c = bus; *c; c++) *c = (char)tolower(*c);
    char path[128];
    snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/local_cpulist", bus);
    FILE* f = fopen(path, "r");
    if (!f) return 0;
    char buf[1024] = {0};
    const size_t got = fread(buf, 1, sizeof(buf) - 1, f);
    fclose(f);
    buf[got] = 0;
    // "0-15,32-47"
    for (char* tok = strtok(buf, ",\n"); tok; tok = strtok(nullptr, ",\n")) {
        int a = -1, b = -1;
        if (sscanf(tok, "%d-%d", &a, &b) == 2) {
        } else if (sscanf(tok, "%d", &a) == 1) {
            b = a;
        } else {
            continue;
        }
        for (int c = a; c <= b && c >= 0 && c < CPU_SETSIZE; c++) CPU_SET(c, set);
    }
    return CPU_COUNT(set);
}

uint64_t env_u64z(const char* name, uint64_t dflt) {  // accepts 0
    const char* v = getenv(name);
    return v && atoll(v) >= 0 ? (uint64_t)atoll(v) : dflt;
}
uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* v = getenv(name);
    return v && atoll(v) > 0 ? (uint64_t)atoll(v) : dflt;
}

cudaError_t grow_pinned(void** p, size_t& cap, size_t need) {
    if (need <= cap) return cudaSuccess;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    cap = 0;
    const cudaError_t e = cudaMallocHost(p, need);
    if (e == cudaSuccess) cap = need;
    return e;
}
PipeStreams& pipe_streams(int dev) {
    static std::mutex m;
    static std::map<int, std::unique_ptr<PipeStreams>> all;
    std::lock_guard<std::mutex> lk(m);
    auto& p = all[dev];
    if (!p) p.reset(new PipeStreams());
    return *p;
}

// One (trace, policy) row: g = (mem != 0 && end != NEVER) ? end - busy : NEVER.
// AVX2 with streaming stores when the row is 32-byte aligned (the grant
// array is write-only here: no read-for-ownership traffic).
__attribute__((target("avx2"))) void grant_row_avx2(const uint32_t* mem, const uint32_t* busy,
                                                    const uint32_t* e, uint32_t* g, uint32_t n) {
    const __m256i never = _mm256_set1_epi32((int)SG_NEVER);
    const __m256i zero = _mm256_setzero_si256();
    uint32_t i = 0;
    for (; i + 8 <= n; i += 8) {
        const __m256i ev = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(e + i));
        const __m256i mv = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(mem + i));
        const __m256i bv = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(busy + i));
        const __m256i no = _mm256_or_si256(_mm256_cmpeq_epi32(mv, zero), _mm256_cmpeq_epi32(ev, never));
        const __m256i gv = _mm256_blendv_epi8(_mm256_sub_epi32(ev, bv), never, no);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(g + i), gv);
    }
    for (; i < n; i++) g[i] = (mem[i] != 0 && e[i] != SG_NEVER) ? e[i] - busy[i] : SG_NEVER;
}

void grant_row_scalar(const uint32_t* mem, const uint32_t* busy, const uint32_t* e, uint32_t* g,
                      uint32_t n) {
    for (uint32_t i = 0; i < n; i++) g[i] = (mem[i] != 0 && e[i] != SG_NEVER) ? e[i] - busy[i] : SG_NEVER;
}

// One (trace, policy) row from the pack16 staging: end = e16 (0xFFFF ->
// NEVER), grant = (b16 != 0xFFFF && e16 != 0xFFFF) ? end - busy : NEVER;
// both written with streaming stores when `vec` (32-byte aligned rows).
__attribute__((target("avx2"))) void tick_row16_avx2(const uint16_t* b16, const uint16_t* e16, uint32_t* g,
                                                     uint32_t* e, uint32_t n) {
    const __m256i never = _mm256_set1_epi32((int)SG_NEVER);
    const __m256i none = _mm256_set1_epi32(0xFFFF);
    uint32_t i = 0;
    for (; i + 8 <= n; i += 8) {
        const __m256i bv = _mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i*>(b16 + i)));
        const __m256i ev = _mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i*>(e16 + i)));
        const __m256i en = _mm256_cmpeq_epi32(ev, none);
        const __m256i no = _mm256_or_si256(_mm256_cmpeq_epi32(bv, none), en);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(e + i), _mm256_or_si256(ev, en));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(g + i),
                            _mm256_blendv_epi8(_mm256_sub_epi32(ev, bv), never, no));
    }
    for (; i < n; i++) {
        e[i] = e16[i] == 0xFFFFu ? SG_NEVER : e16[i];
        g[i] = (b16[i] != 0xFFFFu && e16[i] != 0xFFFFu) ? (uint32_t)e16[i] - b16[i] : SG_NEVER;
    }
}

void tick_row16_scalar(const uint16_t* b16, const uint16_t* e16, uint32_t* g, uint32_t* e, uint32_t n) {
    for (uint32_t i = 0; i < n; i++) {
        e[i] = e16[i] == 0xFFFFu ? SG_NEVER : e16[i];
        g[i] = (b16[i] != 0xFFFFu && e16[i] != 0xFFFFu) ? (uint32_t)e16[i] - b16[i] : SG_NEVER;
    }
}

// end and grant ticks of policies [p0, npol) for traces [t_lo, t_hi) from
// the pack16 staging (stage: npol - p0 rows of end ticks, then the busy
// ticks, n_apps_total each);
// traces with a tick overflow are skipped and reported.
void expand_ticks16(const sg_batch* in, const sg_out* out, const uint16_t* stage, uint32_t p0, uint32_t npol,
                    uint64_t t_lo, uint64_t t_hi, std::vector<uint64_t>& overflow, bool avx2) {
    const uint64_t N = in->n_traces;
    const uint32_t napps = in->apps_per_trace, ndev = in->ndev;
    const uint64_t total = N * napps;
    const sg_trace_stats* st = static_cast<const sg_trace_stats*>(out->stats);
    uint32_t* end = static_cast<uint32_t*>(out->end);
    uint32_t* grant = static_cast<uint32_t*>(out->grant);
    const uint16_t* b16 = stage + (uint64_t)(npol - p0) * total;
    const bool vec = avx2 && (napps % 8 == 0) && (reinterpret_cast<uintptr_t>(grant) & 31u) == 0 &&
                     (reinterpret_cast<uintptr_t>(end) & 31u) == 0 && ((total * 4) & 31u) == 0;
    for (uint64_t t = t_lo; t < t_hi; t++) {
        bool ov = false;
        for (uint32_t p = 0; p < npol; p++)
            for (uint32_t d = 0; d < ndev; d++)
                ov = ov || (st[((uint64_t)p * N + t) * ndev + d].status & SG_ST_TICK_OVERFLOW);
        if (ov) { overflow.push_back(t); continue; }
        for (uint32_t p = p0; p < npol; p++) {
            const uint64_t o = (uint64_t)p * total + t * napps, so = (uint64_t)(p - p0) * total + t * napps;
            if (vec) tick_row16_avx2(b16 + t * napps, stage + so, grant + o, end + o, napps);
            else tick_row16_scalar(b16 + t * napps, stage + so, grant + o, end + o, napps);
        }
    }
    if (vec) _mm_sfence();
}

// grant[p][a] for traces [t_lo, t_hi) of the batch, from the end ticks and
// the input records; overflowing (trace, policy) pairs are skipped and
// reported.
void derive_grants(const sg_batch* in, const sg_out* out, uint32_t p0, uint32_t npol, uint64_t t_lo, uint64_t t_hi,
                   std::vector<uint64_t>& overflow, bool avx2) {
    const uint64_t N = in->n_traces;
    const uint32_t napps = in->apps_per_trace, ndev = in->ndev;
    const uint64_t total = N * napps;
    const sg_trace_stats* st = static_cast<const sg_trace_stats*>(out->stats);
    const uint32_t* end = static_cast<const uint32_t*>(out->end);
    uint32_t* grant = static_cast<uint32_t*>(out->grant);
    std::vector<uint32_t> mem(napps), busy(napps);
    const bool vec = avx2 && (napps % 8 == 0) &&
                     (reinterpret_cast<uintptr_t>(grant) & 31u) == 0 && ((total * 4) & 31u) == 0;
    for (uint64_t t = t_lo; t < t_hi; t++) {
        const sg_app* ap = in->apps + t * napps;
        for (uint32_t i = 0; i < napps; i++) {
            mem[i] = ap[i].mem_mib;
            busy[i] = ap[i].busy;
        }
        bool ov_any = false;
        for (uint32_t p = p0; p < npol; p++) {
            bool ov = false;
            for (uint32_t d = 0; d < ndev; d++)
                ov = ov || (st[((uint64_t)p * N + t) * ndev + d].status & SG_ST_TICK_OVERFLOW);
            if (ov) { ov_any = true; continue; }
            const uint32_t* e = end + (uint64_t)p * total + t * napps;
            uint32_t* g = grant + (uint64_t)p * total + t * napps;
            if (vec) grant_row_avx2(mem.data(), busy.data(), e, g, napps);
            else grant_row_scalar(mem.data(), busy.data(), e, g, napps);
        }
        if (ov_any) overflow.push_back(t);
    }
    if (vec) _mm_sfence();
}

}  // namespace

void sg_last_host_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
    if (h2d_bytes) *h2d_bytes = t_h2d;
    if (d2h_bytes) *d2h_bytes = t_d2h;
}

namespace {
int simulate_host(const sg_batch* in, const sg_out* out, int cuda_device, uint64_t chunk_traces, bool allow_pack);
}

int sg_simulate_batch_host(const sg_batch* in, const sg_out* out, int cuda_device,
                           uint64_t chunk_traces) {
    t_h2d = t_d2h = 0;
    return simulate_host(in, out, cuda_device, chunk_traces, true);
}

}  // extern "C"

namespace {

int simulate_host(const sg_batch* in, const sg_out* out, int cuda_device, uint64_t chunk_traces, bool allow_pack) {
    Shape s;
    int rc = validate(in, s);
    if (rc) return rc;
    if (!out || !out->stats) return fail(E_ARG, "sg_out.stats is required");
    if (out->events) return fail(E_ARG, "event logs are not supported on the host path");
    if (in->trace_offsets) return fail(E_ARG, "host path takes fixed-length traces");
    if (s.program) return fail(E_ARG, "host path takes T0 (burst) traces");
    if (in->n_traces == 0) return 0;
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    const uint64_t N = in->n_traces;
    const uint32_t napps = in->apps_per_trace;
    const uint32_t ndev = in->ndev;
    if (chunk_traces == 0) chunk_traces = 1u << 16;
    if (chunk_traces > N) chunk_traces = N;
    // grants derived on the host when both tick arrays are requested
    const bool host_grant = out->grant != nullptr && out->end != nullptr;
    // With both tick arrays requested, the grants of policies [0, n_dma) are
    // copied from the device and those of [n_dma, npol) derived by host
    // threads.  Deriving all of them measured best on two of three boxes
    // (36.6-37.2 vs 38.6 ms per C2 step; the third favoured copying one
    // policy): the pipeline is host-memory bound ("End to end").
    // SGPU_GRANT_DMA overrides.
    uint32_t n_dma = host_grant ? 0u : s.npol;
    if (const char* ev = getenv("SGPU_GRANT_DMA")) {
        const int v = atoi(ev);
        if (host_grant && v >= 0) n_dma = (uint32_t)v < s.npol ? (uint32_t)v : s.npol;
    }
    const bool derive = host_grant && n_dma < s.npol;
    // All grants derived: end + busy ticks cross PCIe as u16 (K5 pack16)
    // unless SGPU_PACK16=0 or the last call of this shape on the device found
    // most chunks beyond 16 bits (then u32 end ticks, with K5 still flagging
    // each chunk so the choice is re-made on the next call).
    const bool pack_ok = allow_pack && derive && n_dma == 0 &&
                         !(getenv("SGPU_PACK16") && atoi(getenv("SGPU_PACK16")) == 0);
    const int NBUF = (int)std::min<uint64_t>(std::max<uint64_t>(env_u64("SGPU_PIPE_BUFS", 4), 2), kPipeBufs);
    const size_t app_b = chunk_traces * napps * sizeof(sg_app);
    const size_t tick_b = (size_t)s.npol * chunk_traces * napps * sizeof(uint32_t);
    const size_t st_b = (size_t)s.npol * chunk_traces * ndev * sizeof(sg_trace_stats);
    const size_t pct_b = (size_t)s.npol * chunk_traces * ndev * sizeof(double);
    const bool want_pct = out->mem_pct || out->dev_pct;

    struct Buf {
        cudaStream_t st = nullptr;
        sg_app* apps = nullptr;
        uint32_t *grant = nullptr, *end = nullptr;
        sg_trace_stats* stats = nullptr;
        double *mem = nullptr, *dev = nullptr, *spd = nullptr;
        uint16_t *b16 = nullptr, *e16 = nullptr;
        uint32_t* flag = nullptr;
    } B[kPipeBufs];
    std::vector<HostChunk> chunks;
    // Pipeline buffers come from the device's stream-ordered memory pool
    // (cudaMallocAsync), kept cached between calls: repeated calls pay no
    // cudaMalloc/cudaFree or implicit device synchronisation.
    sg::keep_pool_memory();  // after cudaSetDevice(cuda_device)
    // The pipeline's streams persist per device (created once, reused by
    // every call: their work-counter slots stay theirs); one host-pipeline
    // call per device at a time (they would share PCIe and host memory
    // bandwidth anyway).
    PipeStreams& ps = pipe_streams(cuda_device);
    std::unique_lock<std::mutex> pipe_lk(ps.mu);
    const uint64_t shape_key = (uint64_t)napps | (uint64_t)s.npol << 32 | (uint64_t)ndev << 40;
    const bool use_p16 = pack_ok && !ps.prefer_u32[shape_key];
    const bool flag_only = pack_ok && !use_p16;  // u32 transfer, K5 overflow flags only
    // pack16: the first k policies still cross as u32 grant + end rows
    // straight into the caller's arrays (PCIe instead of host memory: the
    // two are balanced at k ~ npol / 2 on a host-memory-bound box;
    // SGPU_DIRECT_POLS=k)
    const uint32_t k_dir = use_p16 ? (uint32_t)std::min<uint64_t>(env_u64z("SGPU_DIRECT_POLS", 0), s.npol - 1u) : 0u;
    uint32_t* d_end_all_c = nullptr;  // (set below; freed here)
    uint32_t* d_grant_all_c = nullptr;
    auto cleanup = [&]() {
        if (d_end_all_c || d_grant_all_c) {  // every stream wrote them: drain them all first
            for (auto& b : B)
                if (b.st) cudaStreamSynchronize(b.st);
            if (d_end_all_c) cudaFreeAsync(d_end_all_c, B[0].st);
            if (d_grant_all_c) cudaFreeAsync(d_grant_all_c, B[0].st);
        }
        d_end_all_c = d_grant_all_c = nullptr;
        for (auto& b : B) {
            if (!b.st) continue;
            cudaFreeAsync(b.apps, b.st); cudaFreeAsync(b.grant, b.st); cudaFreeAsync(b.end, b.st);
            cudaFreeAsync(b.stats, b.st); cudaFreeAsync(b.mem, b.st); cudaFreeAsync(b.dev, b.st);
            cudaFreeAsync(b.spd, b.st); cudaFreeAsync(b.b16, b.st); cudaFreeAsync(b.e16, b.st);
            cudaFreeAsync(b.flag, b.st);
            cudaStreamSynchronize(b.st);
        }
        for (auto& c : chunks) cudaEventDestroy(c.done);
        if (pipe_lk.owns_lock()) pipe_lk.unlock();
    };
    for (int i = 0; i < NBUF; i++) {
        Buf& b = B[i];
        e = cudaSuccess;
        if (!ps.st[i]) e = cudaStreamCreateWithFlags(&ps.st[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) { ps.st[i] = nullptr; cleanup(); return cuda_fail(e, "pipeline streams"); }
        b.st = ps.st[i];
        if (e == cudaSuccess) e = cudaMallocAsync(&b.apps, app_b, b.st);
        if (e == cudaSuccess && out->grant && n_dma > 0) e = cudaMallocAsync(&b.grant, tick_b, b.st);
        if (e == cudaSuccess && out->end && !use_p16) e = cudaMallocAsync(&b.end, tick_b, b.st);
        if (e == cudaSuccess) e = cudaMallocAsync(&b.stats, st_b, b.st);
        if (e == cudaSuccess && want_pct) e = cudaMallocAsync(&b.mem, pct_b, b.st);
        if (e == cudaSuccess && want_pct) e = cudaMallocAsync(&b.dev, pct_b, b.st);
        if (e == cudaSuccess && out->speedup) e = cudaMallocAsync(&b.spd, pct_b, b.st);
        if (e == cudaSuccess && pack_ok) e = cudaMallocAsync(&b.b16, chunk_traces * napps * 2u, b.st);
        if (e == cudaSuccess && pack_ok) e = cudaMallocAsync(&b.e16, tick_b / 2u, b.st);
        if (e == cudaSuccess && pack_ok) e = cudaMallocAsync(&b.flag, 16, b.st);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "allocating pipeline buffers"); }
    }
    const uint64_t nch_max = (N + chunk_traces - 1) / chunk_traces;
    // pack16: the end ticks of the whole batch stay on the device for the
    // call (a chunk whose ticks do not fit 16 bits is then copied as u32
    // rows by the host thread that meets it, with no re-simulation)
    uint32_t* d_end_all = nullptr;
    uint32_t* d_grant_all = nullptr;
    if (use_p16 && k_dir > 0) {  // the kernel writes grants of every policy when asked for any
        e = cudaMallocAsync(&d_grant_all, (size_t)s.npol * N * napps * sizeof(uint32_t), B[0].st);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "allocating the batch's grant ticks"); }
        d_grant_all_c = d_grant_all;
    }
    if (use_p16) {
        e = cudaMallocAsync(&d_end_all, (size_t)s.npol * N * napps * sizeof(uint32_t), B[0].st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(B[0].st);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "allocating the batch's end ticks"); }
        d_end_all_c = d_end_all;
    }
    if (pack_ok) {
        e = use_p16 ? grow_pinned(reinterpret_cast<void**>(&ps.stage), ps.stage_cap,
                                  (s.npol - k_dir + 1u) * N * napps * 2u)
                    : cudaSuccess;
        if (e == cudaSuccess) e = grow_pinned(reinterpret_cast<void**>(&ps.flags), ps.flags_cap, nch_max * 4u + 64u);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "pinned pack16 staging"); }
    }
    const uint64_t n_apps_total = N * napps;
    // SGPU_PIPE_TRACE=1: print host-side pipeline timings (stderr)
    static const bool trace = getenv("SGPU_PIPE_TRACE") != nullptr;
    const auto tp0 = std::chrono::steady_clock::now();
    auto ms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count(); };
    // Chunk schedule: fixed-size chunks.  SGPU_PIPE_TAPER=1 fills (first
    // H2D + simulation before any D2H) and drains (last D2H + grant
    // derivation) on small chunks ramping from chunk/8: measured neutral
    // within box noise on C2 (42.4 vs 44.2 ms, then 47.3 vs 45.4 ms), so off.
    std::vector<std::pair<uint64_t, uint64_t>> sched;
    {
        static const bool taper = getenv("SGPU_PIPE_TAPER") && atoi(getenv("SGPU_PIPE_TAPER")) == 1;
        std::vector<uint64_t> head, tail;
        uint64_t left = N;
        if (taper && N >= 4 * chunk_traces) {
            for (uint64_t c = chunk_traces / 8; c < chunk_traces && c > 0; c *= 2) {
                head.push_back(c);
                tail.push_back(c);
                left -= 2 * c;
            }
        }
        uint64_t t0 = 0;
        for (uint64_t c : head) { sched.push_back({t0, c}); t0 += c; }
        while (left > 0) {
            const uint64_t c = left < chunk_traces ? left : chunk_traces;
            sched.push_back({t0, c});
            t0 += c;
            left -= c;
        }
        for (auto it = tail.rbegin(); it != tail.rend(); ++it) { sched.push_back({t0, *it}); t0 += *it; }
    }
    uint64_t chunk = 0;
    for (const auto& sc : sched) {
        const uint64_t t0 = sc.first, nt = sc.second;
        Buf& b = B[chunk % NBUF];
        chunk++;
        const uint64_t a0 = t0 * napps, na = nt * napps;
        e = cudaMemcpyAsync(b.apps, in->apps + a0, na * sizeof(sg_app), cudaMemcpyHostToDevice, b.st);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "H2D apps"); }
        t_h2d += na * sizeof(sg_app);
        sg_batch cb = *in;
        cb.n_traces = nt;
        cb.apps = b.apps;
        sg_out co;
        memset(&co, 0, sizeof(co));
        co.grant = use_p16 && k_dir ? d_grant_all + a0 : b.grant;
        co.end = use_p16 ? d_end_all + a0 : b.end;  // pack16: the batch-wide rows (stride n_apps_total)
        co.stats = b.stats;
        co.mem_pct = out->mem_pct ? b.mem : nullptr;
        co.dev_pct = out->dev_pct ? b.dev : nullptr;
        co.speedup = b.spd;
        rc = simulate_device(&cb, &co, b.st, use_p16 ? n_apps_total : na);
        if (rc) { cleanup(); return rc; }
        if (use_p16) {  // the chunk's end + busy ticks as u16 (K5) into the pinned staging
            const uint32_t np16 = s.npol - k_dir;
            e = sg::launch_pack16(b.apps, d_end_all + (uint64_t)k_dir * n_apps_total + a0, na, n_apps_total, np16,
                                  b.b16, b.e16, b.flag, b.st);
            for (uint32_t p = 0; p < np16 && e == cudaSuccess; p++)
                e = cudaMemcpyAsync(ps.stage + (uint64_t)p * n_apps_total + a0, b.e16 + (uint64_t)p * na, na * 2u,
                                    cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(ps.stage + (uint64_t)np16 * n_apps_total + a0, b.b16, na * 2u,
                                    cudaMemcpyDeviceToHost, b.st);
            // the first k_dir policies: u32 rows straight into the caller's arrays
            for (uint32_t p = 0; p < k_dir && e == cudaSuccess; p++) {
                const uint64_t o = (uint64_t)p * n_apps_total + a0;
                e = cudaMemcpyAsync(static_cast<uint32_t*>(out->end) + o, d_end_all + o, na * 4u,
                                    cudaMemcpyDeviceToHost, b.st);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(static_cast<uint32_t*>(out->grant) + o, d_grant_all + o, na * 4u,
                                        cudaMemcpyDeviceToHost, b.st);
            }
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(ps.flags + (chunk - 1), b.flag, 4, cudaMemcpyDeviceToHost, b.st);
            if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "K5 pack16"); }
            t_d2h += (np16 + 1u) * na * 2u + 4u + (uint64_t)k_dir * na * 8u;
        } else if (flag_only) {  // does this chunk fit 16 bits?  (re-decides the next call)
            e = sg::launch_pack16(b.apps, b.end, na, na, s.npol, b.b16, b.e16, b.flag, b.st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(ps.flags + (chunk - 1), b.flag, 4, cudaMemcpyDeviceToHost, b.st);
            if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "K5 flags"); }
            t_d2h += 4u;
        }
        for (uint32_t p = 0; p < s.npol; p++) {
            const uint64_t ho = (uint64_t)p * n_apps_total + a0;
            const uint64_t hs = ((uint64_t)p * N + t0) * ndev;
            const uint64_t dsrc = (uint64_t)p * nt * ndev;
            if (b.grant && p < n_dma)
                e = cudaMemcpyAsync(static_cast<uint32_t*>(out->grant) + ho, b.grant + (uint64_t)p * na,
                                    na * 4, cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess && out->end && !use_p16)
                e = cudaMemcpyAsync(static_cast<uint32_t*>(out->end) + ho, b.end + (uint64_t)p * na,
                                    na * 4, cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<sg_trace_stats*>(out->stats) + hs, b.stats + dsrc,
                                    nt * ndev * sizeof(sg_trace_stats), cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess && out->mem_pct)
                e = cudaMemcpyAsync(out->mem_pct + hs, b.mem + dsrc, nt * ndev * 8,
                                    cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess && out->dev_pct)
                e = cudaMemcpyAsync(out->dev_pct + hs, b.dev + dsrc, nt * ndev * 8,
                                    cudaMemcpyDeviceToHost, b.st);
            if (e == cudaSuccess && out->speedup)
                e = cudaMemcpyAsync(out->speedup + hs, b.spd + dsrc, nt * ndev * 8,
                                    cudaMemcpyDeviceToHost, b.st);
            if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "D2H outputs"); }
            t_d2h += (b.grant && p < n_dma ? na * 4u : 0u) + (out->end && !use_p16 ? na * 4u : 0u) +
                     nt * ndev * (sizeof(sg_trace_stats) + 8u * (!!out->mem_pct + !!out->dev_pct + !!out->speedup));
        }
        if (derive) {
            HostChunk c{t0, nt, nullptr, (uint32_t)(chunk - 1)};
            e = cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(c.done, b.st);
            if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "chunk event"); }
            chunks.push_back(c);
        }
    }
    std::vector<uint64_t> overflow;
    if (derive) {
        // host threads follow the pipeline chunk by chunk, each deriving the
        // grants of its contiguous share of every chunk's traces
        const bool avx2 = __builtin_cpu_supports("avx2");
        unsigned nthr = std::thread::hardware_concurrency();
        // one process per GPU shares the host: each rank's pipeline takes its
        // share of the cores (LOCAL_WORLD_SIZE, set by torch.distributed.run)
        if (const char* lw = getenv("LOCAL_WORLD_SIZE")) {
            const int n = atoi(lw);
            if (n > 1) nthr = nthr / (unsigned)n;
        }
        nthr = nthr == 0 ? 1 : (nthr > 16 ? 16 : nthr);
        if (const char* ev = getenv("SGPU_HOST_THREADS")) {  // tuning knob
            const int v = atoi(ev);
            if (v > 0 && v <= 256) nthr = (unsigned)v;
        }
        // threads on the GPU's NUMA node (SGPU_NUMA_BIND=0: no binding)
        cpu_set_t local;
        const bool bind = !(getenv("SGPU_NUMA_BIND") && atoi(getenv("SGPU_NUMA_BIND")) == 0) &&
                          gpu_local_cpus(cuda_device, &local) > 0;
        std::vector<std::vector<uint64_t>> ov(nthr);
        std::vector<cudaError_t> errs(nthr, cudaSuccess);
        std::vector<std::thread> pool;
        if (trace) fprintf(stderr, "[pipe] enqueued %zu chunks at %.2f ms (threads %u, numa bind %d)\n",
                           chunks.size(), ms(), nthr, (int)bind);
        for (unsigned w = 0; w < nthr; w++) {
            pool.emplace_back([&, w]() {
                if (bind) pthread_setaffinity_np(pthread_self(), sizeof(local), &local);
                for (const auto& c : chunks) {
                    const cudaError_t ce = cudaEventSynchronize(c.done);
                    if (ce != cudaSuccess) { errs[w] = ce; return; }
                    const double tr = ms();
                    const uint64_t lo = c.t0 + c.nt * w / nthr, hi = c.t0 + c.nt * (w + 1) / nthr;
                    if (!use_p16) {
                        derive_grants(in, out, n_dma, s.npol, lo, hi, ov[w], avx2);
                    } else if (ps.flags[c.idx]) {
                        // not exact in 16 bits: this thread's traces as u32 end rows
                        // from the device, grants from the input records
                        cudaError_t ce2 = cudaSuccess;
                        for (uint32_t p = k_dir; p < s.npol && ce2 == cudaSuccess && hi > lo; p++) {
                            const uint64_t o = (uint64_t)p * n_apps_total + lo * napps;
                            ce2 = cudaMemcpy(static_cast<uint32_t*>(out->end) + o, d_end_all + o,
                                             (hi - lo) * napps * sizeof(uint32_t), cudaMemcpyDeviceToHost);
                        }
                        if (ce2 != cudaSuccess) { errs[w] = ce2; return; }
                        derive_grants(in, out, k_dir, s.npol, lo, hi, ov[w], avx2);
                    } else {
                        expand_ticks16(in, out, ps.stage, k_dir, s.npol, lo, hi, ov[w], avx2);
                    }
                    if (trace && w == 0) fprintf(stderr, "[pipe] chunk at trace %llu ready %.2f derived %.2f ms\n", (unsigned long long)c.t0, tr, ms());
                }
            });
        }
        for (auto& th : pool) th.join();
        if (trace) fprintf(stderr, "[pipe] joined %.2f ms\n", ms());
        if (pack_ok) {  // most chunks beyond 16 bits: the next call of this shape copies u32 ticks
            uint64_t wide = 0;
            for (const auto& c : chunks) wide += ps.flags[c.idx] ? 1u : 0u;
            ps.prefer_u32[shape_key] = 2 * wide > chunks.size();
        }
        for (unsigned w = 0; w < nthr; w++) {
            if (errs[w] != cudaSuccess) { cleanup(); return cuda_fail(errs[w], "pipeline"); }
            overflow.insert(overflow.end(), ov[w].begin(), ov[w].end());
        }
    }
    for (auto& b : B) {
        e = cudaStreamSynchronize(b.st);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "pipeline"); }
    }
    cleanup();
    if (!overflow.empty()) {
        // the (rare) traces of a chunk whose ticks did not fit 16 bits (both
        // tick arrays) or with a tick overflow (grants): re-simulate them
        // with u32 ticks from the device
        std::sort(overflow.begin(), overflow.end());
        const uint64_t no = overflow.size();
        std::vector<sg_app> h_apps(no * napps);
        for (uint64_t k = 0; k < no; k++)
            memcpy(&h_apps[k * napps], in->apps + overflow[k] * napps, napps * sizeof(sg_app));
        sg_batch rb = *in;
        rb.n_traces = no;
        rb.apps = h_apps.data();
        std::vector<uint32_t> g((size_t)s.npol * no * napps), en(use_p16 ? (size_t)s.npol * no * napps : 0);
        std::vector<sg_trace_stats> rs((size_t)s.npol * no * ndev);
        sg_out ro;
        memset(&ro, 0, sizeof(ro));
        ro.grant = g.data();
        ro.end = use_p16 ? en.data() : nullptr;  // no end buffer: the call copies device grants
        ro.stats = rs.data();
        rc = simulate_host(&rb, &ro, cuda_device, 0, false);
        if (rc) return rc;
        for (uint64_t k = 0; k < no; k++)
            for (uint32_t p = 0; p < s.npol; p++) {
                const uint64_t o = (uint64_t)p * n_apps_total + overflow[k] * napps, r = ((uint64_t)p * no + k) * napps;
                memcpy(static_cast<uint32_t*>(out->grant) + o, &g[r], napps * sizeof(uint32_t));
                if (use_p16) memcpy(static_cast<uint32_t*>(out->end) + o, &en[r], napps * sizeof(uint32_t));
            }
    }
    return 0;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- small batches

namespace {
// Per (thread, device): a stream, pinned staging for inputs and outputs, and
// a device buffer, grown on demand and kept for the thread's lifetime.
struct SmallCtx {
    cudaStream_t st = nullptr;
    uint8_t* h_in = nullptr;
    uint8_t* h_out = nullptr;
    uint8_t* d_buf = nullptr;
    size_t cap_in = 0, cap_out = 0, cap_d = 0;
};
thread_local std::map<int, SmallCtx> t_small;

inline size_t al16(size_t x) { return (x + 15u) & ~(size_t)15u; }

cudaError_t small_grow(SmallCtx& c, size_t in_b, size_t out_b) {
    cudaError_t e = cudaSuccess;
    if (!c.st) e = cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking);
    if (e == cudaSuccess && in_b > c.cap_in) {
        if (c.h_in) cudaFreeHost(c.h_in);
        c.cap_in = std::max<size_t>(in_b, 1u << 16);
        e = cudaMallocHost(reinterpret_cast<void**>(&c.h_in), c.cap_in);
        if (e != cudaSuccess) { c.h_in = nullptr; c.cap_in = 0; }

    }
    if (e == cudaSuccess && out_b > c.cap_out) {
        if (c.h_out) cudaFreeHost(c.h_out);
        c.cap_out = std::max<size_t>(out_b, 1u << 16);
        e = cudaMallocHost(reinterpret_cast<void**>(&c.h_out), c.cap_out);
        if (e != cudaSuccess) { c.h_out = nullptr; c.cap_out = 0; }
    }
    if (e == cudaSuccess && in_b + out_b > c.cap_d) {
        if (c.d_buf) {
            cudaStreamSynchronize(c.st);
            cudaFree(c.d_buf);
        }
        c.cap_d = std::max<size_t>(in_b + out_b, 1u << 17);
        e = cudaMalloc(reinterpret_cast<void**>(&c.d_buf), c.cap_d);
        if (e != cudaSuccess) { c.d_buf = nullptr; c.cap_d = 0; }
        // defined bytes in the alignment gaps of the packed output (copied back whole)
        else e = cudaMemsetAsync(c.d_buf, 0, c.cap_d, c.st);
    }
    return e;
}
}  // namespace

int sg_simulate_small_host(const sg_batch* in, const sg_out* out, int cuda_device) {
    Shape s;
    int rc = validate(in, s);
    if (rc) return rc;
    if (!out || !out->stats) return fail(E_ARG, "sg_out.stats is required");
    if (in->trace_offsets) return fail(E_ARG, "sg_simulate_small_host takes fixed-length traces");
    if (in->n_traces == 0) return 0;
    if (s.program && !in->step_offsets) return fail(E_ARG, "steps given without step_offsets");
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    const uint64_t nt = in->n_traces, A = nt * in->apps_per_trace;
    const uint32_t npol = s.npol, ndev = in->ndev;
    const size_t tsz = s.f64 ? 8 : 4, rec = s.f64 ? sizeof(sg_trace_stats_f64) : sizeof(sg_trace_stats);
    // input region: apps | step_offsets | steps
    uint64_t n_steps = 0;
    uint32_t so0 = 0;
    if (s.program) {
        so0 = in->step_offsets[0];
        n_steps = in->step_offsets[A] - so0;
    }
    const size_t o_apps = 0, o_so = al16(A * sizeof(sg_app)),
                 o_steps = al16(o_so + (s.program ? (A + 1) * 4 : 0)),
                 in_b = al16(o_steps + n_steps * sizeof(sg_step));
    // output region
    const uint64_t nrec = (uint64_t)npol * nt * ndev;
    const size_t o_grant = 0, o_end = al16(out->grant ? npol * A * tsz : 0);
    const size_t o_stats = al16(o_end + (out->end ? npol * A * tsz : 0));
    const size_t o_mem = al16(o_stats + nrec * rec);
    const size_t o_dev = al16(o_mem + (out->mem_pct ? nrec * 8 : 0));
    const size_t o_spd = al16(o_dev + (out->dev_pct ? nrec * 8 : 0));
    const size_t o_ev = al16(o_spd + (out->speedup ? nrec * 8 : 0));
    const size_t ev_b = out->events ? (size_t)npol * nt * out->events_per_trace * sizeof(sg_event) : 0;
    const size_t o_cnt = al16(o_ev + ev_b);
    const size_t out_b = al16(o_cnt + (out->event_counts ? npol * nt * 4 : 0));
    SmallCtx& c = t_small[cuda_device];
    e = small_grow(c, in_b, out_b);
    if (e != cudaSuccess) return cuda_fail(e, "small-batch buffers");
    memcpy(c.h_in + o_apps, in->apps, A * sizeof(sg_app));
    size_t filled = A * sizeof(sg_app);
    if (s.program) {
        memset(c.h_in + filled, 0, o_so - filled);  // alignment gap (no uninitialised bytes go H2D)
        uint32_t* so = reinterpret_cast<uint32_t*>(c.h_in + o_so);
        for (uint64_t i = 0; i <= A; i++) so[i] = in->step_offsets[i] - so0;
        filled = o_so + (A + 1) * 4;
        memset(c.h_in + filled, 0, o_steps - filled);
        memcpy(c.h_in + o_steps, in->steps, n_steps * sizeof(sg_step));
        filled = o_steps + n_steps * sizeof(sg_step);
    }
    memset(c.h_in + filled, 0, in_b - filled);
    uint8_t* d_in = c.d_buf;
    uint8_t* d_out = c.d_buf + in_b;
    e = cudaMemcpyAsync(d_in, c.h_in, in_b, cudaMemcpyHostToDevice, c.st);
    if (e == cudaSuccess && ev_b) e = cudaMemsetAsync(d_out + o_ev, 0, ev_b, c.st);
    if (e != cudaSuccess) return cuda_fail(e, "small-batch H2D");
    sg_batch b = *in;
    b.apps = reinterpret_cast<const sg_app*>(d_in + o_apps);
    b.steps = s.program ? reinterpret_cast<const sg_step*>(d_in + o_steps) : nullptr;
    b.step_offsets = s.program ? reinterpret_cast<const uint32_t*>(d_in + o_so) : nullptr;
    sg_out o;
    memset(&o, 0, sizeof(o));
    o.grant = out->grant ? d_out + o_grant : nullptr;
    o.end = out->end ? d_out + o_end : nullptr;
    o.stats = d_out + o_stats;
    o.mem_pct = out->mem_pct ? reinterpret_cast<double*>(d_out + o_mem) : nullptr;
    o.dev_pct = out->dev_pct ? reinterpret_cast<double*>(d_out + o_dev) : nullptr;
    o.speedup = out->speedup ? reinterpret_cast<double*>(d_out + o_spd) : nullptr;
    o.events = out->events ? reinterpret_cast<sg_event*>(d_out + o_ev) : nullptr;
    o.event_counts = out->event_counts ? reinterpret_cast<uint32_t*>(d_out + o_cnt) : nullptr;
    o.events_per_trace = out->events_per_trace;
    rc = simulate_device(&b, &o, c.st, A);
    if (rc) return rc;
    e = cudaMemcpyAsync(c.h_out, d_out, out_b, cudaMemcpyDeviceToHost, c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) return cuda_fail(e, "small-batch D2H");
    if (out->grant) memcpy(out->grant, c.h_out + o_grant, npol * A * tsz);
    if (out->end) memcpy(out->end, c.h_out + o_end, npol * A * tsz);
    memcpy(out->stats, c.h_out + o_stats, nrec * rec);
    if (out->mem_pct) memcpy(out->mem_pct, c.h_out + o_mem, nrec * 8);
    if (out->dev_pct) memcpy(out->dev_pct, c.h_out + o_dev, nrec * 8);
    if (out->speedup) memcpy(out->speedup, c.h_out + o_spd, nrec * 8);
    if (out->events) memcpy(out->events, c.h_out + o_ev, ev_b);
    if (out->event_counts) memcpy(out->event_counts, c.h_out + o_cnt, npol * nt * 4);
    return 0;
}

int sg_reduce_stats(const sg_trace_stats* stats, uint64_t count, sg_aggr* out, void* stream) {
    if (!out || (count && !stats)) return fail(E_ARG, "null pointer");
    cudaError_t e = sg::launch_reduce(stats, count, out, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "stats_reduce");
    return 0;
}

int sg_generate_traces(const sg_gen_params* p, uint64_t trace_begin, uint64_t n_traces,
                       sg_app* out, void* stream) {
    if (!p || (n_traces && !out)) return fail(E_ARG, "null pointer");
    if (p->apps_per_trace == 0 || p->apps_per_trace > SG_MAX_APPS)
        return fail(E_RANGE, "apps_per_trace must be 1..%d", SG_MAX_APPS);
    if (p->prio_levels < 1 || p->prio_levels > 8) return fail(E_RANGE, "prio_levels must be 1..8");
    if (p->ndev < 1 || p->ndev > SG_MAX_DEV) return fail(E_RANGE, "ndev must be 1..8");
    if (p->arr_hi < p->arr_lo || p->mem_hi < p->mem_lo || p->busy_hi < p->busy_lo)
        return fail(E_RANGE, "empty generator range");
    cudaError_t e = sg::launch_generate(*p, trace_begin, n_traces, out, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "trace_gen");
    return 0;
}

int sg_select_grants_batch(uint64_t n_queues, const uint64_t* qoff, const int64_t* nbytes,
                           const int32_t* prio, const int64_t* free_bytes, const uint32_t* kind,
                           uint8_t* granted, void* stream) {
    if (n_queues && (!qoff || !free_bytes || !kind)) return fail(E_ARG, "null pointer");
    cudaError_t e = sg::launch_select(n_queues, qoff, nbytes, prio, free_bytes, kind, granted,
                                      static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "select_grants");
    return 0;
}

}  // extern "C"
