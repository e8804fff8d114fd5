"""Drop-in for the reference's simulated workload path (memshare/harness.py).

Same public names and semantics as the reference module's SIMULATED mode:
`Phase`, `AppProfile`, `builtin_profiles`, `DEFAULT_DEVICE`, `WorkloadSpec`
(+ `from_json`), `MetricsReport` (+ `summary`/`to_json`/`to_csv`), `TICK_MS`
and `simulate(spec) -> MetricsReport`.  The real-process runner, sequential
baseline and overhead bench of the reference (harness.py:173-370, 575-678)
are out of scope.

`simulate` runs the spec as ONE trace through the CUDA engine
(K1 `trace_sim`, step-program mode, event log on) and rebuilds the
reference's report from the GPU's outputs:
  * times: if every step duration `ms * time_scale / 1000.0` (computed with
    the reference's own float expression, harness.py:483,487) lies on a
    2^-e s grid with all sums exact, the engine runs in integer ticks of
    2^-e s — every event time is then bit-identical to the reference's float
    time; otherwise it runs in float64 mode, which repeats the reference's
    float additions (`now + arg`) in the same order;
  * makespan, utilisation percentages and max concurrent holders come from
    the kernel's fused statistics (harness.py:373-461 semantics);
  * the event list / instance table / 100 ms memory trace are assembled on
    the host from the GPU event log, exactly as the reference formats them
    (stable sort by t, harness.py:567; trace loop, harness.py:439-450).
"""

from __future__ import annotations

import ctypes
import json
import math
import struct
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .batch import STATS_DTYPE, STATS_F64_DTYPE, STEP_DTYPE, simulate_batch
from .device import MIB, DeviceSpec, parse_device_config
from .errors import SchemaError, SgpuUnavailable
from .policy import PolicyKind

TICK_MS = 100  # utilisation sampling tick (harness.py:36)


@dataclass
class Phase:
    cpu_ms: float = 0.0
    alloc_mib: int = 0
    busy_ms: float = 0.0
    free_mib: int = 0


@dataclass
class AppProfile:
    name: str
    phases: list[Phase]
    priority: int = 0

    def peak_mib(self) -> int:
        held = peak = 0
        for p in self.phases:
            held += p.alloc_mib
            peak = max(peak, held)
            held -= p.free_mib
        return peak

    def total_ms(self) -> float:
        """Sequential (uncontended) run time: the speed-up denominator."""
        return sum(p.cpu_ms + p.busy_ms for p in self.phases)


def builtin_profiles() -> dict[str, AppProfile]:
    """The reference's three desk-scale application shapes
    (memshare/harness.py:65-83): ara-like (CPU-heavy, short 768 MiB burst at
    the end), mummer-like (720 MiB held through 10 alternating 500 ms
    cpu/busy rounds), blast-like (1750 MiB, 8 s busy between 1 s cpu)."""
    ara = AppProfile("ara-like", [Phase(cpu_ms=9500),
                                  Phase(alloc_mib=768, busy_ms=500, free_mib=768)])
    rounds = [Phase(cpu_ms=500), Phase(busy_ms=500)] * 10
    mummer = AppProfile("mummer-like", [Phase(alloc_mib=720)] + rounds + [Phase(free_mib=720)])
    blast = AppProfile("blast-like", [Phase(alloc_mib=1750, cpu_ms=1000), Phase(busy_ms=8000),
                                      Phase(cpu_ms=1000, free_mib=1750)])
    return {p.name: p for p in (ara, mummer, blast)}


DEFAULT_DEVICE = {"devices": [{"name": "K20m-sim", "mib": 4799}]}


@dataclass
class WorkloadSpec:
    instances: list[AppProfile]  # one entry per instance, in queue order
    policy: PolicyKind = PolicyKind.FIFO
    backend: str = "shm"
    devices: list[DeviceSpec] = None
    seed: int = 0
    time_scale: float = 1.0
    timeout_ms: float = math.inf
    kill_plan: list[tuple[int, float]] = field(default_factory=list)

    def __post_init__(self):
        if self.devices is None:
            self.devices = parse_device_config(DEFAULT_DEVICE)

    @classmethod
    def from_json(cls, doc: dict) -> "WorkloadSpec":
        """Workload JSON (memshare/harness.py:104-130; README.md:98-109)."""
        profiles = dict(builtin_profiles())
        for p in doc.get("profiles", []):
            phases = [Phase(ph.get("cpu_ms", 0), ph.get("alloc_mib", 0),
                            ph.get("busy_ms", 0), ph.get("free_mib", 0)) for ph in p["phases"]]
            profiles[p["name"]] = AppProfile(p["name"], phases, p.get("priority", 0))
        instances = []
        for name, count in doc.get("instances", []):
            if name not in profiles:
                raise SchemaError(f"unknown profile {name!r}")
            instances.extend([profiles[name]] * int(count))
        if not instances:
            raise SchemaError("workload has no instances")
        devices = parse_device_config(doc["device"]) if "device" in doc else None
        return cls(instances=instances, policy=PolicyKind.parse(doc.get("policy", "fifo")),
                   backend=doc.get("backend", "shm"), devices=devices,
                   seed=int(doc.get("seed", 0)),
                   time_scale=float(doc.get("time_scale", 1.0)),
                   timeout_ms=float(doc.get("timeout_ms", math.inf)))


@dataclass
class MetricsReport:
    makespan_ms: float
    instances: dict[int, dict]
    events: list[dict]
    mem_trace: list[tuple[float, float]]
    avg_mem_util_pct: float
    avg_device_util_pct: float
    oom_count: int
    max_concurrent_holders: int
    final_audit: list[str] = field(default_factory=list)

    def summary(self) -> dict:
        return {
            "makespan_ms": round(self.makespan_ms, 3),
            "avg_mem_util_pct": round(self.avg_mem_util_pct, 4),
            "avg_device_util_pct": round(self.avg_device_util_pct, 4),
            "oom_count": self.oom_count,
            "max_concurrent_holders": self.max_concurrent_holders,
            "instances": len(self.instances),
            "audit_ok": not self.final_audit,
        }

    def to_json(self) -> str:
        return json.dumps(self.summary(), indent=2)

    def to_csv(self) -> str:
        lines = ["t_ms,instance,event,device,bytes"]
        for e in self.events:
            lines.append(f"{e['t_ms']:.3f},{e['instance']},{e['event']},{e['device']},{e['bytes']}")
        s = self.summary()
        lines.append(f"# makespan_ms={s['makespan_ms']} avg_mem_util_pct={s['avg_mem_util_pct']} "
                     f"avg_device_util_pct={s['avg_device_util_pct']} oom_count={s['oom_count']}")
        return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ encoding

@dataclass
class EncodedTrace:
    """One workload as a step program (the general mode of include/sgpu.h)."""
    steps: np.ndarray          # STEP_DTYPE
    step_offsets: np.ndarray   # uint32, n + 1
    attr: np.ndarray           # uint32, n (priority rank | device << 8)
    time_mode: int
    tick_log2: int
    cap_mib: int


def _flatten_profile(prof: AppProfile, time_scale: float) -> list[tuple[int, object]]:
    """harness.py:478-490: cpu -> alloc -> busy -> free per phase, zero fields
    skipped, durations with the reference's float expression."""
    flat = []
    for ph in prof.phases:
        if ph.cpu_ms:
            flat.append((_lib.OP_CPU, ph.cpu_ms * time_scale / 1000.0))
        if ph.alloc_mib:
            flat.append((_lib.OP_ALLOC, ph.alloc_mib))
        if ph.busy_ms:
            flat.append((_lib.OP_BUSY, ph.busy_ms * time_scale / 1000.0))
        if ph.free_mib:
            flat.append((_lib.OP_FREE, ph.free_mib))
    return flat


def _tick_grid(durations: list[float], cap_mib: int, counts=None):
    """Smallest e such that every duration is an integer number of 2^-e s
    ticks and every reference float sum is exact (all times < 2^32 ticks,
    memory integral < 2^53).  None => use float64 mode.  counts[i]: how many
    times durations[i] occurs (default once)."""
    if not durations:
        return 10
    # a finite double is num / 2^k exactly (float.as_integer_ratio)
    fr = [float(d).as_integer_ratio() for d in durations]
    e = max(den.bit_length() - 1 for _, den in fr)
    if e > 62:
        return None
    cnt = counts or [1] * len(fr)
    total = sum(c * (num << (e - (den.bit_length() - 1))) for (num, den), c in zip(fr, cnt))
    if total >= 0xFFFFFFFE or cap_mib * total >= (1 << 53):
        return None
    return e


def encode_spec(spec: WorkloadSpec) -> EncodedTrace:
    """Step programs of the spec's instances for the C ABI.  Instances that
    share an AppProfile object (12 x "ara-like") are flattened, checked and
    encoded once per call."""
    cap_mib = spec.devices[0].total_bytes // MIB
    if spec.devices[0].total_bytes % MIB:
        raise ValueError("device capacity must be a whole number of MiB")
    uniq: dict[int, int] = {}      # id(profile) -> index into flats
    flats: list[list[tuple[int, object]]] = []
    which = []
    for prof in spec.instances:
        k = uniq.get(id(prof))
        if k is None:
            k = uniq[id(prof)] = len(flats)
            flats.append(_flatten_profile(prof, spec.time_scale))
        which.append(k)
    uses = [0] * len(flats)
    for k in which:
        uses[k] += 1
    durations, counts = [], []
    for flat, u in zip(flats, uses):
        for op, arg in flat:
            if op in (_lib.OP_CPU, _lib.OP_BUSY):
                if not (arg >= 0) or math.isinf(arg):
                    raise ValueError(f"step durations must be finite and >= 0 (got {arg!r})")
                durations.append(arg)
                counts.append(u)
            else:
                if int(arg) != arg or not 0 < int(arg) < 0x7FFFFFFF:
                    raise ValueError(f"memory sizes must be whole MiB in (0, 2^31) (got {arg!r})")
    e = _tick_grid(durations, cap_mib, counts)
    mode = _lib.TIME_TICKS if e is not None else _lib.TIME_F64
    # priorities: only order and equality matter (policy.py:58-63) -> dense ranks
    prios = sorted({int(p.priority) for p in spec.instances})
    if len(prios) > 256:
        raise ValueError("at most 256 distinct priorities per workload")
    rank = {p: i for i, p in enumerate(prios)}
    enc_rows = []
    for flat in flats:
        rows = []
        for op, arg in flat:
            if op in (_lib.OP_CPU, _lib.OP_BUSY):
                if mode == _lib.TIME_TICKS:
                    num, den = float(arg).as_integer_ratio()
                    dur = num << (e - (den.bit_length() - 1))
                else:
                    dur = struct.unpack("<Q", struct.pack("<d", float(arg)))[0]
                rows.append((op, 0, dur))
            else:
                rows.append((op, int(arg), 0))
        enc_rows.append(rows)
    offs_l = [0]
    all_rows = []
    for k in which:
        all_rows += enc_rows[k]
        offs_l.append(len(all_rows))
    offs = np.array(offs_l, dtype=np.uint32)
    steps = np.array(all_rows, dtype=STEP_DTYPE) if all_rows else np.zeros(1, dtype=STEP_DTYPE)
    attr = np.array([rank[int(p.priority)] for p in spec.instances], dtype=np.uint32)
    return EncodedTrace(steps, offs, attr, mode, e if e is not None else 0, cap_mib)


# ------------------------------------------------------------------ simulate

_CUDA_OK = None
_TLS = threading.local()


def _gpu_device() -> int:
    """The current CUDA device index (torch's), checked once per process."""
    global _CUDA_OK
    import torch
    if _CUDA_OK is None:
        _CUDA_OK = torch.cuda.is_available()
    if not _CUDA_OK:
        raise SgpuUnavailable("simulate() runs on the GPU; no CUDA device is available")
    return torch.cuda.current_device()


_EVENT_DTYPE = np.dtype([("t", "<u8"), ("app", "<u2"), ("kind", "u1"), ("dev", "u1"), ("mib", "<u4")])


def run_encoded(enc: EncodedTrace, policy) -> dict:
    """Run one encoded trace on the GPU with the event log through the C
    ABI's small-batch call (sg_simulate_small_host: one H2D copy, one
    launch, one D2H copy from persistent pinned staging); returns host
    outputs."""
    from .policy import as_policy
    L = _lib.lib()
    dev = _gpu_device()
    n = len(enc.attr)
    apps = np.zeros((n, 4), dtype=np.uint32)
    apps[:, 3] = enc.attr
    steps = np.ascontiguousarray(enc.steps)
    offs = np.ascontiguousarray(enc.step_offsets, dtype=np.uint32)
    ev_cap = 2 * n + 3 * int(offs[-1]) + 8
    f64 = enc.time_mode == _lib.TIME_F64
    stats = np.empty(1, dtype=STATS_F64_DTYPE if f64 else STATS_DTYPE)
    pct = np.empty(2, dtype=np.float64)
    events = np.empty(ev_cap, dtype=_EVENT_DTYPE)
    count = np.zeros(1, dtype=np.uint32)
    cache = getattr(_TLS, "abi", None)
    if cache is None:  # the ctypes argument structs, reused per thread
        cache = _TLS.abi = (_lib.SgBatch(), _lib.SgOut())
    b, o = cache
    ctypes.memset(ctypes.byref(b), 0, ctypes.sizeof(b))
    ctypes.memset(ctypes.byref(o), 0, ctypes.sizeof(o))
    b.n_traces = 1
    b.apps_per_trace = n
    b.max_apps = n
    b.apps = apps.ctypes.data
    b.steps = steps.ctypes.data
    b.step_offsets = offs.ctypes.data
    b.policy_mask = 1 << as_policy(policy).code
    b.ndev = 1
    b.cap_mib[0] = enc.cap_mib
    b.time_mode = enc.time_mode
    b.tick_log2 = enc.tick_log2
    o.stats = stats.ctypes.data
    o.mem_pct = pct.ctypes.data
    o.dev_pct = pct.ctypes.data + 8
    o.events = events.ctypes.data
    o.event_counts = count.ctypes.data
    o.events_per_trace = ev_cap
    _lib.check(L.sg_simulate_small_host(ctypes.byref(b), ctypes.byref(o), dev), "sg_simulate_small_host")
    c = int(count[0])
    return {"stats": stats[0], "events": events[:min(c, ev_cap)], "count": c, "ev_cap": ev_cap,
            "mem_pct": float(pct[0]), "dev_pct": float(pct[1])}


def _time_of(enc: EncodedTrace, raw: int) -> float:
    if enc.time_mode == _lib.TIME_TICKS:
        return math.ldexp(float(raw), -enc.tick_log2)
    return struct.unpack("<d", struct.pack("<Q", int(raw)))[0]


_BYTES_KIND_SET = frozenset((_lib.EV_REQUEST, _lib.EV_GRANT, _lib.EV_ALLOC, _lib.EV_FREE))


def simulate(spec: WorkloadSpec) -> MetricsReport:
    """Discrete-event prediction of `spec` (memshare/harness.py:475-572) on
    the GPU.  Deterministic; bit-identical to the reference's report.  The
    report is assembled from the GPU's event log (every float is produced by
    the same IEEE operation the reference performs)."""
    if not spec.instances:
        return MetricsReport(0.0, {}, [], [], 0.0, 0.0, 0, 0)
    enc = encode_spec(spec)
    out = run_encoded(enc, spec.policy)
    st = out["stats"]
    if out["count"] > out["ev_cap"]:
        raise _lib.SgpuError("event log overflow")
    status = int(st["status"])
    if status & (_lib.ST_TICK_OVERFLOW | _lib.ST_COUNTER_OVERFLOW | _lib.ST_BAD_DEVICE):
        raise _lib.SgpuError(f"simulation status 0x{status:x}")
    capacity = spec.devices[0].total_bytes
    ev = out["events"]
    kind_l = ev["kind"].tolist()
    app_l = ev["app"].tolist()
    mib_l = ev["mib"].tolist()
    if enc.time_mode == _lib.TIME_TICKS:
        # t = ticks * 2^-e exactly (as math.ldexp(float(ticks), -e))
        sc = 2.0 ** -enc.tick_log2
        t_all = [float(x) * sc for x in ev["t"].tolist()]
        t_end = math.ldexp(float(st["makespan"]), -enc.tick_log2)
    else:
        t_all = ev["t"].view(np.float64).tolist()
        t_end = float(st["makespan_s"])
    # plain Python below: a workload's log is short, and list operations beat
    # numpy's per-call overhead at this size
    order = sorted(range(len(t_all)), key=t_all.__getitem__)  # harness.py:567 (stable sort by t)
    names = _lib.EVENT_NAMES
    byte_kinds = _BYTES_KIND_SET
    makespan_s = max(t_end - 0.0, 1e-9)
    out_events = []
    n = len(enc.attr)
    starts = [None] * n
    ends = [None] * n
    mem_pts = []  # (t, delta bytes) of alloc / free, in sorted event order
    ev_start, ev_end, ev_alloc, ev_free = _lib.EV_START, _lib.EV_END, _lib.EV_ALLOC, _lib.EV_FREE
    for k in order:
        t = t_all[k]
        kd = kind_l[k]
        a = app_l[k]
        nb = mib_l[k] * MIB if kd in byte_kinds else 0
        t_ms = (t - 0.0) * 1000.0
        out_events.append({"t_ms": t_ms, "instance": a, "event": names[kd], "device": 0, "bytes": nb})
        if kd == ev_start:
            starts[a] = t_ms
        elif kd == ev_end:
            ends[a] = t_ms
        elif kd == ev_alloc:
            mem_pts.append((t, nb))
        elif kd == ev_free:
            mem_pts.append((t, -nb))
    # every app emits start at t = 0 (index order, first in the sorted log)
    # and at most one end: the reference's setdefault walk gives
    # {i: {"start_ms": .., "end_ms": ..}} in index order
    instances: dict[int, dict] = {}
    for i in range(n):
        d = {}
        if starts[i] is not None:
            d["start_ms"] = starts[i]
        if ends[i] is not None:
            d["end_ms"] = ends[i]
        instances[i] = d
    # 100 ms memory-utilisation samples (harness.py:439-450): the level at a
    # sample is the sum of every alloc/free delta at or before it
    mem_pts.sort(key=lambda x: x[0])
    trace = []
    level = 0
    j = 0
    npts = len(mem_pts)
    t = 0.0
    lim = makespan_s + 1e-9
    step = TICK_MS / 1000.0
    while t <= lim:
        while j < npts and mem_pts[j][0] <= t:
            level += mem_pts[j][1]
            j += 1
        trace.append((t * 1000.0, level / capacity))
        t += step
    report = MetricsReport(makespan_ms=makespan_s * 1000.0, instances=instances,
                           events=out_events, mem_trace=trace,
                           avg_mem_util_pct=out["mem_pct"], avg_device_util_pct=out["dev_pct"],
                           oom_count=0, max_concurrent_holders=int(st["max_holders"]))
    for idx, prof in enumerate(spec.instances):
        report.instances.setdefault(idx, {})["name"] = prof.name
        report.instances[idx]["exit"] = 0
    return report


def sequential_ms(spec: WorkloadSpec) -> float:
    """Sequential makespan of the spec (sum of AppProfile.total_ms scaled),
    the denominator of the concurrent speed-up (test_harness.py:119-126)."""
    return sum(p.total_ms() for p in spec.instances) * spec.time_scale


def speedup_vs_sequential(spec: WorkloadSpec, report: MetricsReport) -> float:
    """Concurrent speed-up over running the instances one after another:
    sum(p.total_ms() for p in instances) * time_scale / makespan_ms, in the
    reference's float order (harness.py:61-62; pkg/tests/test_harness.py:
    119-126, where sequential = 12 x 10 s).  The batch API emits the same
    value per (policy, trace, device) from the kernel (sg_out.speedup)."""
    return sequential_ms(spec) / report.makespan_ms


__all__ = ["Phase", "AppProfile", "builtin_profiles", "DEFAULT_DEVICE", "WorkloadSpec",
           "MetricsReport", "simulate", "encode_spec", "sequential_ms", "speedup_vs_sequential",
           "TICK_MS"]
