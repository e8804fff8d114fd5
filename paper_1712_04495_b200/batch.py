"""Batched trace simulation on the GPU: the data-parallel form of
memshare.harness.simulate (memshare/harness.py:475-572) over millions of
independent traces.

Device path (`simulate_batch`): inputs and outputs are CUDA tensors; one
launch of K1 `trace_sim` (one warp per trace, all requested policies per
trace) on the current torch stream.

Host path (`simulate_batch_host`): numpy / pinned host buffers; the C ABI
pipelines H2D copies, simulation and D2H copies in chunks over three CUDA
streams.  This is the end-to-end call a CPU user makes.

Layouts (include/sgpu.h):
  apps        (n_traces, n_apps, 4) uint32 T0 records, or (total_apps, 4)
              with CSR trace_offsets for ragged traces
  grant/end   (n_policies, total_apps) uint32 ticks (0xFFFFFFFF = never)
  stats       (n_policies, n_traces, ndev) STATS_DTYPE records (32 B)
  mem/dev pct (n_policies, n_traces, ndev) float64, reference op order
  speedup     (n_policies, n_traces, ndev) float64: sequential / concurrent
              makespan, sum(total_ms) * time_scale / makespan_ms in the
              reference's float order (harness.py:61-62,
              pkg/tests/test_harness.py:119-126), ticks mode
"""

from __future__ import annotations

import os

import ctypes
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from .errors import SgpuUnavailable
from .policy import PolicyKind, policy_mask

STATS_DTYPE = np.dtype([("makespan", "<u4"), ("busy", "<u4"), ("mem_integral", "<u8"),
                        ("grants", "<u4"), ("pops", "<u4"), ("max_holders", "<u2"),
                        ("unfinished", "<u2"), ("status", "<u4")])
STATS_F64_DTYPE = np.dtype([("makespan_s", "<f8"), ("mem_integral", "<f8"), ("busy_s", "<f8"),
                            ("grants", "<u4"), ("pops", "<u4"), ("max_holders", "<u2"),
                            ("unfinished", "<u2"), ("status", "<u4")])
STEP_DTYPE = np.dtype([("op", "<u4"), ("mib", "<u4"), ("dur", "<u8")])
EVENT_DTYPE = np.dtype([("t", "<u8"), ("app", "<u2"), ("kind", "u1"), ("dev", "u1"),
                        ("mib", "<u4")])
assert STATS_DTYPE.itemsize == 32 and STATS_F64_DTYPE.itemsize == 40
assert STEP_DTYPE.itemsize == 16 and EVENT_DTYPE.itemsize == 16


def _torch():
    import torch
    return torch


def _vp(t) -> Optional[ctypes.c_void_p]:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _require_cuda(t, name: str):
    if t is not None and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor for the device path")


def _caps(cap_mib) -> tuple[int, ...]:
    caps = tuple(int(c) for c in np.atleast_1d(np.asarray(cap_mib)).tolist())
    if not 1 <= len(caps) <= _lib.MAX_DEV:
        raise ValueError(f"1..{_lib.MAX_DEV} simulated devices per trace")
    return caps


@dataclass
class BatchResult:
    """Outputs of one simulate_batch call (CUDA tensors, policy-major)."""
    policies: tuple[PolicyKind, ...]
    n_traces: int
    ndev: int
    cap_mib: tuple[int, ...]
    time_mode: int
    tick_log2: int
    grant: object          # (npol, total_apps) int32 (uint32 bits) / float64 in F64 mode
    end: object
    stats_raw: object      # (npol, n_traces, ndev, 8 or 10) int32
    mem_pct: object        # (npol, n_traces, ndev) float64 or None
    dev_pct: object
    events: object = None  # (npol, n_traces, events_per_trace, 4) int32 or None
    event_counts: object = None
    speedup: object = None  # (npol, n_traces, ndev) float64 or None

    def stats(self) -> np.ndarray:
        """Per-(policy, trace, device) statistics as a numpy structured array."""
        dt = STATS_F64_DTYPE if self.time_mode == _lib.TIME_F64 else STATS_DTYPE
        raw = self.stats_raw.cpu().numpy()
        return np.ascontiguousarray(raw).view(dt).reshape(raw.shape[:3])

    def ticks(self, which: str = "grant") -> np.ndarray:
        t = getattr(self, which).cpu().numpy()
        return t if self.time_mode == _lib.TIME_F64 else t.view(np.uint32)

    def policy_index(self, policy) -> int:
        from .policy import as_policy
        return self.policies.index(as_policy(policy))


def simulate_batch(apps, policies: Iterable = ("fifo",), cap_mib=184_320, *,
                   trace_offsets=None, max_apps: Optional[int] = None,
                   steps=None, step_offsets=None, time_mode: int = _lib.TIME_TICKS,
                   tick_log2: int = 10, want_ticks: bool = True, want_pct: bool = True,
                   want_speedup: bool = True, events_per_trace: int = 0,
                   apps_total: Optional[int] = None, stream=None) -> BatchResult:
    """Simulate every trace under every requested policy on the GPU.

    apps: CUDA int32/uint32 tensor (n_traces, n_apps, 4), or (total_apps, 4)
    with `trace_offsets` (CUDA int64, n_traces + 1).  In step-program mode
    `steps` (CUDA int32 (n_steps, 4) = STEP_DTYPE records) and
    `step_offsets` (CUDA int32, total_apps + 1) define each app's program;
    apps[..., 3] still carries prio | device << 8.  With `trace_offsets`,
    `apps_total` (= offsets[-1] - offsets[0]) and `max_apps` avoid a device
    read on the host; the call is then asynchronous and graph-capturable.
    """
    torch = _torch()
    L = _lib.lib()
    if not torch.cuda.is_available():
        raise SgpuUnavailable("simulate_batch needs a CUDA device (there is no CPU fallback)")
    _require_cuda(apps, "apps")
    _require_cuda(trace_offsets, "trace_offsets")
    _require_cuda(steps, "steps")
    _require_cuda(step_offsets, "step_offsets")
    if apps.dtype not in (torch.int32, torch.uint32) or apps.shape[-1] != 4:
        raise ValueError("apps must be an int32 tensor with a trailing dimension of 4")
    apps = apps.contiguous()
    dev = apps.device
    mask, ordered = policy_mask(policies)
    caps = _caps(cap_mib)
    npol, ndev = len(ordered), len(caps)
    if trace_offsets is not None:
        if trace_offsets.dtype != torch.int64:
            raise ValueError("trace_offsets must be int64")
        n_traces = int(trace_offsets.numel()) - 1
        total_apps = int(apps.shape[0]) if apps_total is None else int(apps_total)
        if total_apps > int(apps.shape[0]):
            raise ValueError("apps_total exceeds the apps tensor")
        if max_apps is None:
            max_apps = int((trace_offsets[1:] - trace_offsets[:-1]).max().item()) if n_traces else 0
        napp = 0
    else:
        if apps.dim() != 3:
            raise ValueError("apps must be (n_traces, n_apps, 4) without trace_offsets")
        n_traces, napp = int(apps.shape[0]), int(apps.shape[1])
        total_apps = n_traces * napp
        max_apps = napp
    f64 = time_mode == _lib.TIME_F64
    tdt = torch.float64 if f64 else torch.int32
    grant = torch.empty((npol, total_apps), dtype=tdt, device=dev) if want_ticks else None
    end = torch.empty((npol, total_apps), dtype=tdt, device=dev) if want_ticks else None
    rec_words = 10 if f64 else 8
    stats = torch.empty((npol, n_traces, ndev, rec_words), dtype=torch.int32, device=dev)
    mem_pct = torch.empty((npol, n_traces, ndev), dtype=torch.float64, device=dev) if want_pct else None
    dev_pct = torch.empty_like(mem_pct) if want_pct else None
    speedup = torch.empty((npol, n_traces, ndev), dtype=torch.float64, device=dev) if want_speedup else None
    events = counts = None
    if events_per_trace:
        # zeroed: readers copy whole slices, of which the log fills event_counts
        events = torch.zeros((npol, n_traces, events_per_trace, 4), dtype=torch.int32, device=dev)
        counts = torch.empty((npol, n_traces), dtype=torch.int32, device=dev)

    b = _lib.SgBatch()
    b.n_traces = n_traces
    b.trace_offsets = _vp(trace_offsets)
    b.apps_per_trace = napp
    b.max_apps = int(max_apps)
    b.apps = _vp(apps)
    b.steps = _vp(steps.contiguous()) if steps is not None else None
    b.step_offsets = _vp(step_offsets.contiguous()) if step_offsets is not None else None
    b.policy_mask = mask
    b.ndev = ndev
    for i, c in enumerate(caps):
        b.cap_mib[i] = c
    b.time_mode = time_mode
    b.tick_log2 = tick_log2
    b.apps_total = total_apps
    o = _lib.SgOut()
    o.grant, o.end, o.stats = _vp(grant), _vp(end), _vp(stats)
    o.mem_pct, o.dev_pct = _vp(mem_pct), _vp(dev_pct)
    o.speedup = _vp(speedup)
    o.events, o.event_counts = _vp(events), _vp(counts)
    o.events_per_trace = events_per_trace
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = L.sg_simulate_batch(ctypes.byref(b), ctypes.byref(o), ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc, "sg_simulate_batch")
    return BatchResult(ordered, n_traces, ndev, caps, time_mode, tick_log2, grant, end, stats,
                       mem_pct, dev_pct, events, counts, speedup)


@dataclass
class HostResult:
    policies: tuple[PolicyKind, ...]
    grant: Optional[np.ndarray]   # (npol, total_apps) uint32
    end: Optional[np.ndarray]
    stats: np.ndarray             # (npol, n_traces, ndev) STATS_DTYPE
    mem_pct: Optional[np.ndarray]
    dev_pct: Optional[np.ndarray]
    speedup: Optional[np.ndarray] = None
    h2d_bytes: int = 0            # bytes the call copied host -> device
    d2h_bytes: int = 0            # bytes the call copied device -> host (sg_last_host_transfer)


class HostBuffers:
    """Pinned host output buffers for repeated simulate_batch_host calls."""

    def __init__(self, npol: int, n_traces: int, n_apps: int, ndev: int,
                 want_ticks: bool = True, want_pct: bool = True, want_speedup: bool = True):
        torch = _torch()
        pin = torch.cuda.is_available()

        def alloc(shape, dt):
            return torch.empty(shape, dtype=dt, pin_memory=pin).numpy()

        self.grant = alloc((npol, n_traces * n_apps), torch.int32).view(np.uint32) if want_ticks else None
        self.end = alloc((npol, n_traces * n_apps), torch.int32).view(np.uint32) if want_ticks else None
        self.stats = alloc((npol, n_traces, ndev, 8), torch.int32).view(STATS_DTYPE).reshape(
            npol, n_traces, ndev)
        self.mem_pct = alloc((npol, n_traces, ndev), torch.float64) if want_pct else None
        self.dev_pct = alloc((npol, n_traces, ndev), torch.float64) if want_pct else None
        self.speedup = alloc((npol, n_traces, ndev), torch.float64) if want_speedup else None

def pinned_apps(n_traces: int, n_apps: int) -> np.ndarray:
    """A pinned (page-locked) host array for T0 records, (n_traces, n_apps, 4) uint32."""
    torch = _torch()
    t = torch.empty((n_traces, n_apps, 4), dtype=torch.int32, pin_memory=torch.cuda.is_available())
    return t.numpy().view(np.uint32)


def simulate_batch_host(apps: np.ndarray, policies: Iterable = ("fifo",), cap_mib=184_320, *,
                        device: int = 0, chunk_traces: int = 0, want_ticks: bool = True,
                        want_pct: bool = True, want_speedup: bool = True,
                        out: Optional[HostBuffers] = None, tick_log2: int = 10) -> HostResult:
    """Host-buffer simulation through the C ABI pipeline (sg_simulate_batch_host).
    apps: (n_traces, n_apps, 4) uint32 (pinned memory gives full copy speed)."""
    L = _lib.lib()
    a = np.asarray(apps)
    if a.dtype.names is not None:
        a = a.view(np.uint32).reshape(a.shape + (4,))
    if a.ndim != 3 or a.shape[-1] != 4 or a.dtype.itemsize != 4:
        raise ValueError("apps must be (n_traces, n_apps, 4) 32-bit records")
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    mask, ordered = policy_mask(policies)
    caps = _caps(cap_mib)
    n_traces, napp = a.shape[0], a.shape[1]
    if out is None:
        out = HostBuffers(len(ordered), n_traces, napp, len(caps), want_ticks, want_pct, want_speedup)
    want_speedup = want_speedup and out.speedup is not None
    b = _lib.SgBatch()
    b.n_traces = n_traces
    b.apps_per_trace = napp
    b.max_apps = napp
    b.apps = ctypes.c_void_p(a.ctypes.data)
    b.policy_mask = mask
    b.ndev = len(caps)
    for i, c in enumerate(caps):
        b.cap_mib[i] = c
    b.time_mode = _lib.TIME_TICKS
    b.tick_log2 = tick_log2
    o = _lib.SgOut()

    def p(x):
        return None if x is None else ctypes.c_void_p(x.ctypes.data)

    o.grant, o.end, o.stats = p(out.grant if want_ticks else None), p(out.end if want_ticks else None), p(out.stats)
    o.mem_pct = p(out.mem_pct if want_pct else None)
    o.dev_pct = p(out.dev_pct if want_pct else None)
    o.speedup = p(out.speedup if want_speedup else None)
    rc = L.sg_simulate_batch_host(ctypes.byref(b), ctypes.byref(o), int(device), int(chunk_traces))
    _lib.check(rc, "sg_simulate_batch_host")
    h2d, d2h = ctypes.c_uint64(0), ctypes.c_uint64(0)
    L.sg_last_host_transfer(ctypes.byref(h2d), ctypes.byref(d2h))
    return HostResult(ordered, out.grant if want_ticks else None, out.end if want_ticks else None,
                      out.stats, out.mem_pct if want_pct else None, out.dev_pct if want_pct else None,
                      out.speedup if want_speedup else None, int(h2d.value), int(d2h.value))


def k1_engine(apps_per_trace: int, n_policies: int, ndev: int = 1) -> str:
    """K1 engine of a T0 simulate_batch call: "lane" (trace_sim_lane, <= 128
    apps), "lane256" (trace_sim_lane256, 129..256 apps on one device),
    "octet" (trace_sim_octet, SGPU_K1=octet) or "warp" (trace_sim).
    Mirrors the choice in sgpu_abi.cu simulate_device and the SGPU_K1
    override."""
    n_pad = 32
    while n_pad < apps_per_trace:
        n_pad *= 2
    eng = os.environ.get("SGPU_K1", "")
    if eng == "warp" or n_policies * ndev > 32:
        return "warp"
    wide_ok = n_pad == 256 and ndev == 1 and n_policies <= 4
    if eng == "octet" and wide_ok:
        return "octet"
    if eng == "lane":
        return "lane" if n_pad <= 256 else "warp"
    if wide_ok:
        return "lane256"
    lane = n_pad <= 64 or (n_pad <= 128 and n_policies * ndev >= 2)
    return "lane" if lane else "warp"


K1_KERNELS = {"lane": "trace_sim_lane_kernel", "lane256": "trace_sim_lane256_kernel",
              "octet": "trace_sim_octet_kernel", "warp": "trace_sim_kernel"}


def k1_launches(apps_per_trace: int, n_policies: int, ndev: int = 1) -> int:
    """Kernel launches of one T0 simulate_batch call: two on the lane engine
    (the main pass + the 64-bit-key retry pass, sgpu_lane.cu
    launch_sim_lane), one on the others."""
    return 2 if k1_engine(apps_per_trace, n_policies, ndev) == "lane" else 1


def reduce_stats(stats_raw, stream=None) -> dict:
    """K2: sums / maxima of integer statistics over all records of a
    BatchResult.stats_raw tensor (ticks mode).  Returns {field: int}."""
    torch = _torch()
    st = stats_raw.contiguous()
    if st.shape[-1] != 8:
        raise ValueError("reduce_stats takes ticks-mode records")
    count = st.numel() // 8
    out = torch.empty(16, dtype=torch.int64, device=st.device)
    if stream is None:
        stream = torch.cuda.current_stream(st.device)
    with torch.cuda.device(st.device):
        rc = _lib.lib().sg_reduce_stats(_vp(st), count, _vp(out), ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc, "sg_reduce_stats")
    return out


def aggr_to_dict(aggr) -> dict:
    v = aggr.cpu().numpy().view(np.uint64) if hasattr(aggr, "cpu") else np.asarray(aggr, np.uint64)
    return {k: int(x) for k, x in zip(_lib.AGGR_FIELDS, v) if not k.startswith("reserved")}


def generate_traces(gen, trace_begin: int, n_traces: int, device=None, out=None, stream=None):
    """K3 on the GPU: (n_traces, apps_per_trace, 4) int32 CUDA tensor,
    bit-identical to tracegen.generate(gen, trace_begin, n_traces)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if out is None:
        out = torch.empty((n_traces, gen.apps_per_trace, 4), dtype=torch.int32, device=dev)
    p = _lib.SgGenParams()
    for name, _ in _lib.SgGenParams._fields_:
        setattr(p, name, int(getattr(gen, name)))
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().sg_generate_traces(ctypes.byref(p), int(trace_begin), int(n_traces),
                                           _vp(out), ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc, "sg_generate_traces")
    return out


def pct_host(stats: np.ndarray, cap_mib, tick_log2: int = 10):
    """(makespan_ms, avg_mem_util_pct, avg_device_util_pct) from ticks-mode
    records with the reference's float operation order (harness.py:378,427,437).
    Host-side formatting of GPU results (used to rebuild MetricsReports)."""
    T = stats["makespan"].astype(np.float64)
    scale = 2.0 ** -tick_log2
    makespan_s = np.where(stats["makespan"] > 0, T * scale, 1e-9)
    cap_bytes = np.asarray(cap_mib, dtype=np.float64) * float(1 << 20)
    zero_span = (stats["status"] & _lib.ST_ZERO_SPAN_LEVEL) != 0
    integral = np.where(zero_span,
                        stats["mem_integral"].astype(np.float64) * float(1 << 20) * 1e-9,
                        stats["mem_integral"].astype(np.float64) * (float(1 << 20) * scale))
    mem_pct = (100.0 * integral) / (cap_bytes * makespan_s)
    dev_pct = (100.0 * (stats["busy"].astype(np.float64) * scale)) / makespan_s
    empty = stats["pops"] == 0
    mem_pct = np.where(empty, 0.0, mem_pct)
    dev_pct = np.where(empty, 0.0, dev_pct)
    ms = np.where(empty, 0.0, makespan_s * 1000.0)
    return ms, mem_pct, dev_pct


__all__ = ["BatchResult", "HostResult", "HostBuffers", "STATS_DTYPE", "STATS_F64_DTYPE",
           "STEP_DTYPE", "EVENT_DTYPE", "simulate_batch", "simulate_batch_host",
           "reduce_stats", "aggr_to_dict", "generate_traces", "pinned_apps", "pct_host"]
