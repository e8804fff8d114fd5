"""ctypes wrapper of the CPU oracle (oracle/sim_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the checker.  The product package never
imports it.  Builds oracle/_build/liboracle.so on demand with make/gcc.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

STATS_DTYPE = np.dtype([("makespan", "<u4"), ("busy", "<u4"), ("mem_integral", "<u8"),
                        ("grants", "<u4"), ("pops", "<u4"), ("max_holders", "<u2"),
                        ("unfinished", "<u2"), ("status", "<u4")])
assert STATS_DTYPE.itemsize == 32
STEP_DTYPE = np.dtype([("op", "<u4"), ("mib", "<u4"), ("dur", "<u8")])
EVENT_DTYPE = np.dtype([("t", "<u8"), ("app", "<u2"), ("kind", "u1"), ("dev", "u1"),
                        ("mib", "<u4")])
POLICY_CODES = {"fifo": 0, "mmu": 1, "pfifo": 2, "pmmu": 3}

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "sim_oracle.c"))):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.orc_select_grants.argtypes = [ctypes.c_uint32, P, P, ctypes.c_int64,
                                        ctypes.c_uint32, P]
        L.orc_select_grants.restype = ctypes.c_int
        L.orc_simulate_trace.argtypes = [ctypes.c_uint32, P, P, P, ctypes.c_uint32, P,
                                         ctypes.c_uint32, P, P, P, P, ctypes.c_uint32, P]
        L.orc_simulate_trace.restype = ctypes.c_int
        L.orc_simulate_burst_batch.argtypes = [ctypes.c_uint64, ctypes.c_uint32, P,
                                               ctypes.c_uint32, P, ctypes.c_uint32,
                                               P, P, P, ctypes.c_int]
        L.orc_simulate_burst_batch.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _policy_code(policy) -> int:
    if isinstance(policy, int):
        return policy
    return POLICY_CODES[str(getattr(policy, "value", policy)).lower()]


def select_grants(nbytes, prio, free: int, policy) -> np.ndarray:
    """Granted mask of one queue (memshare/policy.py:52-74)."""
    nb = np.ascontiguousarray(nbytes, dtype=np.int64)
    pr = np.ascontiguousarray(prio, dtype=np.int32)
    g = np.zeros(len(nb), dtype=np.uint8)
    lib().orc_select_grants(len(nb), _ptr(nb), _ptr(pr), int(free), _policy_code(policy),
                            _ptr(g))
    return g.astype(bool)


def simulate_burst(apps: np.ndarray, cap_mib, policy, threads: int = 0):
    """apps: (n_traces, n) structured APP_DTYPE (or (..., 4) uint32).
    Returns (grant (n_traces, n) u32, end, stats (n_traces, ndev) STATS_DTYPE)."""
    a = np.ascontiguousarray(apps)
    if a.dtype != np.uint32:
        a = a.view(np.uint32).reshape(a.shape + (4,))
    n_traces, n = a.shape[0], a.shape[1]
    caps = np.ascontiguousarray(np.atleast_1d(np.asarray(cap_mib, dtype=np.uint32)))
    ndev = len(caps)
    grant = np.empty((n_traces, n), dtype=np.uint32)
    end = np.empty((n_traces, n), dtype=np.uint32)
    stats = np.empty((n_traces, ndev), dtype=STATS_DTYPE)
    rc = lib().orc_simulate_burst_batch(n_traces, n, _ptr(a), ndev, _ptr(caps),
                                        _policy_code(policy), _ptr(grant), _ptr(end),
                                        _ptr(stats), int(threads))
    if rc:
        raise RuntimeError(f"oracle simulate_burst failed ({rc})")
    return grant, end, stats


def simulate_program(steps: np.ndarray, step_offsets: np.ndarray, attr: np.ndarray,
                     cap_mib, policy, events: bool = False):
    """One trace in step-program mode (ticks).  steps: STEP_DTYPE array;
    step_offsets: n+1 (relative).  Returns grant, end, stats[ndev] and, with
    events=True, the emission-order event log."""
    st = np.ascontiguousarray(steps, dtype=STEP_DTYPE)
    so = np.ascontiguousarray(step_offsets, dtype=np.uint32)
    at = np.ascontiguousarray(attr, dtype=np.uint32)
    n = len(at)
    caps = np.ascontiguousarray(np.atleast_1d(np.asarray(cap_mib, dtype=np.uint32)))
    grant = np.empty(n, dtype=np.uint32)
    end = np.empty(n, dtype=np.uint32)
    stats = np.empty(len(caps), dtype=STATS_DTYPE)
    ev_cap = 8 * int(len(st)) + 8 * n + 16
    ev = np.empty(ev_cap, dtype=EVENT_DTYPE) if events else None
    cnt = np.zeros(1, dtype=np.uint32)
    rc = lib().orc_simulate_trace(n, _ptr(st), _ptr(so), _ptr(at), len(caps), _ptr(caps),
                                  _policy_code(policy), _ptr(grant), _ptr(end), _ptr(stats),
                                  _ptr(ev), ev_cap, _ptr(cnt))
    if rc:
        raise RuntimeError(f"oracle simulate_trace failed ({rc})")
    if events:
        return grant, end, stats, ev[:int(cnt[0])].copy()
    return grant, end, stats


def pct_from_stats(stats: np.ndarray, cap_mib, tick_log2: int = 10):
    """avg_mem_util_pct / avg_device_util_pct / makespan_ms from the integer
    forms with the reference's float operation order (harness.py:378, 427, 437)."""
    T = stats["makespan"].astype(np.float64)
    scale = 2.0 ** -tick_log2
    makespan_s = np.where(stats["makespan"] > 0, T * scale, 1e-9)
    cap_bytes = np.asarray(cap_mib, dtype=np.float64) * float(1 << 20)
    integral = stats["mem_integral"].astype(np.float64) * (float(1 << 20) * scale)
    zero_span = (stats["status"] & 0x10) != 0
    integral = np.where(zero_span, stats["mem_integral"].astype(np.float64) * float(1 << 20)
                        * 1e-9, integral)
    mem_pct = (100.0 * integral) / (cap_bytes * makespan_s)
    busy_s = stats["busy"].astype(np.float64) * scale
    dev_pct = (100.0 * busy_s) / makespan_s
    return makespan_s * 1000.0, mem_pct, dev_pct


def seq_ticks(apps: np.ndarray, ndev: int = 1) -> np.ndarray:
    """Sequential makespan in ticks per (trace, device) of T0 traces:
    sum of arrival + busy over the device's apps (AppProfile.total_ms() of
    [Phase(cpu_ms=a), Phase(alloc, busy_ms=b, free)], harness.py:61-62).
    Devices out of range count as device 0."""
    a = np.ascontiguousarray(apps)
    if a.dtype != np.uint32:
        a = a.view(np.uint32).reshape(a.shape + (4,))
    per_app = a[..., 0].astype(np.uint64) + a[..., 2].astype(np.uint64)
    if ndev == 1:
        return per_app.sum(axis=1, dtype=np.uint64)[:, None]
    dev = (a[..., 3] >> 8) & 0xFF
    dev = np.where(dev < ndev, dev, 0)
    return np.stack([np.where(dev == d, per_app, 0).sum(axis=1, dtype=np.uint64)
                     for d in range(ndev)], axis=1)


def speedup_from(seq: np.ndarray, makespan: np.ndarray, napps: np.ndarray,
                 tick_log2: int = 10) -> np.ndarray:
    """Speed-up vs sequential, the reference's float order with cpu/busy ms =
    ticks and time_scale = 1000 * 2^-tick_log2 (pkg/tests/test_harness.py:
    119-126): (S * time_scale) / (max(T * 2^-tick_log2, 1e-9) * 1000.0);
    NaN for an empty (sub-)trace."""
    scale = 2.0 ** -tick_log2
    seq_ms = np.asarray(seq, dtype=np.uint64).astype(np.float64) * (1000.0 * scale)
    T = np.asarray(makespan)
    span = np.where(T > 0, T.astype(np.float64) * scale, 1e-9)
    with np.errstate(invalid="ignore", divide="ignore"):
        sp = seq_ms / (span * 1000.0)
    return np.where(np.asarray(napps) > 0, sp, np.nan)
