"""ctypes binding of libsgpu.so (include/sgpu.h).

The product has no CPU fallback: if the shared library is missing, cannot
be loaded, or its ABI version differs, every entry point raises
`SgpuUnavailable`.  Build it with `python -m paper_1712_04495_b200.build`
(or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import SgpuError, SgpuUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
# SGPU_LIB: developer override (A/B builds of the same ABI); default in-tree
LIB_PATH = os.environ.get("SGPU_LIB") or os.path.join(HERE, "libsgpu.so")
ABI_VERSION = 2
MAX_APPS = 1024
MAX_DEV = 8

POLICY_FIFO, POLICY_MMU, POLICY_PFIFO, POLICY_PMMU = 0, 1, 2, 3
OP_CPU, OP_ALLOC, OP_BUSY, OP_FREE = 0, 1, 2, 3
TIME_TICKS, TIME_F64 = 0, 1
EV_START, EV_REQUEST, EV_GRANT, EV_ALLOC, EV_BUSY_START, EV_BUSY_END, EV_FREE, EV_END = range(8)
EVENT_NAMES = ("start", "request", "grant", "alloc", "busy_start", "busy_end", "free", "end")

ST_TICK_OVERFLOW = 0x1
ST_COUNTER_OVERFLOW = 0x2
ST_BAD_DEVICE = 0x4
ST_EVENT_OVERFLOW = 0x8
ST_ZERO_SPAN_LEVEL = 0x10
NEVER = 0xFFFFFFFF

EXPORTS = ("sg_abi_version", "sg_last_error", "sg_device_info", "sg_simulate_batch",
           "sg_simulate_batch_host", "sg_simulate_small_host", "sg_reduce_stats",
           "sg_generate_traces", "sg_select_grants_batch", "sg_last_host_transfer")

P = ctypes.c_void_p
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64


class SgBatch(ctypes.Structure):
    _fields_ = [("n_traces", U64), ("trace_offsets", P), ("apps_per_trace", U32),
                ("max_apps", U32), ("apps", P), ("steps", P), ("step_offsets", P),
                ("policy_mask", U32), ("ndev", U32), ("cap_mib", U32 * MAX_DEV),
                ("time_mode", U32), ("tick_log2", ctypes.c_int32), ("apps_total", U64)]


class SgOut(ctypes.Structure):
    _fields_ = [("grant", P), ("end", P), ("stats", P), ("mem_pct", P), ("dev_pct", P),
                ("events", P), ("event_counts", P), ("events_per_trace", U32),
                ("reserved", U32), ("speedup", P)]


class SgGenParams(ctypes.Structure):
    _fields_ = [("seed", U64), ("apps_per_trace", U32), ("arrival_kind", U32),
                ("arr_lo", U32), ("arr_hi", U32), ("mem_lo", U32), ("mem_hi", U32),
                ("busy_lo", U32), ("busy_hi", U32), ("prio_kind", U32),
                ("prio_levels", U32), ("ndev", U32)]


AGGR_FIELDS = ("records", "sum_makespan", "sum_busy", "sum_mem_integral", "sum_grants",
               "sum_pops", "sum_unfinished", "sum_max_holders", "stuck_records",
               "error_records", "reserved_sum0", "reserved_sum1", "max_makespan",
               "max_holders", "status_or", "reserved_max0")
AGGR_NSUM = 12

_lock = threading.Lock()
_lib = None


def _load():
    if not os.path.exists(LIB_PATH):
        raise SgpuUnavailable(
            f"{LIB_PATH} is missing: build it with `python -m paper_1712_04495_b200.build` "
            "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise SgpuUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name in EXPORTS:
        if not hasattr(L, name):
            raise SgpuUnavailable(f"{LIB_PATH} does not export {name}")
    L.sg_abi_version.restype = ctypes.c_int
    L.sg_last_error.restype = ctypes.c_char_p
    L.sg_device_info.argtypes = [ctypes.c_int, P, P]
    L.sg_simulate_batch.argtypes = [ctypes.POINTER(SgBatch), ctypes.POINTER(SgOut), P]
    L.sg_simulate_batch_host.argtypes = [ctypes.POINTER(SgBatch), ctypes.POINTER(SgOut),
                                         ctypes.c_int, U64]
    L.sg_simulate_small_host.argtypes = [ctypes.POINTER(SgBatch), ctypes.POINTER(SgOut), ctypes.c_int]
    L.sg_reduce_stats.argtypes = [P, U64, P, P]
    L.sg_generate_traces.argtypes = [ctypes.POINTER(SgGenParams), U64, U64, P, P]
    L.sg_select_grants_batch.argtypes = [U64, P, P, P, P, P, P, P]
    L.sg_last_host_transfer.argtypes = [P, P]
    for name in EXPORTS[2:-1]:
        getattr(L, name).restype = ctypes.c_int
    L.sg_last_host_transfer.restype = None
    v = L.sg_abi_version()
    if v != ABI_VERSION:
        raise SgpuUnavailable(f"libsgpu ABI version {v} != expected {ABI_VERSION}")
    return L


def lib():
    """The loaded library (raises SgpuUnavailable when it cannot be used)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = _load()
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().sg_last_error().decode(errors="replace")
        raise SgpuError(f"{what} failed ({rc}): {msg}")


def loaded_path() -> str:
    lib()
    return LIB_PATH
