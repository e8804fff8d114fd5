"""Synthetic trace generator and the benchmark configurations.

Integer-only, counter-based: every field of every app is a pure function of
(seed, trace_id, app_id, field) through SplitMix64 finalisers, so any trace
range can be generated independently (per-GPU shards, CPU baselines, tests)
and the CUDA twin (`sg_generate_traces`, csrc/sgpu_gen.cu) is bit-identical.

Configurations follow SURVEY.md §8(d) / BASELINE.json `configs`:

  C1  1 trace x 8 apps, FIFO, 4799 MiB    README burst (README.md:103-104)
  C2  1M x 64 apps, all four policies      arrival U[0,4096), mem U[1024,46080] MiB,
                                           busy U[1,2048], prio U{0..3}
  C3  1M x 256 apps, pfifo + pmmu          skewed 8:4:2:1 priorities, cubic arrivals
  C4  4M x 128 apps, all four policies     mem U[46080,184320] (1/4..1x capacity)
  C5  16M x 64 apps over 8 simulated devices per trace, device = app mod 8
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

ARR_UNIFORM, ARR_CUBIC = 0, 1
PRIO_UNIFORM, PRIO_SKEWED = 0, 1

FIELD_ARRIVAL, FIELD_MEM, FIELD_BUSY, FIELD_PRIO = 0, 1, 2, 3

CAP_180G_MIB = 184_320
CAP_K20M_MIB = 4_799


def mix64_int(z: int) -> int:
    """SplitMix64 finaliser on a Python int (reference scalar form)."""
    z = (z + GOLDEN) & _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


@dataclass(frozen=True)
class GenParams:
    """Mirror of `sg_gen_params` (include/sgpu.h)."""
    seed: int = 1
    apps_per_trace: int = 64
    arrival_kind: int = ARR_UNIFORM
    arr_lo: int = 0
    arr_hi: int = 4095
    mem_lo: int = 1024
    mem_hi: int = 46080
    busy_lo: int = 1
    busy_hi: int = 2048
    prio_kind: int = PRIO_UNIFORM
    prio_levels: int = 4
    ndev: int = 1


@dataclass(frozen=True)
class BenchConfig:
    name: str
    n_traces: int
    gen: GenParams
    policies: tuple[str, ...]
    cap_mib: tuple[int, ...]
    description: str = ""
    gpus: int = 1

    @property
    def ndev(self) -> int:
        return len(self.cap_mib)

    def with_traces(self, n: int) -> "BenchConfig":
        return replace(self, n_traces=n)


ALL_POLICIES = ("fifo", "mmu", "pfifo", "pmmu")

CONFIGS: dict[str, BenchConfig] = {
    "C1": BenchConfig(
        "C1", 1,
        GenParams(seed=1, apps_per_trace=8, arr_lo=900, arr_hi=900, mem_lo=700,
                  mem_hi=700, busy_lo=100, busy_hi=100, prio_levels=1),
        ("fifo",), (CAP_K20M_MIB,),
        "single trace of 8 burst apps (cpu 900, alloc 700, busy 100) on 4799 MiB, FIFO"),
    "C2": BenchConfig(
        "C2", 1 << 20, GenParams(seed=1, apps_per_trace=64),
        ALL_POLICIES, (CAP_180G_MIB,),
        "1M traces x 64 apps, all four policies, 180 GiB device"),
    "C3": BenchConfig(
        "C3", 1 << 20,
        GenParams(seed=1, apps_per_trace=256, arrival_kind=ARR_CUBIC, arr_lo=0,
                  arr_hi=16383, prio_kind=PRIO_SKEWED),
        ("pfifo", "pmmu"), (CAP_180G_MIB,),
        "1M traces x 256 apps, skewed 8:4:2:1 priorities, cubic (bursty) arrivals"),
    "C4": BenchConfig(
        "C4", 4 << 20,
        GenParams(seed=1, apps_per_trace=128, arr_lo=0, arr_hi=8191, mem_lo=46080,
                  mem_hi=184320),
        ALL_POLICIES, (CAP_180G_MIB,),
        "4M traces x 128 apps, requests 1/4..1x of the 180 GiB budget"),
    "C5": BenchConfig(
        "C5", 16 << 20, GenParams(seed=1, apps_per_trace=64, ndev=8),
        ALL_POLICIES, (CAP_180G_MIB,) * 8,
        "16M traces x 64 apps over 8 simulated devices per trace (device = app mod 8)",
        gpus=8),
}

APP_DTYPE = np.dtype([("arrival", "<u4"), ("mem_mib", "<u4"), ("busy", "<u4"),
                      ("attr", "<u4")])


def trace_keys(seed: int, trace_ids: np.ndarray) -> np.ndarray:
    k0 = np.uint64(mix64_int(seed & _MASK))
    return _mix64(k0 ^ trace_ids.astype(np.uint64))


def _uniform(h: np.ndarray, lo: int, hi: int) -> np.ndarray:
    span = np.uint64(hi - lo + 1)
    return (np.uint64(lo) + (((h >> np.uint64(32)) * span) >> np.uint64(32))).astype(np.uint32)


def generate(p: GenParams, trace_begin: int, n_traces: int) -> np.ndarray:
    """Apps of traces [trace_begin, trace_begin + n_traces) as a structured
    array of shape (n_traces, apps_per_trace) with dtype APP_DTYPE (16 B/app,
    the T0 layout of sg_app)."""
    n = p.apps_per_trace
    if not (1 <= p.prio_levels <= 8):
        raise ValueError("prio_levels must be 1..8")
    if p.ndev < 1 or p.ndev > 8:
        raise ValueError("ndev must be 1..8")
    tids = np.arange(trace_begin, trace_begin + n_traces, dtype=np.uint64)
    kt = trace_keys(p.seed, tids)[:, None]
    app = np.arange(n, dtype=np.uint64)[None, :]

    def h(fld: int) -> np.ndarray:
        return _mix64(kt ^ ((app << np.uint64(3)) | np.uint64(fld)))

    out = np.empty((n_traces, n), dtype=APP_DTYPE)
    ha = h(FIELD_ARRIVAL)
    if p.arrival_kind == ARR_UNIFORM:
        out["arrival"] = _uniform(ha, p.arr_lo, p.arr_hi)
    elif p.arrival_kind == ARR_CUBIC:
        u = ha >> np.uint64(40)
        c = (((u * u) >> np.uint64(24)) * u) >> np.uint64(24)
        span = np.uint64(p.arr_hi - p.arr_lo + 1)
        out["arrival"] = (np.uint64(p.arr_lo) + ((c * span) >> np.uint64(24))).astype(np.uint32)
    else:
        raise ValueError(f"unknown arrival_kind {p.arrival_kind}")
    out["mem_mib"] = _uniform(h(FIELD_MEM), p.mem_lo, p.mem_hi)
    out["busy"] = _uniform(h(FIELD_BUSY), p.busy_lo, p.busy_hi)
    hp = h(FIELD_PRIO) >> np.uint64(32)
    levels = p.prio_levels
    if p.prio_kind == PRIO_UNIFORM:
        prio = ((hp * np.uint64(levels)) >> np.uint64(32)).astype(np.uint32)
    elif p.prio_kind == PRIO_SKEWED:
        total = (1 << levels) - 1
        r = ((hp * np.uint64(total)) >> np.uint64(32)).astype(np.int64)
        prio = np.zeros(r.shape, dtype=np.uint32)
        cum = 0
        for k in range(levels):
            cum += 1 << (levels - 1 - k)
            prio += (r >= cum).astype(np.uint32)
    else:
        raise ValueError(f"unknown prio_kind {p.prio_kind}")
    dev = (np.arange(n, dtype=np.uint32) % np.uint32(p.ndev))[None, :]
    out["attr"] = prio | (dev << np.uint32(8))
    return out


def as_u32x4(apps: np.ndarray) -> np.ndarray:
    """View a structured APP_DTYPE array as (..., 4) uint32."""
    return apps.view(np.uint32).reshape(apps.shape + (4,))


__all__ = ["APP_DTYPE", "BenchConfig", "CONFIGS", "GenParams", "ALL_POLICIES",
           "generate", "as_u32x4", "mix64_int", "CAP_180G_MIB", "CAP_K20M_MIB"]
