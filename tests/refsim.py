"""Run the REAL reference simulator (memshare.harness.simulate) on T0 traces.

Only usable where /root/reference exists (this build container): the golden
fixtures in tests/golden/ are produced through this module by
tests/golden/make_golden.py and committed, so the GPU box never needs the
reference tree.  The reference module is imported read-only; raw event times
are captured by wrapping the module-level `_metrics_from_events` it calls
(memshare/harness.py:568) — the reference code itself is not modified.
"""

from __future__ import annotations

import os
import sys

REF_SRC = os.environ.get("MEMSHARE_REF_SRC", "/root/reference/pkg/src")
TIME_SCALE_DYADIC = 1000.0 / 1024.0   # SURVEY.md §8 "Ticks": t = ticks / 1024 s exactly

KIND_CODES = {"start": 0, "request": 1, "grant": 2, "alloc": 3, "busy_start": 4,
              "busy_end": 5, "free": 6, "end": 7}


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "memshare"))


def ref_modules():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import memshare.device as device
    import memshare.harness as harness
    import memshare.policy as policy
    return harness, policy, device


def burst_profiles(apps_row):
    """T0 apps -> reference AppProfiles."""
    harness, _, _ = ref_modules()
    profs = []
    for i, (a, m, b, attr) in enumerate(apps_row):
        profs.append(harness.AppProfile(
            f"app{i}",
            [harness.Phase(cpu_ms=int(a)),
             harness.Phase(alloc_mib=int(m), busy_ms=int(b), free_mib=int(m))],
            priority=int(attr) & 0xFF))
    return profs


def run_spec(spec):
    """simulate(spec) returning (report, raw_events) where raw_events are the
    reference's own event dicts with float-seconds `t`, before sorting."""
    harness, _, _ = ref_modules()
    captured = {}
    orig = harness._metrics_from_events

    def wrapper(events, capacity):
        captured["events"] = [dict(e) for e in events]
        captured["capacity"] = capacity
        return orig(events, capacity)

    harness._metrics_from_events = wrapper
    try:
        report = harness.simulate(spec)
    finally:
        harness._metrics_from_events = orig
    return report, captured.get("events", [])


def run_burst(apps_row, cap_mib: int, policy: str, tick_log2: int = 10):
    """One T0 trace through the reference.  Returns a dict of exact values:
    per-app first-grant / end ticks (None if never), T ticks, the report's
    floats and max holders."""
    harness, pol, device = ref_modules()
    assert tick_log2 == 10
    spec = harness.WorkloadSpec(
        instances=burst_profiles(apps_row), policy=pol.PolicyKind.parse(policy),
        devices=device.parse_device_config({"devices": [{"mib": int(cap_mib)}]}),
        time_scale=TIME_SCALE_DYADIC)
    report, events = run_spec(spec)
    out = summarize(report, events, len(apps_row))
    out["speedup"] = speedup_of(spec, report)
    return out


def speedup_of(spec, report) -> float:
    """The reference's speed-up vs sequential execution: sequential makespan
    = sum(AppProfile.total_ms()) * time_scale (harness.py:61-62), as in
    pkg/tests/test_harness.py:119-126 (120_000 / makespan_ms for 12 x 10 s).
    NaN where the reference would divide 0.0 by 0.0 (no events)."""
    seq = sum(p.total_ms() for p in spec.instances) * spec.time_scale
    if report.makespan_ms == 0.0:
        return float("nan")
    return seq / report.makespan_ms


def to_ticks(t: float, tick_log2: int = 10) -> int:
    v = t * (1 << tick_log2)
    iv = int(v)
    assert iv == v, f"event time {t!r} is not on the 2^-{tick_log2} s grid"
    return iv


def summarize(report, events, n: int, tick_log2: int = 10):
    grant = [None] * n
    end = [None] * n
    for e in events:   # sorted by t (stable), harness.py:567
        if e["event"] == "grant" and grant[e["instance"]] is None:
            grant[e["instance"]] = to_ticks(e["t"], tick_log2)
        if e["event"] == "end":
            end[e["instance"]] = to_ticks(e["t"], tick_log2)
    T = max((to_ticks(e["t"], tick_log2) for e in events), default=0)
    return {
        "grant": grant, "end": end, "T": T,
        "makespan_ms": report.makespan_ms,
        "mem_pct": report.avg_mem_util_pct,
        "dev_pct": report.avg_device_util_pct,
        "max_holders": report.max_concurrent_holders,
        "unfinished": sum(1 for x in end if x is None),
        "grants": sum(1 for e in events if e["event"] == "grant"),
        "n_events": len(events),
    }
