"""The oracle (oracle/sim_oracle.c) pinned against the reference's golden
vectors (tests/golden/, produced by the real memshare simulator).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from util import GOLDEN, POLICIES, floats_equal, golden


@pytest.mark.parametrize("cname", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("pol", POLICIES)
def test_oracle_matches_reference_burst(cname, pol):
    z = golden("ref_burst.npz")
    apps = z[f"{cname}_apps"]
    cap = int(z[f"{cname}_cap"][0])
    g, e, st = O.simulate_burst(apps, (cap,), pol)
    np.testing.assert_array_equal(g, z[f"{cname}_{pol}_grant"])
    np.testing.assert_array_equal(e, z[f"{cname}_{pol}_end"])
    np.testing.assert_array_equal(st[:, 0]["makespan"], z[f"{cname}_{pol}_T"])
    ms, mp, dp = O.pct_from_stats(st[:, 0], cap)
    fl = z[f"{cname}_{pol}_floats"]
    assert floats_equal(ms, fl[:, 0])
    assert floats_equal(mp, fl[:, 1])
    assert floats_equal(dp, fl[:, 2])
    ints = z[f"{cname}_{pol}_ints"]
    np.testing.assert_array_equal(st[:, 0]["max_holders"], ints[:, 0])
    np.testing.assert_array_equal(st[:, 0]["grants"], ints[:, 1])
    np.testing.assert_array_equal(st[:, 0]["unfinished"], ints[:, 2])


@pytest.mark.parametrize("pol", POLICIES)
def test_oracle_multidev_decomposition(pol):
    """The per-device extension equals simulate() on each device's sub-trace."""
    z = golden("ref_multidev.npz")
    apps = z["apps"]
    caps = tuple(int(c) for c in z["cap"])
    g, e, st = O.simulate_burst(apps, caps, pol)
    np.testing.assert_array_equal(g, z[f"{pol}_grant"])
    np.testing.assert_array_equal(e, z[f"{pol}_end"])
    np.testing.assert_array_equal(st["makespan"], z[f"{pol}_T"])
    fl = z[f"{pol}_floats"]
    for d in range(len(caps)):
        _, mp, dp = O.pct_from_stats(st[:, d], caps[d])
        assert floats_equal(mp, fl[:, d, 1])
        assert floats_equal(dp, fl[:, d, 2])
    ints = z[f"{pol}_ints"]
    np.testing.assert_array_equal(st["max_holders"], ints[..., 0])
    np.testing.assert_array_equal(st["grants"], ints[..., 1])


def test_oracle_select_grants_golden():
    z = golden("ref_select.npz")
    off = z["offsets"]
    got = []
    for q in range(len(off) - 1):
        sl = slice(off[q], off[q + 1])
        got.append(O.select_grants(z["nbytes"][sl], z["prio"][sl], int(z["free"][q]),
                                   int(z["kind"][q])).astype(np.uint8))
    np.testing.assert_array_equal(np.concatenate(got), z["granted"])


def _dyadic_records():
    with open(os.path.join(GOLDEN, "ref_reports.json")) as f:
        recs = json.load(f)
    return [r for r in recs if r["spec"]["from_json"] is None]


def _encode_ticks(rec):
    """Reference spec (fixture) -> oracle step program in ticks, when the
    durations lie on a dyadic grid (the same rule as harness.encode_spec)."""
    from fractions import Fraction
    sp = rec["spec"]
    ts = float.fromhex(sp["time_scale"])
    progs, durs = [], []
    for inst in sp["instances"]:
        flat = []
        for cpu, alloc, busy, free in inst["phases"]:
            if cpu:
                flat.append((0, 0, cpu * ts / 1000.0))
            if alloc:
                flat.append((1, alloc, 0.0))
            if busy:
                flat.append((2, 0, busy * ts / 1000.0))
            if free:
                flat.append((3, free, 0.0))
        progs.append(flat)
        durs += [d for op, _, d in flat if op in (0, 2)]
    e = max([Fraction(d).denominator.bit_length() - 1 for d in durs] or [0])
    if e > 40:
        return None
    rows, offs = [], [0]
    for flat in progs:
        for op, mib, d in flat:
            rows.append((op, mib, int(Fraction(d) * (1 << e))))
        offs.append(len(rows))
    prios = sorted({i["priority"] for i in sp["instances"]})
    attr = [prios.index(i["priority"]) for i in sp["instances"]]
    steps = np.array(rows, dtype=O.STEP_DTYPE) if rows else np.zeros(1, O.STEP_DTYPE)
    return steps, np.array(offs, np.uint32), np.array(attr, np.uint32), e


@pytest.mark.parametrize("rec", _dyadic_records(), ids=lambda r: r["name"])
def test_oracle_program_mode_reports(rec):
    enc = _encode_ticks(rec)
    if enc is None:
        pytest.skip("non-dyadic time scale (float mode is checked on the GPU)")
    steps, offs, attr, e = enc
    cap = rec["spec"]["device_mib"][0]
    g, en, st, ev = O.simulate_program(steps, offs, attr, (cap,), rec["spec"]["policy"],
                                       events=True)
    ms, mp, dp = O.pct_from_stats(st, cap, tick_log2=e)
    assert ms[0] == float.fromhex(rec["makespan_ms"])
    assert mp[0] == float.fromhex(rec["avg_mem_util_pct"])
    assert dp[0] == float.fromhex(rec["avg_device_util_pct"])
    assert st[0]["max_holders"] == rec["max_concurrent_holders"]
    # the emission-order log, stably sorted, is the reference's event list
    order = np.argsort(ev["t"], kind="stable")
    names = ("start", "request", "grant", "alloc", "busy_start", "busy_end", "free", "end")
    got = [[float.hex((int(ev["t"][i]) / (1 << e)) * 1000.0), int(ev["app"][i]),
            names[ev["kind"][i]], 0,
            int(ev["mib"][i]) << 20 if ev["kind"][i] in (1, 2, 3, 6) else 0] for i in order]
    assert got == rec["events"]
