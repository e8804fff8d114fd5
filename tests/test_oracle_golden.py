"""The oracle (oracle/sim_oracle.c) pinned against the reference's golden
vectors (tests/golden/, produced by the real memshare simulator).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate
from util import GOLDEN, POLICIES, brute_select, criterion5_flags, criterion5_queues, floats_equal, golden


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


def test_speedup_restatement_matches_reference():
    """Speed-up vs sequential (pkg/tests/test_harness.py:119-126): the
    oracle's restatement from sequential ticks and makespan equals the value
    the reference computes from its own report, bit for bit (the GPU kernels
    implement the same expression, sgpu_tracesim.cuh speedup_ticks)."""
    z = golden("ref_burst.npz")
    for cname in ("C1", "C2", "C3", "C4"):
        apps = z[f"{cname}_apps"]
        S = O.seq_ticks(apps)[:, 0]
        for pol in POLICIES:
            sp = O.speedup_from(S, z[f"{cname}_{pol}_T"], np.full(len(apps), apps.shape[1]))
            assert floats_equal(sp, z[f"{cname}_{pol}_speedup"]), (cname, pol)
    z = golden("ref_multidev.npz")
    apps = z["apps"]
    nd = len(z["cap"])
    dev = (apps[..., 3] >> 8) & 0xFF
    cnt = np.stack([(dev == d).sum(axis=1) for d in range(nd)], axis=1)
    for pol in POLICIES:
        sp = O.speedup_from(O.seq_ticks(apps, nd), z[f"{pol}_T"], cnt)
        assert floats_equal(sp, z[f"{pol}_speedup"]), pol


def test_oracle_flags_bad_device():
    """ndev > 1: an app whose device index is out of range is simulated on
    device 0 and flags every record of its trace (SG_ST_BAD_DEVICE)."""
    apps = as_u32x4(generate(CONFIGS["C5"].gen, 0, 4)).copy()
    apps[1, 3, 3] = (apps[1, 3, 3] & 0xFF) | (9 << 8)
    caps = CONFIGS["C5"].cap_mib
    _, _, st = O.simulate_burst(apps, caps, "fifo")
    assert np.all(st[1]["status"] & 0x4)
    assert not np.any(st[[0, 2, 3]]["status"] & 0x4)
    moved = apps.copy()
    moved[1, 3, 3] &= 0xFF   # the same app on device 0: same schedule, no flag
    g0, e0, s0 = O.simulate_burst(moved, caps, "fifo")
    g1, e1, s1 = O.simulate_burst(apps, caps, "fifo")
    np.testing.assert_array_equal(g0, g1)
    np.testing.assert_array_equal(e0, e1)
    np.testing.assert_array_equal(s0["makespan"], s1["makespan"])


def test_criterion5_oracle_and_brute_force():
    """Acceptance criterion 5 (test_acceptance.py:174-226): the reference's
    select_grants on its 100k random queues x 4 policies (fixture) equals the
    oracle's restatement everywhere and the test's brute-force oracle on a
    sample."""
    queues = criterion5_queues()
    flags = criterion5_flags()
    k = 0
    for qi, (sizes, prios, free) in enumerate(queues):
        n = len(sizes)
        for code in range(4):
            want = flags[k:k + n]
            k += n
            got = O.select_grants(sizes, prios, free, code)
            assert np.array_equal(got, want), (qi, code)
            if qi % 50 == 0:
                b = np.zeros(n, bool)
                b[brute_select(sizes, prios, free, code)] = True
                assert np.array_equal(b, want), (qi, code)
    assert k == len(flags)
