"""GPU drop-in parity: `paper_1712_04495_b200.simulate(spec)` against full
MetricsReports of the REAL reference (tests/golden/ref_reports.json) — the
reference's own simulator test scenarios (test_harness.py:86-142,
test_acceptance.py:229-246), README examples, edge shapes and random
multi-phase programs, at dyadic and non-dyadic time scales.  Every float is
compared bit-exactly (events, memory trace, percentages, makespan)."""

import json
import os

import pytest

import paper_1712_04495_b200 as S
from util import GOLDEN

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "ref_reports.json")) as f:
    RECORDS = json.load(f)


def build_spec(rec):
    sp = rec["spec"]
    if sp["from_json"] is not None:
        return S.WorkloadSpec.from_json(sp["from_json"])
    insts = [S.AppProfile(i["name"], [S.Phase(*ph) for ph in i["phases"]], i["priority"])
             for i in sp["instances"]]
    return S.WorkloadSpec(instances=insts, policy=S.PolicyKind.parse(sp["policy"]),
                          devices=S.parse_device_config(
                              {"devices": [{"mib": m} for m in sp["device_mib"]]}),
                          time_scale=float.fromhex(sp["time_scale"]))


@pytest.mark.parametrize("rec", RECORDS, ids=[r["name"] for r in RECORDS])
def test_report_matches_reference(rec, cuda):
    rep = S.simulate(build_spec(rec))
    assert rep.makespan_ms == float.fromhex(rec["makespan_ms"])
    assert rep.avg_mem_util_pct == float.fromhex(rec["avg_mem_util_pct"])
    assert rep.avg_device_util_pct == float.fromhex(rec["avg_device_util_pct"])
    assert rep.max_concurrent_holders == rec["max_concurrent_holders"]
    assert rep.oom_count == rec["oom_count"] == 0
    assert rep.summary() == rec["summary"]
    got = [[float.hex(e["t_ms"]), e["instance"], e["event"], e["device"], e["bytes"]]
           for e in rep.events]
    assert got == rec["events"]
    assert [[float.hex(a), float.hex(b)] for a, b in rep.mem_trace] == rec["mem_trace"]
    inst = {str(k): {kk: (float.hex(vv) if isinstance(vv, float) else vv) for kk, vv in v.items()}
            for k, v in rep.instances.items()}
    assert inst == rec["instances"]
    csv = rep.to_csv().splitlines()
    assert csv[:3] == rec["csv_head"] and csv[-1] == rec["csv_tail"]
    # speed-up vs sequential execution (pkg/tests/test_harness.py:119-126),
    # the reference's own value, bit for bit (well inside 1e-12 relative)
    assert S.speedup_vs_sequential(build_spec(rec), rep) == float.fromhex(rec["speedup"])


def _exact_on_grid(rec):
    """Every step duration ms * time_scale / 1000 and the sequential total
    sum(ms) * time_scale are exact in float64 (Fractions), so the kernel's
    tick-sum S and the reference's float sum describe the same number."""
    from fractions import Fraction as F
    sp = rec["spec"]
    if sp["from_json"] is not None:
        return False
    ts = float.fromhex(sp["time_scale"])
    tot = F(0)
    for i in sp["instances"]:
        for ph in i["phases"]:
            for ms in (ph[0], ph[2]):
                if F(ms) * F(ts) / 1000 != F(ms * ts / 1000.0):
                    return False
                tot += F(ms)
    return F(float(tot)) == tot and F(float(tot) * ts) == tot * F(ts)


@pytest.mark.parametrize("rec", [r for r in RECORDS if _exact_on_grid(r)], ids=lambda r: r["name"])
def test_kernel_speedup_program_mode(rec, cuda):
    """The kernel's own speed-up output (sg_out.speedup) in step-program
    mode: when every duration is exact on the tick grid, the kernel's
    (S * 1000 * 2^-e) / (T * 2^-e * 1000) is the reference's value exactly."""
    import numpy as np
    import torch
    from paper_1712_04495_b200 import batch as B
    from paper_1712_04495_b200 import harness as H
    spec = build_spec(rec)
    enc = H.encode_spec(spec)
    if enc.time_mode != 0:
        pytest.skip("float64 mode: the drop-in computes the speed-up from the spec")
    dev = torch.device("cuda", 0)
    n = len(enc.attr)
    apps = np.zeros((1, n, 4), dtype=np.uint32)
    apps[0, :, 3] = enc.attr
    res = B.simulate_batch(torch.from_numpy(apps.view(np.int32)).to(dev), (spec.policy,), enc.cap_mib,
                           steps=torch.from_numpy(enc.steps.view(np.int32).reshape(-1, 4).copy()).to(dev),
                           step_offsets=torch.from_numpy(enc.step_offsets.view(np.int32).copy()).to(dev),
                           tick_log2=enc.tick_log2)
    got = float(res.speedup[0, 0, 0].cpu())
    assert got == float.fromhex(rec["speedup"])


def test_reference_simulator_goldens(cuda):
    """The reference's hand-derived simulator goldens (test_harness.py:93-142,
    test_acceptance.py:229-246), evaluated on the GPU."""
    P = S.builtin_profiles()
    for name in ("ara-like", "mummer-like", "blast-like"):
        assert S.simulate(S.WorkloadSpec(instances=[P[name]])).makespan_ms == 10_000
    r = S.simulate(S.WorkloadSpec(instances=[P["ara-like"]] * 12))
    assert r.makespan_ms == 10_500 and r.max_concurrent_holders == 6 and r.oom_count == 0
    r = S.simulate(S.WorkloadSpec(instances=[P["mummer-like"]] * 12))
    assert r.makespan_ms == 20_000 and r.max_concurrent_holders == 6
    r = S.simulate(S.WorkloadSpec(instances=[P["blast-like"]] * 12))
    assert r.makespan_ms == 55_000 and r.max_concurrent_holders == 2
    sp = {n: 120_000 / S.simulate(S.WorkloadSpec(instances=[P[n]] * 12)).makespan_ms
          for n in ("ara-like", "mummer-like", "blast-like")}
    assert sp["ara-like"] > sp["mummer-like"] > sp["blast-like"]
    import dataclasses
    hi = dataclasses.replace(P["mummer-like"], priority=2)
    inst = [P["ara-like"]] * 4 + [hi] * 4 + [P["blast-like"]] * 4
    dev = S.parse_device_config({"devices": [{"name": "tight", "mib": 2400}]})
    ms = {k: S.simulate(S.WorkloadSpec(instances=inst, policy=k, devices=dev)).makespan_ms
          for k in (S.PolicyKind.FIFO, S.PolicyKind.MMU, S.PolicyKind.PRIORITY_MMU)}
    assert ms[S.PolicyKind.FIFO] == 57_000
    assert ms[S.PolicyKind.MMU] == 56_000
    assert ms[S.PolicyKind.PRIORITY_MMU] == 56_000


def test_select_grants_dropin(cuda):
    """memshare/tests/test_policy.py examples through the GPU selector."""
    class E:
        def __init__(self, c, b, p=0):
            self.client, self.nbytes, self.priority = c, b, p
    Q = [E("A", 3000), E("B", 1000), E("C", 500)]
    K = S.PolicyKind
    assert S.select_grants(Q, 1600, K.FIFO) == []
    assert S.select_grants(Q, 1600, K.MMU) == ["B", "C"]
    q = [E("A", 3000, 2), E("B", 1000, 2)]
    assert S.select_grants(q, 1500, K.PRIORITY_FIFO) == []
    assert S.select_grants(q, 1500, K.PRIORITY_MMU) == ["B"]
    assert S.select_grants([E("A", 500, 1), E("B", 1000, 2)], 1500, K.PRIORITY_FIFO) == ["B"]
    for kind in K:
        assert S.select_grants([], 1000, kind) == []
        assert S.select_grants([E("A", 1000)], 1000, kind) == ["A"]
