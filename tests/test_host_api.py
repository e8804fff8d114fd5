"""Host-side mirror of the reference interface (CPU only): PolicyKind,
WorkloadSpec.from_json, encoding of specs into step programs, the tick-grid
rule, MetricsReport formatting, and loud failure without a GPU."""

import math

import numpy as np
import pytest
import torch

import paper_1712_04495_b200 as S
from paper_1712_04495_b200 import _lib
from paper_1712_04495_b200.harness import encode_spec, sequential_ms


def test_policy_kind_codes_and_parse():
    K = S.PolicyKind
    assert [k.code for k in K] == [0, 1, 2, 3]
    assert K.parse("PMMU") is K.PRIORITY_MMU and K.from_code(2) is K.PRIORITY_FIFO
    with pytest.raises(ValueError, match="unknown policy"):
        K.parse("lifo")


def test_workload_json_like_reference():
    spec = S.WorkloadSpec.from_json({"instances": [["ara-like", 2], ["blast-like", 1]],
                                     "policy": "mmu", "time_scale": 0.25, "seed": 9})
    assert [p.name for p in spec.instances] == ["ara-like", "ara-like", "blast-like"]
    assert spec.policy is S.PolicyKind.MMU and spec.time_scale == 0.25
    spec = S.WorkloadSpec.from_json({"profiles": [{"name": "tiny", "priority": 3, "phases": [
        {"alloc_mib": 10, "busy_ms": 50, "free_mib": 10}]}], "instances": [["tiny", 2]]})
    assert spec.instances[0].priority == 3 and spec.instances[0].peak_mib() == 10
    with pytest.raises(S.SchemaError):
        S.WorkloadSpec.from_json({"instances": [["nope", 1]]})
    with pytest.raises(S.SchemaError):
        S.WorkloadSpec.from_json({"instances": []})
    spec = S.WorkloadSpec.from_json({"instances": [["ara-like", 1]],
                                     "device": {"devices": [{"mib": 1000}]}})
    assert spec.devices[0].total_bytes == 1000 * S.MIB


def test_builtin_profiles_shapes():
    p = S.builtin_profiles()
    assert {k: (v.peak_mib(), v.total_ms()) for k, v in p.items()} == {
        "ara-like": (768, 10_000), "mummer-like": (720, 10_000), "blast-like": (1750, 10_000)}


def test_device_config_errors():
    for bad in ({}, {"devices": []}, {"devices": [{"name": "x"}]}, {"devices": [{"mib": 0}]},
                {"devices": [{"mib": 1.5}]}):
        with pytest.raises(S.SchemaError):
            S.parse_device_config(bad)


def test_encode_dyadic_grid_and_flattening():
    P = S.builtin_profiles()
    enc = encode_spec(S.WorkloadSpec(instances=[P["blast-like"]]))
    assert enc.time_mode == _lib.TIME_TICKS and enc.tick_log2 == 0  # whole seconds
    ops = [(int(s["op"]), int(s["mib"]), int(s["dur"])) for s in enc.steps]
    # blast: cpu 1 s, alloc 1750, busy 8 s, cpu 1 s, free 1750 (harness.py:478-490)
    assert ops[:5] == [(0, 0, 1), (1, 1750, 0), (2, 0, 8), (0, 0, 1), (3, 1750, 0)]
    enc = encode_spec(S.WorkloadSpec(instances=[P["ara-like"]]))
    assert enc.tick_log2 == 1 and int(enc.steps[0]["dur"]) == 19  # 9.5 s = 19 half-seconds
    # 0.9 s is not dyadic: float64 mode
    b = S.AppProfile("b", [S.Phase(cpu_ms=900, alloc_mib=700), S.Phase(busy_ms=100, free_mib=700)])
    enc = encode_spec(S.WorkloadSpec(instances=[b]))
    assert enc.time_mode == _lib.TIME_F64
    assert np.frombuffer(np.uint64(enc.steps[0]["dur"]).tobytes(), np.float64)[0] == 0.9


def test_encode_shared_profiles_like_distinct_ones():
    """Instances sharing an AppProfile object are encoded once per call; the
    encoding equals that of a spec whose instances are distinct copies
    (steps, offsets, attributes, tick grid), including the tick-grid bound
    that counts every instance (harness.py:478-490)."""
    import copy
    P = S.builtin_profiles()
    shared = [P["ara-like"]] * 5 + [P["mummer-like"]] * 3 + [P["blast-like"]] * 2 + [P["ara-like"]]
    distinct = [copy.deepcopy(p) for p in shared]
    for t_scale in (1.0, 0.75, 1000 / 1024):
        a = encode_spec(S.WorkloadSpec(instances=shared, time_scale=t_scale))
        b = encode_spec(S.WorkloadSpec(instances=distinct, time_scale=t_scale))
        assert (a.time_mode, a.tick_log2, a.cap_mib) == (b.time_mode, b.tick_log2, b.cap_mib)
        assert a.steps.tobytes() == b.steps.tobytes()
        assert a.step_offsets.tolist() == b.step_offsets.tolist()
        assert a.attr.tolist() == b.attr.tolist()
    # the exact-sum bound counts every instance: many copies push a dyadic
    # grid past 2^32 ticks and into float64 mode
    long = S.AppProfile("long", [S.Phase(cpu_ms=2 ** 21 * 1000.0)])
    assert encode_spec(S.WorkloadSpec(instances=[long] * 2)).time_mode == _lib.TIME_TICKS
    assert encode_spec(S.WorkloadSpec(instances=[long] * 4096)).time_mode == _lib.TIME_F64


def test_priorities_become_dense_ranks():
    prof = lambda p: S.AppProfile("x", [S.Phase(alloc_mib=1, free_mib=1)], priority=p)
    enc = encode_spec(S.WorkloadSpec(instances=[prof(100), prof(-5), prof(100), prof(7)]))
    assert enc.attr.tolist() == [2, 0, 2, 1]


def test_sequential_ms():
    P = S.builtin_profiles()
    assert sequential_ms(S.WorkloadSpec(instances=[P["ara-like"]] * 12)) == 120_000


def test_report_formatting():
    r = S.MetricsReport(1100.0, {0: {"start_ms": 0.0}}, [
        {"t_ms": 0.0, "instance": 0, "event": "start", "device": 0, "bytes": 0}],
        [(0.0, 0.0)], 10.5, 18.25, 0, 6)
    assert r.summary()["audit_ok"] is True and r.summary()["instances"] == 1
    csv = r.to_csv().splitlines()
    assert csv[0] == "t_ms,instance,event,device,bytes" and csv[1] == "0.000,0,start,0,0"
    assert csv[-1].startswith("# makespan_ms=1100.0 ")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    with pytest.raises(S.SgpuUnavailable):
        S.simulate(S.WorkloadSpec(instances=[S.builtin_profiles()["ara-like"]]))

    class E:
        client, nbytes, priority = "a", 1, 0
    with pytest.raises(S.SgpuUnavailable):
        S.select_grants([E()], 10, "fifo")


def test_empty_spec_report():
    r = S.simulate(S.WorkloadSpec(instances=[]))
    assert r.makespan_ms == 0.0 and r.instances == {} and r.events == []
