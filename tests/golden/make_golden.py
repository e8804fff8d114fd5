"""Generate the golden fixtures in tests/golden/ from the REAL reference.

    python tests/golden/make_golden.py        (needs /root/reference)

Every value here comes from memshare.harness.simulate / memshare.policy
.select_grants imported read-only from /root/reference/pkg/src (through
tests/refsim.py).  Outputs (committed, small):

  ref_burst.npz      random T0 traces of configs C1-C4 (tracegen, seeds 7..),
                     all four policies, dyadic time scale 1000/1024: per-app
                     first-grant / end ticks, makespan ticks, the report's
                     makespan_ms / avg_mem_util_pct / avg_device_util_pct
                     (exact float64), max holders, grants, unfinished, and
                     the speed-up vs sequential execution
                     sum(total_ms) * time_scale / makespan_ms
  ref_multidev.npz   C5-shaped traces (8 simulated devices per trace) pinned
                     by decomposition: simulate() on each device's sub-trace
  ref_reports.json   full MetricsReports (summary, float-exact events,
                     mem_trace, instances) for the reference's own test
                     scenarios and README examples, incl. non-dyadic scales
  ref_select.npz     random queues x 4 policies -> select_grants masks
  ref_criterion5.npz the 100k queues of acceptance criterion 5
                     (test_acceptance.py:174-226, seed 20260823) x 4
                     policies -> the reference's select_grants flags
"""

from __future__ import annotations

import dataclasses
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import refsim  # noqa: E402
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate  # noqa: E402

POLICIES = ("fifo", "mmu", "pfifo", "pmmu")
NONE = 0xFFFFFFFF


def burst_fixture(path: str):
    plan = [("C1", 1, 1), ("C2", 48, 7), ("C3", 4, 8), ("C4", 24, 9)]
    out = {}
    for cname, nt, seed in plan:
        cfg = CONFIGS[cname]
        gen = dataclasses.replace(cfg.gen, seed=seed)
        apps = as_u32x4(generate(gen, 0, nt))
        out[f"{cname}_apps"] = apps
        out[f"{cname}_cap"] = np.array(cfg.cap_mib, dtype=np.uint32)
        out[f"{cname}_seed"] = np.array([seed])
        for pol in POLICIES:
            g = np.full(apps.shape[:2], NONE, dtype=np.uint32)
            e = np.full(apps.shape[:2], NONE, dtype=np.uint32)
            T = np.zeros(nt, dtype=np.uint32)
            f = np.zeros((nt, 3), dtype=np.float64)
            ints = np.zeros((nt, 3), dtype=np.int64)
            spd = np.zeros(nt, dtype=np.float64)
            for t in range(nt):
                r = refsim.run_burst(apps[t], cfg.cap_mib[0], pol)
                spd[t] = r["speedup"]
                g[t] = [NONE if x is None else x for x in r["grant"]]
                e[t] = [NONE if x is None else x for x in r["end"]]
                T[t] = r["T"]
                f[t] = (r["makespan_ms"], r["mem_pct"], r["dev_pct"])
                ints[t] = (r["max_holders"], r["grants"], r["unfinished"])
            out[f"{cname}_{pol}_grant"] = g
            out[f"{cname}_{pol}_end"] = e
            out[f"{cname}_{pol}_T"] = T
            out[f"{cname}_{pol}_floats"] = f
            out[f"{cname}_{pol}_ints"] = ints
            out[f"{cname}_{pol}_speedup"] = spd
    np.savez_compressed(path, **out)


def multidev_fixture(path: str, nt: int = 12, seed: int = 11):
    cfg = CONFIGS["C5"]
    gen = dataclasses.replace(cfg.gen, seed=seed)
    apps = as_u32x4(generate(gen, 0, nt))
    ndev = cfg.ndev
    out = {"apps": apps, "cap": np.array(cfg.cap_mib, dtype=np.uint32)}
    for pol in POLICIES:
        g = np.full(apps.shape[:2], NONE, dtype=np.uint32)
        e = np.full(apps.shape[:2], NONE, dtype=np.uint32)
        T = np.zeros((nt, ndev), dtype=np.uint32)
        f = np.zeros((nt, ndev, 3), dtype=np.float64)
        ints = np.zeros((nt, ndev, 3), dtype=np.int64)
        spd = np.zeros((nt, ndev), dtype=np.float64)
        for t in range(nt):
            devs = (apps[t, :, 3] >> 8) & 0xFF
            for d in range(ndev):
                idx = np.flatnonzero(devs == d)
                r = refsim.run_burst(apps[t, idx], cfg.cap_mib[d], pol)
                for k, a in enumerate(idx):
                    g[t, a] = NONE if r["grant"][k] is None else r["grant"][k]
                    e[t, a] = NONE if r["end"][k] is None else r["end"][k]
                T[t, d] = r["T"]
                f[t, d] = (r["makespan_ms"], r["mem_pct"], r["dev_pct"])
                ints[t, d] = (r["max_holders"], r["grants"], r["unfinished"])
                spd[t, d] = r["speedup"]
        out[f"{pol}_grant"], out[f"{pol}_end"], out[f"{pol}_T"] = g, e, T
        out[f"{pol}_speedup"] = spd
        out[f"{pol}_floats"], out[f"{pol}_ints"] = f, ints
    np.savez_compressed(path, **out)


def report_scenarios():
    """The reference's own simulator scenarios (test_harness.py:86-142,
    test_acceptance.py:229-246, README.md:98-109) plus stress shapes."""
    harness, pol, device = refsim.ref_modules()
    P = harness.builtin_profiles()
    Ph = harness.Phase
    AP = harness.AppProfile
    dev2400 = {"devices": [{"name": "tight", "mib": 2400}]}
    hi = dataclasses.replace(P["mummer-like"], priority=2)
    mixed = [P["ara-like"]] * 4 + [P["mummer-like"]] * 4 + [P["blast-like"]] * 4
    crit6 = [P["ara-like"]] * 4 + [hi] * 4 + [P["blast-like"]] * 4
    burst = AP("burst", [Ph(cpu_ms=900, alloc_mib=700), Ph(busy_ms=100, free_mib=700)])
    sc = []
    for name in ("ara-like", "mummer-like", "blast-like"):
        sc.append((f"{name} x1", {"instances": [[name, 1]]}))
        sc.append((f"{name} x12", {"instances": [[name, 12]]}))
        sc.append((f"{name} x12 ts0.05", {"instances": [[name, 12]], "time_scale": 0.05}))
    sc.append(("ara-like x12 ts0.1", {"instances": [["ara-like", 12]], "time_scale": 0.1}))
    for p in POLICIES:
        sc.append((f"mixed 4+4+4 @2400 {p}", {"_inst": mixed, "policy": p, "device": dev2400}))
        sc.append((f"crit6 @2400 {p}", {"_inst": crit6, "policy": p, "device": dev2400}))
        sc.append((f"mixed 4+4+4 @4799 {p} ts0.15", {"_inst": mixed, "policy": p,
                                                    "time_scale": 0.15}))
    sc.append(("readme burst x8 ts1.0", {"_inst": [burst] * 8}))
    sc.append(("readme burst x8 dyadic", {"_inst": [burst] * 8,
                                          "time_scale": refsim.TIME_SCALE_DYADIC}))
    sc.append(("readme json mmu ts0.25", {"json": {
        "profiles": [{"name": "burst", "phases": [{"cpu_ms": 900, "alloc_mib": 700},
                                                  {"busy_ms": 100, "free_mib": 700}]}],
        "instances": [["burst", 8], ["blast-like", 2]], "policy": "mmu", "time_scale": 0.25}}))
    # edge shapes: zero-length steps, alloc without free, oversize request, priorities
    tiny = AP("tiny", [Ph(alloc_mib=10, busy_ms=50, free_mib=10)], priority=3)
    hold = AP("hold", [Ph(alloc_mib=100)])
    huge = AP("huge", [Ph(cpu_ms=5, alloc_mib=5000, busy_ms=10, free_mib=5000)])
    nop = AP("nop", [Ph()])
    double = AP("double", [Ph(alloc_mib=300), Ph(cpu_ms=20, alloc_mib=200), Ph(busy_ms=30),
                           Ph(free_mib=500)], priority=1)
    for p in POLICIES:
        sc.append((f"edge mix {p}", {"_inst": [tiny, hold, huge, nop, double, tiny, double],
                                     "policy": p, "device": {"devices": [{"mib": 1000}]}}))
    sc.append(("hold only t=0", {"_inst": [hold, hold]}))
    sc.append(("nop only", {"_inst": [nop, nop, nop]}))
    rng = random.Random(5)
    for k in range(24):
        n = rng.randint(2, 14)
        insts = []
        for i in range(n):
            phases = []
            for _ in range(rng.randint(1, 4)):
                phases.append(Ph(cpu_ms=rng.choice([0, 0, 1, 3, 7.5, 12.25]),
                                 alloc_mib=rng.choice([0, 50, 120, 300]),
                                 busy_ms=rng.choice([0, 2, 5, 9.5]),
                                 free_mib=0))
            held = sum(ph.alloc_mib for ph in phases)
            if held and rng.random() < 0.85:
                phases.append(Ph(free_mib=held))
            insts.append(AP(f"r{i}", phases, priority=rng.randint(0, 3)))
        p = POLICIES[k % 4]
        ts = rng.choice([1.0, 0.5, 0.3, refsim.TIME_SCALE_DYADIC])
        sc.append((f"random programs #{k} {p} ts{ts}",
                   {"_inst": insts, "policy": p, "time_scale": ts,
                    "device": {"devices": [{"mib": rng.choice([400, 700, 1000])}]}}))
    return sc


def _spec_from(doc):
    harness, pol, device = refsim.ref_modules()
    if "json" in doc:
        return harness.WorkloadSpec.from_json(doc["json"]), doc["json"]
    kw = {}
    if "policy" in doc:
        kw["policy"] = pol.PolicyKind.parse(doc["policy"])
    if "device" in doc:
        kw["devices"] = device.parse_device_config(doc["device"])
    if "time_scale" in doc:
        kw["time_scale"] = doc["time_scale"]
    if "_inst" in doc:
        insts = doc["_inst"]
    else:
        P = harness.builtin_profiles()
        insts = [P[n] for n, c in doc["instances"] for _ in range(c)]
    return harness.WorkloadSpec(instances=insts, **kw), None


def spec_to_json(spec, doc_json):
    """Serialisable description of a reference WorkloadSpec."""
    return {
        "instances": [{"name": p.name, "priority": p.priority,
                       "phases": [[ph.cpu_ms, ph.alloc_mib, ph.busy_ms, ph.free_mib]
                                  for ph in p.phases]} for p in spec.instances],
        "policy": spec.policy.value,
        "device_mib": [d.total_bytes // (1 << 20) for d in spec.devices],
        "time_scale": float.hex(float(spec.time_scale)),
        "from_json": doc_json,
    }


def reports_fixture(path: str):
    recs = []
    for name, doc in report_scenarios():
        spec, js = _spec_from(doc)
        rep, raw = refsim.run_spec(spec)
        recs.append({
            "name": name,
            "spec": spec_to_json(spec, js),
            "makespan_ms": float.hex(rep.makespan_ms),
            "avg_mem_util_pct": float.hex(rep.avg_mem_util_pct),
            "avg_device_util_pct": float.hex(rep.avg_device_util_pct),
            "max_concurrent_holders": rep.max_concurrent_holders,
            # sum(p.total_ms() for p in spec.instances) * time_scale / makespan_ms
            "speedup": float.hex(refsim.speedup_of(spec, rep)),
            "oom_count": rep.oom_count,
            "summary": rep.summary(),
            "events": [[float.hex(e["t_ms"]), e["instance"], e["event"], e["device"], e["bytes"]]
                       for e in rep.events],
            "mem_trace": [[float.hex(a), float.hex(b)] for a, b in rep.mem_trace],
            "instances": {str(k): {kk: (float.hex(vv) if isinstance(vv, float) else vv)
                                   for kk, vv in v.items()} for k, v in rep.instances.items()},
            "csv_head": rep.to_csv().splitlines()[:3],
            "csv_tail": rep.to_csv().splitlines()[-1],
        })
    with open(path, "w") as f:
        json.dump(recs, f, separators=(",", ":"))


def select_fixture(path: str, trials: int = 4000, seed: int = 20260823):
    """Random queues as in the reference's acceptance criterion 5
    (test_acceptance.py:204-226): n U[0,8], sizes U[1,2000], prio U[0,3],
    free U[0,6000]; plus longer queues (up to 70 entries)."""
    _, pol, _ = refsim.ref_modules()

    class E:
        __slots__ = ("client", "nbytes", "priority")

        def __init__(self, c, b, p):
            self.client, self.nbytes, self.priority = c, b, p

    rng = random.Random(seed)
    offs, sizes, prios, frees, kinds, granted = [0], [], [], [], [], []
    for k in range(trials):
        n = rng.randint(0, 8) if k % 4 else rng.randint(0, 70)
        sz = [rng.randint(1, 2000) for _ in range(n)]
        pr = [rng.randint(0, 3) for _ in range(n)]
        fr = rng.randint(0, 6000 if n <= 8 else 40000)
        for kind in pol.PolicyKind:
            q = [E(i, sz[i], pr[i]) for i in range(n)]
            got = set(pol.select_grants(q, fr, kind))
            sizes += sz
            prios += pr
            frees.append(fr)
            kinds.append(kind.code)
            granted += [1 if i in got else 0 for i in range(n)]
            offs.append(len(sizes))
    np.savez_compressed(path, offsets=np.array(offs, np.int64), nbytes=np.array(sizes, np.int64),
                        prio=np.array(prios, np.int32), free=np.array(frees, np.int64),
                        kind=np.array(kinds, np.uint32), granted=np.array(granted, np.uint8))


def criterion5_fixture(path: str):
    """The reference's own select_grants on the 100k criterion-5 queues x 4
    policies (policy-major within a queue), granted flags packed as bits."""
    _, pol, _ = refsim.ref_modules()

    class E:
        __slots__ = ("client", "nbytes", "priority")

        def __init__(self, c, b, p):
            self.client, self.nbytes, self.priority = c, b, p

    flags = []
    from util import criterion5_queues
    for sizes, prios, free in criterion5_queues():
        q = [E(i, sizes[i], prios[i]) for i in range(len(sizes))]
        for kind in pol.PolicyKind:
            got = set(pol.select_grants(q, free, kind))
            flags += [1 if i in got else 0 for i in range(len(sizes))]
    np.savez_compressed(path, granted_bits=np.packbits(np.array(flags, np.uint8)),
                        n_flags=np.array([len(flags)], np.int64))


def main():
    if not refsim.available():
        raise SystemExit("the reference tree is not available here")
    burst_fixture(os.path.join(HERE, "ref_burst.npz"))
    multidev_fixture(os.path.join(HERE, "ref_multidev.npz"))
    reports_fixture(os.path.join(HERE, "ref_reports.json"))
    select_fixture(os.path.join(HERE, "ref_select.npz"))
    criterion5_fixture(os.path.join(HERE, "ref_criterion5.npz"))
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
