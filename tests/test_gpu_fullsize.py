"""Full-size GPU checks at BASELINE.json's configurations (C2: 1M x 64 apps,
C3: 1M x 256, C4: 4M x 128, C5: one GPU's 2M-trace shard of 16M x 64 apps
on 8 simulated devices), where the CPU oracle cannot check every trace:

* the K1 engines (lane kernel v7, warp kernel v3 and, at 256 apps, the
  octet kernel v8: different algorithms sharing only the output record
  code) agree bit for bit on every output of the whole batch;
* a stratified sample of traces across the batch matches the oracle
  (oracle/, the C restatement of memshare.harness.simulate) bit for bit;
* size-independent invariants hold on every record: every app is granted
  and ends (requests fit the device), grants per device = apps on that
  device, busy union <= makespan, memory integral <= capacity x makespan,
  makespan >= the device's last arrival;
* and C2 in full: every one of its 1,048,576 traces x 4 policies against
  the oracle.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1712_04495_b200 import batch as B
from paper_1712_04495_b200.tracegen import CONFIGS
from util import floats_equal

pytestmark = pytest.mark.gpu

SHARD = {"C2": 1 << 20, "C3": 1 << 20, "C4": 4 << 20, "C5": (16 << 20) // 8}


def bits(t):
    """Bit pattern of a float64 tensor (NaN-safe exact comparison)."""
    return t.view(torch.int64) if t.dtype == torch.float64 else t


def run_engine(apps, cfg, engine, monkeypatch):
    monkeypatch.setenv("SGPU_K1", engine)
    res = B.simulate_batch(apps, cfg.policies, cfg.cap_mib)
    torch.cuda.synchronize()
    monkeypatch.delenv("SGPU_K1", raising=False)
    return res


@pytest.mark.parametrize("cname", ["C2", "C3", "C4", "C5"])
def test_full_size(cname, cuda, monkeypatch):
    cfg = CONFIGS[cname]
    n = SHARD[cname]
    napp = cfg.gen.apps_per_trace
    apps = B.generate_traces(cfg.gen, 0, n, device=0)
    lane = run_engine(apps, cfg, "lane", monkeypatch)
    warp = run_engine(apps, cfg, "warp", monkeypatch)
    for f in ("grant", "end", "stats_raw", "mem_pct", "dev_pct", "speedup"):
        assert torch.equal(bits(getattr(lane, f)), bits(getattr(warp, f))), f"{cname}: engines differ in {f}"
    if cname == "C3":  # 256-app traces: the octet kernel (v8) is the default engine there
        octet = run_engine(apps, cfg, "octet", monkeypatch)
        for f in ("grant", "end", "stats_raw", "mem_pct", "dev_pct", "speedup"):
            assert torch.equal(bits(getattr(octet, f)), bits(getattr(warp, f))), f"C3: octet and warp engines differ in {f}"
        del octet
        l256 = run_engine(apps, cfg, "lane256", monkeypatch)
        for f in ("grant", "end", "stats_raw", "mem_pct", "dev_pct", "speedup"):
            assert torch.equal(bits(getattr(l256, f)), bits(getattr(warp, f))), f"C3: lane256 and warp engines differ in {f}"
        del l256
    del warp

    # stratified oracle sample: 1,200 traces spread over the batch
    idx = torch.linspace(0, n - 1, 1200, device=apps.device).long()
    sample = apps.index_select(0, idx).cpu().numpy().view(np.uint32)
    grant = lane.grant.view(len(lane.policies), n, napp).index_select(1, idx).cpu().numpy().view(np.uint32)
    end = lane.end.view(len(lane.policies), n, napp).index_select(1, idx).cpu().numpy().view(np.uint32)
    st_all = lane.stats()
    st = st_all[:, idx.cpu().numpy()]
    mem = lane.mem_pct.index_select(1, idx).cpu().numpy()
    for pi, pol in enumerate(lane.policies):
        g, e, s = O.simulate_burst(sample, cfg.cap_mib, pol.value)
        np.testing.assert_array_equal(grant[pi], g, err_msg=f"{cname} grant {pol}")
        np.testing.assert_array_equal(end[pi], e, err_msg=f"{cname} end {pol}")
        np.testing.assert_array_equal(st[pi].view(np.uint8), s.view(np.uint8), err_msg=f"{cname} stats {pol}")
        for d in range(cfg.ndev):
            _, mp, _ = O.pct_from_stats(s[:, d], cfg.cap_mib[d])
            assert floats_equal(mem[pi][:, d], mp), (cname, pol)

    # invariants on every record
    a = apps.view(n, napp, 4)
    arrival = a[..., 0].long()
    dev = (a[..., 3] >> 8) & 0xFF if cfg.ndev > 1 else torch.zeros_like(arrival)
    per_dev = torch.stack([(dev == d).sum(1) for d in range(cfg.ndev)], 1).cpu().numpy()
    last_arr = torch.stack([torch.where(dev == d, arrival, torch.zeros_like(arrival)).max(1).values
                            for d in range(cfg.ndev)], 1).cpu().numpy()
    cap = np.array(cfg.cap_mib, dtype=np.uint64)
    for pi in range(len(lane.policies)):
        r = st_all[pi]
        assert (r["status"] == 0).all() and (r["unfinished"] == 0).all()
        np.testing.assert_array_equal(r["grants"], per_dev)
        assert (r["busy"] <= r["makespan"]).all()
        assert (r["mem_integral"] <= cap[None, :] * r["makespan"].astype(np.uint64)).all()
        assert (r["makespan"].astype(np.int64) >= last_arr).all()
    assert int((lane.grant == -1).sum()) == 0 and int((lane.end == -1).sum()) == 0


def test_c2_every_trace_against_oracle(cuda, monkeypatch):
    """C2 at its full BASELINE size: all 1,048,576 traces x 4 policies of the
    default engine against the oracle (C restatement, all host cores),
    every grant / end tick and every statistics record."""
    cfg = CONFIGS["C2"]
    n = cfg.n_traces
    monkeypatch.delenv("SGPU_K1", raising=False)
    apps_t = B.generate_traces(cfg.gen, 0, n, device=0)
    res = B.simulate_batch(apps_t, cfg.policies, cfg.cap_mib)
    torch.cuda.synchronize()
    apps = apps_t.cpu().numpy().view(np.uint32)
    grant, end, st = res.ticks("grant"), res.ticks("end"), res.stats()
    for pi, pol in enumerate(res.policies):
        g, e, s = O.simulate_burst(apps, cfg.cap_mib, pol.value)
        assert np.array_equal(grant[pi].reshape(g.shape), g), pol
        assert np.array_equal(end[pi].reshape(e.shape), e), pol
        assert np.array_equal(st[pi].view(np.uint8), s.view(np.uint8)), pol
