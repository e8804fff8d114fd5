"""GPU parity: the sm_100a engine through the C ABI against the reference's
golden vectors (tests/golden/, produced by the real memshare simulator) and
the CPU oracle (oracle/, a C restatement of the same simulator) on seeded
inputs.  Bit-exact on every integer and on the float64 percentages."""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1712_04495_b200 import batch as B
from paper_1712_04495_b200.tracegen import CONFIGS, GenParams, as_u32x4, generate
from util import NEVER, POLICIES, criterion5_flags, criterion5_queues, floats_equal, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "warp"], autouse=True)
def engine(request, monkeypatch):
    """Every parity test runs on both K1 engines: `auto` takes the lane kernel
    (v5) wherever the batch is eligible (T0, <= 128 apps) and the octet
    kernel (v8) for 129..256-app single-device T0 traces, `warp` forces the
    warp-per-trace kernel (v3)."""
    if request.param == "warp":
        monkeypatch.setenv("SGPU_K1", "warp")
    else:
        monkeypatch.delenv("SGPU_K1", raising=False)
    return request.param


def to_dev(apps_u32, dev):
    a = np.ascontiguousarray(apps_u32, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).to(dev)


def run(apps_u32, policies, caps, dev, **kw):
    res = B.simulate_batch(to_dev(apps_u32, dev), policies, caps, **kw)
    torch.cuda.synchronize()
    return res


def check_against_oracle(apps, caps, dev, policies=POLICIES):
    res = run(apps, policies, caps, dev)
    st = res.stats()
    grant = res.ticks("grant").reshape(len(res.policies), *apps.shape[:2])
    end = res.ticks("end").reshape(len(res.policies), *apps.shape[:2])
    mem = res.mem_pct.cpu().numpy()
    devp = res.dev_pct.cpu().numpy()
    spd = res.speedup.cpu().numpy()
    ndev = len(caps)
    seq = O.seq_ticks(apps, ndev)
    dv = (apps[..., 3] >> 8) & 0xFF if ndev > 1 else np.zeros(apps.shape[:2], np.uint32)
    dv = np.where(dv < ndev, dv, 0)
    cnt = np.stack([(dv == d).sum(axis=1) for d in range(ndev)], axis=1)
    for pi, pol in enumerate(res.policies):
        g, e, s = O.simulate_burst(apps, caps, pol.value)
        want = O.speedup_from(seq, s["makespan"], cnt)
        assert np.array_equal(np.isnan(spd[pi]), np.isnan(want)), pol
        assert floats_equal(np.nan_to_num(spd[pi]), np.nan_to_num(want)), f"speedup {pol}"
        np.testing.assert_array_equal(grant[pi], g, err_msg=f"grant {pol}")
        np.testing.assert_array_equal(end[pi], e, err_msg=f"end {pol}")
        for f in ("makespan", "busy", "mem_integral", "grants", "pops", "max_holders",
                  "unfinished", "status"):
            np.testing.assert_array_equal(st[pi][f], s[f], err_msg=f"{f} {pol}")
        for d in range(len(caps)):
            _, mp, dp = O.pct_from_stats(s[:, d], caps[d])
            assert floats_equal(mem[pi][:, d], mp), pol
            assert floats_equal(devp[pi][:, d], dp), pol
    return res


# ------------------------------------------------------------ golden vectors

@pytest.mark.parametrize("cname", ["C1", "C2", "C3", "C4"])
def test_golden_burst(cname, cuda):
    z = golden("ref_burst.npz")
    apps = z[f"{cname}_apps"]
    caps = tuple(int(c) for c in z[f"{cname}_cap"])
    res = run(apps, POLICIES, caps, cuda)
    st = res.stats()
    n_tr, n = apps.shape[:2]
    grant = res.ticks("grant").reshape(4, n_tr, n)
    end = res.ticks("end").reshape(4, n_tr, n)
    mem = res.mem_pct.cpu().numpy()[..., 0]
    devp = res.dev_pct.cpu().numpy()[..., 0]
    spd = res.speedup.cpu().numpy()[..., 0]
    for pi, pol in enumerate(POLICIES):
        assert res.policies[pi].value == pol
        # speed-up vs sequential, as the reference computes it (bit-exact)
        assert floats_equal(spd[pi], z[f"{cname}_{pol}_speedup"]), pol
        np.testing.assert_array_equal(grant[pi], z[f"{cname}_{pol}_grant"])
        np.testing.assert_array_equal(end[pi], z[f"{cname}_{pol}_end"])
        np.testing.assert_array_equal(st[pi][:, 0]["makespan"], z[f"{cname}_{pol}_T"])
        fl = z[f"{cname}_{pol}_floats"]
        ms, _, _ = B.pct_host(st[pi][:, 0], caps[0])
        assert floats_equal(ms, fl[:, 0])
        assert floats_equal(mem[pi], fl[:, 1])
        assert floats_equal(devp[pi], fl[:, 2])
        ints = z[f"{cname}_{pol}_ints"]
        np.testing.assert_array_equal(st[pi][:, 0]["max_holders"], ints[:, 0])
        np.testing.assert_array_equal(st[pi][:, 0]["grants"], ints[:, 1])
        np.testing.assert_array_equal(st[pi][:, 0]["unfinished"], ints[:, 2])


def test_golden_readme_burst_c1(cuda):
    """README burst x8 @4799 (config 1): grants at 900 and 1000 ticks,
    6 concurrent holders, identical for all four policies."""
    apps = as_u32x4(generate(CONFIGS["C1"].gen, 0, 1))
    res = run(apps, POLICIES, (4799,), cuda)
    st = res.stats()
    for pi in range(4):
        g = res.ticks("grant")[pi]
        assert sorted(set(g.tolist())) == [900, 1000]
        assert (g == 900).sum() == 6
        assert st[pi][0, 0]["max_holders"] == 6
        assert st[pi][0, 0]["makespan"] == 1100


def test_golden_multidev(cuda):
    z = golden("ref_multidev.npz")
    apps = z["apps"]
    caps = tuple(int(c) for c in z["cap"])
    res = run(apps, POLICIES, caps, cuda)
    st = res.stats()
    n_tr, n = apps.shape[:2]
    mem = res.mem_pct.cpu().numpy()
    devp = res.dev_pct.cpu().numpy()
    spd = res.speedup.cpu().numpy()
    for pi, pol in enumerate(POLICIES):
        assert floats_equal(spd[pi], z[f"{pol}_speedup"]), pol
        np.testing.assert_array_equal(res.ticks("grant")[pi].reshape(n_tr, n), z[f"{pol}_grant"])
        np.testing.assert_array_equal(res.ticks("end")[pi].reshape(n_tr, n), z[f"{pol}_end"])
        np.testing.assert_array_equal(st[pi]["makespan"], z[f"{pol}_T"])
        fl = z[f"{pol}_floats"]
        assert floats_equal(mem[pi], fl[..., 1])
        assert floats_equal(devp[pi], fl[..., 2])
        ints = z[f"{pol}_ints"]
        np.testing.assert_array_equal(st[pi]["max_holders"], ints[..., 0])
        np.testing.assert_array_equal(st[pi]["grants"], ints[..., 1])
        np.testing.assert_array_equal(st[pi]["unfinished"], ints[..., 2])


@pytest.mark.parametrize("n,ndev,pols", [(128, 8, POLICIES), (100, 4, POLICIES), (128, 2, ("pmmu",)),
                                          (40, 8, ("fifo", "pfifo")), (64, 3, POLICIES)])
def test_multidev_lane_shapes(n, ndev, pols, cuda):
    """Multi-device traces at the lane kernel's shape limits: 128 apps x 8
    devices x 4 policies (32 lanes per trace, one trace per warp), 100 apps
    over 4 devices, one policy on 2 devices, 8 devices x 2 policies, an odd
    device count; random device per app, per-device capacities."""
    rng = np.random.default_rng(300 + n + ndev)
    nt = 400
    apps = np.zeros((nt, n, 4), dtype=np.uint32)
    apps[:, :, 0] = rng.integers(0, 3000, (nt, n))
    apps[:, :, 1] = rng.integers(0, 700, (nt, n))
    apps[:, :, 2] = rng.integers(0, 900, (nt, n))
    prio = rng.integers(0, 4, (nt, n)).astype(np.uint32)
    dev = rng.integers(0, ndev, (nt, n)).astype(np.uint32)
    apps[:, :, 3] = prio | (dev << 8)
    caps = tuple(int(c) for c in rng.integers(600, 2000, ndev))
    check_against_oracle(apps, caps, cuda, policies=pols)


# ------------------------------------------------------------ oracle, seeded

@pytest.mark.parametrize("cname,nt", [("C2", 3000), ("C3", 300), ("C4", 2000), ("C5", 1500)])
def test_oracle_seeded(cname, nt, cuda):
    cfg = CONFIGS[cname]
    apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=101), 5000, nt))
    check_against_oracle(apps, cfg.cap_mib, cuda, cfg.policies)


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 100, 255, 256, 257, 700, 1024])
def test_apps_per_trace_shapes(n, cuda):
    """Every K instantiation (1, 2, 4, 8, 32 apps per lane) incl. max size."""
    g = GenParams(seed=n, apps_per_trace=n, arr_hi=3 * n, mem_lo=1, mem_hi=60_000)
    apps = as_u32x4(generate(g, 0, 40 if n < 500 else 8))
    check_against_oracle(apps, (184_320,), cuda)


@pytest.mark.parametrize("n", [65, 100, 128, 200, 256])
def test_lane_kernel_long_traces_forced(n, cuda, monkeypatch):
    """The lane kernel's scan path (65..256 apps; taken only when forced)."""
    monkeypatch.setenv("SGPU_K1", "lane")
    g = GenParams(seed=n, apps_per_trace=n, arr_hi=3 * n, mem_lo=1, mem_hi=60_000, prio_levels=5)
    apps = as_u32x4(generate(g, 0, 64))
    check_against_oracle(apps, (184_320,), cuda)


@pytest.mark.parametrize("k1", ["octet", "lane256"])
@pytest.mark.parametrize("pols", [POLICIES, ("pfifo", "pmmu"), ("mmu",), ("fifo", "mmu", "pmmu")])
def test_octet_kernel_shapes(pols, k1, cuda, monkeypatch):
    """K1 v8 (octet per simulation, 129..256-app traces): C3-shaped traces,
    edge traces (zero fields, simultaneous arrivals, stuck requests, ties),
    and the shapes its exact fallback takes over (more than 32 busy apps at
    once, more than eight priority classes, priorities of 32 and above)."""
    monkeypatch.setenv("SGPU_K1", k1)  # (both 129..256-app kernels; the fixture's warp run covers v3)
    rng = np.random.default_rng(808)
    cfg = CONFIGS["C3"]
    c3 = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=808), 0, 24))
    edge = np.zeros((24, 256, 4), dtype=np.uint32)
    edge[..., 0] = rng.choice([0, 0, 1, 5, 9, 40, 41], (24, 256))
    edge[..., 1] = rng.choice([0, 100, 250, 500, 1000, 1001], (24, 256))
    edge[..., 2] = rng.choice([0, 0, 1, 3, 7, 30], (24, 256))
    edge[..., 3] = rng.integers(0, 4, (24, 256))
    many = np.zeros((16, 256, 4), dtype=np.uint32)   # tiny requests: up to 256 busy at once
    many[..., 0] = rng.integers(0, 64, (16, 256))
    many[..., 1] = rng.integers(1, 8, (16, 256))
    many[..., 2] = rng.integers(50, 400, (16, 256))
    many[..., 3] = rng.integers(0, 4, (16, 256))
    many[:8, :, 2] = rng.integers(1, 3, (8, 256))      # ... or only a few
    many[:4, :, 3] = rng.integers(0, 12, (4, 256))     # > 8 classes
    many[4:6, :, 3] = rng.integers(30, 40, (2, 256))   # priorities >= 32
    for apps, caps in ((c3, cfg.cap_mib), (edge, (1000,)), (many, (300,))):
        check_against_oracle(apps, caps, cuda, policies=pols)
    for n in (129, 200, 255):   # shorter traces on the same kernel (n_pad 256)
        g = GenParams(seed=n, apps_per_trace=n, arr_hi=2 * n, mem_lo=1, mem_hi=30_000, prio_levels=5)
        check_against_oracle(as_u32x4(generate(g, 0, 16)), (100_000,), cuda, policies=pols)


@pytest.mark.parametrize("k1", ["octet", "lane256"])
def test_octet_kernel_ragged(k1, cuda, monkeypatch):
    """Ragged batches up to 256 apps per trace on the octet and lane256 kernels."""
    monkeypatch.setenv("SGPU_K1", k1)
    rng = np.random.default_rng(19)
    lens = rng.integers(129, 257, 40)
    total = int(lens.sum())
    g = GenParams(seed=5, apps_per_trace=1, arr_hi=500, mem_lo=1000, mem_hi=60_000)
    flat = as_u32x4(generate(dataclasses.replace(g, apps_per_trace=total), 0, 1))[0]
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    res = B.simulate_batch(to_dev(flat, cuda), POLICIES, 184_320,
                           trace_offsets=torch.from_numpy(offs).to(cuda),
                           apps_total=total, max_apps=int(lens.max()))
    torch.cuda.synchronize()
    st = res.stats()
    for pi, pol in enumerate(res.policies):
        for t in range(len(lens)):
            a = flat[offs[t]:offs[t + 1]][None]
            gg, ee, ss = O.simulate_burst(a, (184_320,), pol.value)
            np.testing.assert_array_equal(res.ticks("grant")[pi][offs[t]:offs[t + 1]], gg[0])
            np.testing.assert_array_equal(res.ticks("end")[pi][offs[t]:offs[t + 1]], ee[0])
            for f in ("makespan", "busy", "mem_integral", "max_holders", "pops", "grants", "unfinished"):
                assert st[pi][t, 0][f] == ss[0, 0][f], (pol, t, f)


def test_edge_cases(cuda):
    """Zero fields, stuck oversize requests, simultaneous arrivals, exact fits."""
    rng = np.random.default_rng(3)
    traces = []
    n = 48
    for k in range(64):
        a = np.zeros((n, 4), dtype=np.uint32)
        a[:, 0] = rng.choice([0, 0, 1, 5, 9], n)              # many simultaneous arrivals
        a[:, 1] = rng.choice([0, 100, 250, 500, 1000, 1001], n)  # 0 = no alloc, 1001 > cap
        a[:, 2] = rng.choice([0, 0, 1, 3, 7], n)              # busy 0 => free at grant
        a[:, 3] = rng.integers(0, 4, n)
        traces.append(a)
    apps = np.stack(traces)
    check_against_oracle(apps, (1000,), cuda)
    # all-zero apps: end at t=0
    z = np.zeros((3, 5, 4), dtype=np.uint32)
    res = check_against_oracle(z, (10,), cuda)
    assert (res.ticks("end") == 0).all() and (res.ticks("grant") == NEVER).all()


def test_lane_fallback_heap_overflow(cuda):
    """More than 32 apps busy at once (no-alloc apps with long busy steps)
    overflow a lane's heap; those lanes are re-simulated exactly in-kernel."""
    rng = np.random.default_rng(5)
    n, nt = 64, 96
    apps = np.zeros((nt, n, 4), dtype=np.uint32)
    apps[:, :, 0] = rng.integers(0, 40, (nt, n))
    apps[:, :, 1] = np.where(rng.random((nt, n)) < 0.7, 0, rng.integers(1, 300, (nt, n)))
    apps[:, :, 2] = rng.integers(500, 900, (nt, n))
    apps[:, :, 3] = rng.integers(0, 4, (nt, n))
    apps[::2, :, 1] = rng.integers(1, 20, (nt // 2, n))      # mixed: some lanes stay on the fast path
    check_against_oracle(apps, (1000,), cuda)


def test_lane_fallback_tick_range(cuda):
    """Traces with arrivals >= 2^31 or busy steps >= 2^21 ticks (whose times
    could approach the 32-bit tick range) take the exact fallback."""
    rng = np.random.default_rng(8)
    n, nt = 40, 64
    apps = np.zeros((nt, n, 4), dtype=np.uint32)
    apps[:, :, 0] = rng.integers(0, 1000, (nt, n))
    apps[:, :, 1] = rng.integers(1, 600, (nt, n))
    apps[:, :, 2] = rng.integers(1, 50, (nt, n))
    apps[:8, 0, 0] = np.uint32(0xF0000000)                  # arrival >= 2^31
    apps[8:16, 1, 2] = np.uint32(1 << 22)                    # busy >= 2^21, still in range
    check_against_oracle(apps, (1000,), cuda)


@pytest.mark.parametrize("n,ndev", [(32, 1), (64, 1), (100, 1), (128, 1), (64, 2)])
def test_lane_retry_pass(n, ndev, cuda):
    """Traces that need 64-bit event keys (arrival max + busy sum past
    LaneKey::LIM) with 6..26 apps busy at once: those whose 64-bit-key lanes
    overflow the main pass's 10-event heap are re-simulated by the second
    launch (20-event heap), the busiest ones again by the warp fallback,
    mixed in one batch with traces that keep 32-bit keys."""
    rng = np.random.default_rng(40 + n + ndev)
    nt = 240
    apps = np.zeros((nt, n, 4), dtype=np.uint32)
    apps[:, :, 0] = rng.integers(0, 64, (nt, n))
    conc = np.linspace(6, 26, nt).astype(np.uint32)
    apps[:, :, 1] = (1000 // conc)[:, None]
    apps[:, :, 2] = rng.integers(1 << 14, 1 << 16, (nt, n))      # 64-bit keys
    apps[::5, :, 2] = rng.integers(1, 64, (len(apps[::5]), n))    # 32-bit keys
    apps[:, :, 3] = rng.integers(0, 3, (nt, n))
    if ndev > 1:
        apps[:, :, 3] |= (np.arange(n) % ndev).astype(np.uint32)[None, :] << 8
    check_against_oracle(apps, (1000,) * ndev, cuda)


def test_wide_sort_keys(cuda):
    """Arrivals >= 2^22 and requests >= 2^24 MiB take the 64-bit key sorts of
    the lane kernel's staging (narrow 32-bit sorts otherwise)."""
    rng = np.random.default_rng(12)
    n, nt = 64, 128
    apps = np.zeros((nt, n, 4), dtype=np.uint32)
    apps[:, :, 0] = rng.integers(0, 1 << 30, (nt, n))
    apps[:, :, 1] = rng.integers(1 << 20, 1 << 26, (nt, n))
    apps[:, :, 2] = rng.integers(1, 1 << 20, (nt, n))
    apps[:, :, 3] = rng.integers(0, 3, (nt, n))
    apps[::3, :, 0] = rng.integers(0, 50_000, (len(apps[::3]), n))  # some traces narrow
    check_against_oracle(apps, (1 << 27,), cuda)


def test_ragged_offsets(cuda):
    rng = np.random.default_rng(9)
    lens = rng.integers(0, 90, 300)
    lens[:3] = [0, 1, 0]
    total = int(lens.sum())
    g = GenParams(seed=4, apps_per_trace=1)
    flat = as_u32x4(generate(dataclasses.replace(g, apps_per_trace=total), 0, 1))[0]
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    res = B.simulate_batch(to_dev(flat, cuda), POLICIES, 184_320,
                           trace_offsets=torch.from_numpy(offs).to(cuda),
                           apps_total=total, max_apps=int(lens.max()))
    torch.cuda.synchronize()
    st = res.stats()
    for pi, pol in enumerate(res.policies):
        for t in range(len(lens)):
            a = flat[offs[t]:offs[t + 1]][None]
            gg, ee, ss = O.simulate_burst(a, (184_320,), pol.value)
            np.testing.assert_array_equal(res.ticks("grant")[pi][offs[t]:offs[t + 1]], gg[0])
            np.testing.assert_array_equal(res.ticks("end")[pi][offs[t]:offs[t + 1]], ee[0])
            for f in ("makespan", "busy", "mem_integral", "max_holders", "pops", "grants"):
                assert st[pi][t, 0][f] == ss[0, 0][f], (pol, t, f)


def test_single_policy_subsets(cuda):
    cfg = CONFIGS["C2"]
    apps = as_u32x4(generate(cfg.gen, 0, 200))
    for pols in (("pmmu",), ("mmu", "pfifo")):
        check_against_oracle(apps, cfg.cap_mib, cuda, pols)


# ------------------------------------------------------------ other kernels

@pytest.mark.parametrize("cname", ["C2", "C3", "C5"])
def test_generator_bit_identical(cname, cuda):
    gen = CONFIGS[cname].gen
    t = B.generate_traces(gen, 12345, 777, device=0)
    torch.cuda.synchronize()
    want = as_u32x4(generate(gen, 12345, 777))
    np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), want)


def test_reduce_stats(cuda):
    cfg = CONFIGS["C4"]
    apps = as_u32x4(generate(cfg.gen, 0, 5000))
    res = run(apps, POLICIES, cfg.cap_mib, cuda)
    agg = B.aggr_to_dict(B.reduce_stats(res.stats_raw))
    st = res.stats().reshape(-1)
    assert agg["records"] == st.size
    assert agg["sum_makespan"] == int(st["makespan"].astype(np.uint64).sum())
    assert agg["sum_mem_integral"] == int(st["mem_integral"].astype(np.uint64).sum())
    assert agg["sum_busy"] == int(st["busy"].astype(np.uint64).sum())
    assert agg["sum_grants"] == int(st["grants"].astype(np.uint64).sum())
    assert agg["sum_pops"] == int(st["pops"].astype(np.uint64).sum())
    assert agg["max_makespan"] == int(st["makespan"].max())
    assert agg["max_holders"] == int(st["max_holders"].max())
    assert agg["sum_unfinished"] == int(st["unfinished"].astype(np.uint64).sum())


def test_select_grants_batch_golden(cuda):
    from paper_1712_04495_b200.policy import select_grants_batch
    z = golden("ref_select.npz")
    off = z["offsets"]
    queues = [(z["nbytes"][off[i]:off[i + 1]], z["prio"][off[i]:off[i + 1]])
              for i in range(len(off) - 1)]
    masks = select_grants_batch(queues, z["free"], z["kind"].tolist())
    got = np.concatenate([m.astype(np.uint8) for m in masks])
    np.testing.assert_array_equal(got, z["granted"])


def test_host_pipeline_matches_device(cuda):
    cfg = CONFIGS["C2"]
    apps = as_u32x4(generate(cfg.gen, 0, 10_000))
    dres = run(apps, POLICIES, cfg.cap_mib, cuda)
    pin = B.pinned_apps(*apps.shape[:2])
    pin[...] = apps
    host = B.simulate_batch_host(pin, POLICIES, cfg.cap_mib, chunk_traces=1536)
    np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
    np.testing.assert_array_equal(host.end, dres.ticks("end"))
    np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))
    assert floats_equal(host.mem_pct, dres.mem_pct.cpu().numpy())
    assert floats_equal(host.dev_pct, dres.dev_pct.cpu().numpy())


@pytest.mark.parametrize("case", ["overflow", "busy16", "end16", "c5", "long", "c3", "grant_only"])
def test_host_pipeline_cases(case, cuda):
    """The host pipeline moves end and busy ticks as u16 (K5 pack16) and
    derives the grants on the host (end - busy); a chunk they do not fit
    exactly (a busy step >= 0xFFFF ticks, "busy16", or an end tick >= 0xFFFF,
    "end16", beside chunks with apps that request no memory) and traces
    with a tick overflow are re-simulated with u32 ticks; multi-device, long
    (warp-kernel) traces and a grant-only request follow the same contract."""
    rng = np.random.default_rng(21)
    caps = (184_320,)
    if case in ("busy16", "end16"):
        # chunks of 128 traces: chunk 1 holds busy steps of 0xFFFF and more
        # (or ends past 0xFFFF), chunk 3 apps without a memory request
        # (busy16 = 0xFFFF marks them)
        cfg = CONFIGS["C2"]
        apps = as_u32x4(generate(cfg.gen, 0, 700))
        if case == "busy16":
            apps[130, 5, 2] = 0xFFFF
            apps[131, 7, 2] = 0x10000
        else:
            apps[130, 5, 0] = 0xFFFF - apps[130, 5, 2]
            apps[130, 5, 1] = 1
            apps[200:202, :, 0] += 100_000
        apps[400:402, ::3, 1] = 0
    elif case == "overflow":
        n, nt = 40, 300
        apps = np.zeros((nt, n, 4), dtype=np.uint32)
        apps[:, :, 0] = rng.integers(0, 1000, (nt, n))
        apps[:, :, 1] = rng.integers(1, 60_000, (nt, n))
        apps[:, :, 2] = rng.integers(1, 50, (nt, n))
        apps[5:9, :, 2] = np.uint32(0x7FFFFFF)   # sum(busy) past 2^32 ticks
        apps[40:42, 0, 0] = np.uint32(0xFFFFFF00)
    elif case == "c5":
        cfg = CONFIGS["C5"]
        apps, caps = as_u32x4(generate(cfg.gen, 0, 700)), cfg.cap_mib
    elif case == "long":
        cfg = CONFIGS["C4"]
        apps, caps = as_u32x4(generate(cfg.gen, 0, 400)), cfg.cap_mib
    elif case == "c3":   # 256-app traces: the octet kernel behind the pipeline
        cfg = CONFIGS["C3"]
        apps, caps = as_u32x4(generate(cfg.gen, 0, 300)), cfg.cap_mib
    else:
        apps = as_u32x4(generate(CONFIGS["C2"].gen, 0, 900))
    dres = run(apps, POLICIES, caps, cuda)
    pin = B.pinned_apps(*apps.shape[:2])
    pin[...] = apps
    want_end = case != "grant_only"
    out = B.HostBuffers(4, apps.shape[0], apps.shape[1], len(caps))
    if not want_end:
        out.end = None
    host = B.simulate_batch_host(pin, POLICIES, caps, chunk_traces=128, out=out)
    np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
    if want_end:
        np.testing.assert_array_equal(host.end, dres.ticks("end"))
    np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))
    if case == "overflow":
        assert (dres.stats()["status"] & 1).any()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_host_pipeline_direct_policies(k, cuda, monkeypatch):
    """SGPU_DIRECT_POLS=k: the first k policies cross PCIe as u32 grant + end
    rows, the others as pack16; with chunks that fit 16 bits, a chunk that
    does not, apps without a request and a tick overflow."""
    monkeypatch.setenv("SGPU_DIRECT_POLS", str(k))
    apps = as_u32x4(generate(CONFIGS["C2"].gen, 0, 700))
    apps[200:202, :, 0] += 100_000          # chunk 1: ends beyond 16 bits
    apps[400:402, ::3, 1] = 0               # apps without a memory request
    apps[600, :, 2] = np.uint32(0x7FFFFFF)  # sum(busy) past 2^32 ticks
    dres = run(apps, POLICIES, (184_320,), cuda)
    pin = B.pinned_apps(*apps.shape[:2])
    pin[...] = apps
    for _ in range(2):
        host = B.simulate_batch_host(pin, POLICIES, (184_320,), chunk_traces=128)
        np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
        np.testing.assert_array_equal(host.end, dres.ticks("end"))
        np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))


def test_host_pipeline_transfer_format_switch(cuda):
    """The pipeline's transfer format follows the data: C4-shaped traces
    (ticks beyond 16 bits in every chunk) make the next call of that shape
    copy u32 end ticks, a batch of the same shape that fits 16 bits switches
    it back; every call is bit-exact with the device path."""
    wide = as_u32x4(generate(CONFIGS["C4"].gen, 0, 600))
    g = dataclasses.replace(CONFIGS["C4"].gen, arr_hi=2000, busy_hi=300, mem_lo=1000, mem_hi=30_000)
    narrow = as_u32x4(generate(g, 0, 600))
    for apps in (wide, wide, narrow, narrow, wide):
        dres = run(apps, POLICIES, (184_320,), cuda)
        pin = B.pinned_apps(*apps.shape[:2])
        pin[...] = apps
        host = B.simulate_batch_host(pin, POLICIES, (184_320,), chunk_traces=128)
        np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
        np.testing.assert_array_equal(host.end, dres.ticks("end"))
        np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))


@pytest.mark.parametrize("thr", [1, 3])
def test_host_pipeline_threads(thr, cuda, monkeypatch):
    """One and three host threads deriving grants, ragged last chunk, two
    calls in a row (the pinned busy16 staging and streams persist)."""
    monkeypatch.setenv("SGPU_HOST_THREADS", str(thr))
    cfg = CONFIGS["C2"]
    apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=77), 0, 3001))
    dres = run(apps, POLICIES, cfg.cap_mib, cuda)
    pin = B.pinned_apps(*apps.shape[:2])
    pin[...] = apps
    for _ in range(2):
        host = B.simulate_batch_host(pin, POLICIES, cfg.cap_mib, chunk_traces=500)
        np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
        np.testing.assert_array_equal(host.end, dres.ticks("end"))
        np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))
        assert host.h2d_bytes == apps.nbytes
        # end + busy ticks as u16 (K5 pack16), one overflow flag per chunk
        assert host.d2h_bytes == 5 * apps.size // 2 + 4 * 7 + sum(
            a.nbytes for a in (host.stats, host.mem_pct, host.dev_pct, host.speedup))


def test_work_counters_across_streams_and_sizes(cuda):
    """Dynamic scheduling hands out work items from one counter per stream,
    reset by the last warp of each launch: many launches of varying size,
    interleaved over several streams (and both engines, via the fixture),
    must each cover every trace exactly once."""
    cfg = CONFIGS["C2"]
    streams = [torch.cuda.Stream() for _ in range(3)]
    rng = np.random.default_rng(11)
    for i in range(24):
        n = int(rng.choice([1, 7, 33, 100, 257, 1000]))
        apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=200 + i), 0, n))
        s = streams[i % 3]
        with torch.cuda.stream(s):
            res = B.simulate_batch(to_dev(apps, cuda), ("fifo", "pmmu"), cfg.cap_mib, stream=s)
        s.synchronize()
        for pi, pol in enumerate(res.policies):
            g, e, st = O.simulate_burst(apps, cfg.cap_mib, pol.value)
            np.testing.assert_array_equal(res.ticks("end")[pi].reshape(e.shape), e, err_msg=f"launch {i}")
            np.testing.assert_array_equal(res.stats()[pi].view(np.uint8), st.view(np.uint8))


def test_work_counters_concurrent_host_threads(cuda):
    """Launches from several host threads at once, two of them sharing one
    stream (whose launches the stream orders, so its counter is back at zero
    when each starts): every launch covers each of its traces exactly once."""
    import threading
    cfg = CONFIGS["C2"]
    shared = torch.cuda.Stream()
    streams = [shared, shared, torch.cuda.Stream(), torch.cuda.Stream()]
    cases = []
    for i in range(4):
        apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=300 + i), 0, 500 + 37 * i))
        cases.append((apps, to_dev(apps, cuda)))
    results = [[] for _ in range(4)]

    def work(k):
        torch.cuda.set_device(cuda)
        for _ in range(6):
            with torch.cuda.stream(streams[k]):
                r = B.simulate_batch(cases[k][1], ("mmu", "pfifo"), cfg.cap_mib, stream=streams[k])
            streams[k].synchronize()
            results[k].append((r.ticks("end"), r.stats()))

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(4):
        apps = cases[k][0]
        for pi, pol in enumerate(("mmu", "pfifo")):
            _, e, st = O.simulate_burst(apps, cfg.cap_mib, pol)
            for end, stats in results[k]:
                np.testing.assert_array_equal(end[pi].reshape(e.shape), e)
                np.testing.assert_array_equal(stats[pi].view(np.uint8), st.view(np.uint8))


@pytest.mark.parametrize("n", [24, 64, 128])
def test_many_priority_classes(n, cuda):
    """More distinct priorities per trace than the lane kernel keeps class
    sets for (8): those traces take the in-kernel exact fallback; priorities
    up to 255 exercise the warp kernel's full presence set."""
    rng = np.random.default_rng(n)
    apps = np.zeros((96, n, 4), np.uint32)
    apps[..., 0] = rng.integers(0, 200, apps.shape[:2])
    apps[..., 1] = rng.integers(1, 30_000, apps.shape[:2])
    apps[..., 2] = rng.integers(1, 100, apps.shape[:2])
    levels = rng.choice([4, 9, 16, 256], size=96)
    apps[..., 3] = (rng.integers(0, 1 << 30, apps.shape[:2]) % levels[:, None]).astype(np.uint32)
    check_against_oracle(apps, (60_000,), cuda)


@pytest.mark.parametrize("pols", [("mmu",), ("fifo", "pfifo"), ("mmu", "pfifo", "pmmu")])
def test_host_pipeline_policy_subsets(pols, cuda):
    """Host-buffer pipeline with 1-3 policies against the device path."""
    cfg = CONFIGS["C2"]
    apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=41), 0, 3000))
    dres = run(apps, pols, cfg.cap_mib, cuda)
    pin = B.pinned_apps(*apps.shape[:2])
    pin[...] = apps
    host = B.simulate_batch_host(pin, pols, cfg.cap_mib, chunk_traces=700)
    np.testing.assert_array_equal(host.grant, dres.ticks("grant"))
    np.testing.assert_array_equal(host.end, dres.ticks("end"))
    np.testing.assert_array_equal(host.stats.view(np.uint8), dres.stats().view(np.uint8))


@pytest.mark.parametrize("tick_scale", [1, 256])
def test_cuda_graph_replay(tick_scale, cuda):
    """K1 launched inside a captured CUDA graph and replayed on new inputs:
    the work counters reset at the end of every launch, so each replay
    covers every trace again.  At tick scale 256 the traces need 64-bit
    event keys: the retry launch and its graph-owned deferred list run in
    every replay."""
    cfg = CONFIGS["C2"]
    cfg = dataclasses.replace(cfg, gen=dataclasses.replace(
        cfg.gen, arr_hi=4095 * tick_scale, busy_hi=2048 * tick_scale, busy_lo=tick_scale))
    n = 5000
    apps_t = B.generate_traces(cfg.gen, 0, n, device=0)
    B.simulate_batch(apps_t, POLICIES, cfg.cap_mib)  # warm-up: kernel attributes, counter pool
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res = B.simulate_batch(apps_t, POLICIES, cfg.cap_mib, stream=s)
    for k in range(3):
        fresh = B.generate_traces(dataclasses.replace(cfg.gen, seed=900 + k), 0, n, device=0)
        apps_t.copy_(fresh)
        g.replay()
        torch.cuda.synchronize()
        apps = apps_t.cpu().numpy().view(np.uint32)
        st = res.stats()
        for pi, pol in enumerate(res.policies):
            gr, e, sref = O.simulate_burst(apps, cfg.cap_mib, pol.value)
            np.testing.assert_array_equal(res.ticks("end")[pi].reshape(e.shape), e, err_msg=f"replay {k}")
            np.testing.assert_array_equal(st[pi].view(np.uint8), sref.view(np.uint8))


@pytest.mark.parametrize("k1", ["octet", "lane256"])
def test_octet_kernel_graph_replay(k1, cuda, monkeypatch):
    """The 256-app kernels (C3-shaped traces) inside a captured CUDA graph,
    replayed on fresh inputs: each replay simulates the whole batch (lane256:
    its global staging scratch is a graph allocation)."""
    monkeypatch.setenv("SGPU_K1", k1)
    cfg = CONFIGS["C3"]
    n = 600
    apps_t = B.generate_traces(cfg.gen, 0, n, device=0)
    B.simulate_batch(apps_t, cfg.policies, cfg.cap_mib)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res = B.simulate_batch(apps_t, cfg.policies, cfg.cap_mib, stream=s)
    for k in range(2):
        apps_t.copy_(B.generate_traces(dataclasses.replace(cfg.gen, seed=700 + k), 0, n, device=0))
        g.replay()
        torch.cuda.synchronize()
        apps = apps_t.cpu().numpy().view(np.uint32)
        st = res.stats()
        for pi, pol in enumerate(res.policies):
            gr, e, sref = O.simulate_burst(apps, cfg.cap_mib, pol.value)
            np.testing.assert_array_equal(res.ticks("grant")[pi].reshape(gr.shape), gr, err_msg=f"replay {k}")
            np.testing.assert_array_equal(res.ticks("end")[pi].reshape(e.shape), e, err_msg=f"replay {k}")
            np.testing.assert_array_equal(st[pi].view(np.uint8), sref.view(np.uint8))


def test_cuda_graph_replay_beside_its_capture_stream(cuda):
    """A captured K1 launch owns its work counters and deferred list (graph
    allocations, zeroed by a memset node at every replay), so replays on
    another stream interleaved with new K1 work on the capturing stream each
    simulate their whole batch.  (torch's blocking streams serialise the two
    here; the separation is by construction, sgpu_sim.cu work_counters.)"""
    cfg = CONFIGS["C2"]
    n = 20000
    a_graph = B.generate_traces(cfg.gen, 0, n, device=0)
    a_live = B.generate_traces(dataclasses.replace(cfg.gen, seed=77), 0, n, device=0)
    B.simulate_batch(a_graph, POLICIES, cfg.cap_mib)
    torch.cuda.synchronize()
    s, t = torch.cuda.Stream(), torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res_g = B.simulate_batch(a_graph, POLICIES, cfg.cap_mib, stream=s)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(t):
            g.replay()
        res_live = B.simulate_batch(a_live, POLICIES, cfg.cap_mib, stream=s)
    torch.cuda.synchronize()
    for apps_t, res in ((a_graph, res_g), (a_live, res_live)):
        apps = apps_t.cpu().numpy().view(np.uint32)
        for pi, pol in enumerate(res.policies):
            _, e, sref = O.simulate_burst(apps, cfg.cap_mib, pol.value)
            np.testing.assert_array_equal(res.ticks("end")[pi].reshape(e.shape), e)
            np.testing.assert_array_equal(res.stats()[pi].view(np.uint8), sref.view(np.uint8))


def test_bad_device_index_flagged(cuda):
    """ndev > 1: an app whose device index is >= ndev runs on device 0 and
    sets SG_ST_BAD_DEVICE on every record of its trace (both engines, the
    oracle restates the same; check_against_oracle compares status)."""
    cfg = CONFIGS["C5"]
    apps = as_u32x4(generate(cfg.gen, 0, 64)).copy()
    apps[5, 7, 3] = (apps[5, 7, 3] & 0xFF) | (200 << 8)
    apps[9, 0, 3] = (apps[9, 0, 3] & 0xFF) | (8 << 8)
    res = check_against_oracle(apps, cfg.cap_mib, cuda)
    st = res.stats()
    bad = (st["status"] & 0x4) != 0
    assert bad[:, [5, 9], :].all()
    assert bad.sum() == 2 * len(POLICIES) * cfg.ndev


def test_ragged_graph_capture(cuda):
    """A CSR (ragged) batch with apps_total / max_apps given makes no host
    read of device memory, so it captures into a CUDA graph and replays."""
    rng = np.random.default_rng(21)
    lens = rng.integers(0, 70, 500)
    total = int(lens.sum())
    flat = as_u32x4(generate(GenParams(seed=8, apps_per_trace=total), 0, 1))[0]
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    a_t = to_dev(flat, cuda)
    o_t = torch.from_numpy(offs).to(cuda)
    kw = dict(trace_offsets=o_t, apps_total=total, max_apps=int(lens.max()))
    B.simulate_batch(a_t, POLICIES, 184_320, **kw)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        res = B.simulate_batch(a_t, POLICIES, 184_320, stream=s, **kw)
    res.end.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    for pi, pol in enumerate(res.policies):
        for t in range(0, len(lens), 7):
            a = flat[offs[t]:offs[t + 1]][None]
            _, ee, ss = O.simulate_burst(a, (184_320,), pol.value)
            np.testing.assert_array_equal(res.ticks("end")[pi][offs[t]:offs[t + 1]], ee[0])
            assert res.stats()[pi][t, 0]["makespan"] == ss[0, 0]["makespan"]


def test_device_info_reports_residency(cuda):
    """sg_device_info: SMs and the lane kernel's resident warps per SM (C2
    shape), the residency the persistent grid is sized for."""
    import ctypes
    from paper_1712_04495_b200 import _lib
    sms, wps = ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(_lib.lib().sg_device_info(0, ctypes.byref(sms), ctypes.byref(wps)), "sg_device_info")
    assert sms.value == torch.cuda.get_device_properties(0).multi_processor_count
    assert 8 <= wps.value <= 64 and wps.value % 2 == 0


def test_criterion5_select_grants_full(cuda):
    """Acceptance criterion 5 at full size (test_acceptance.py:174-226): K4
    on all 100,000 queues x 4 policies (seed 20260823) in one launch equals
    the reference's select_grants everywhere (0 mismatches)."""
    from paper_1712_04495_b200.policy import select_grants_batch
    queues = criterion5_queues()
    qs, fr, kinds = [], [], []
    for sizes, prios, free in queues:
        for code in range(4):
            qs.append((sizes, prios))
            fr.append(free)
            kinds.append(code)
    got = select_grants_batch(qs, fr, kinds)
    flat = np.concatenate([g for g in got if len(g)])
    want = criterion5_flags()
    assert flat.shape == want.shape
    assert np.array_equal(flat, want), f"{int((flat != want).sum())} entries differ"


# ------------------------------------------------------------ step programs

def _program_batch(rng, n_traces, n, long_every=0, huge_every=0):
    """Random multi-phase programs (tests/test_proglanesim_host.py
    random_trace), n apps per trace, as one simulate_batch in step-program
    mode.  long_every: every k-th trace gets more steps than a lane slot
    holds; huge_every: every k-th trace has a cpu step near 2^32 ticks (time
    overflow: the warp engine's status flag)."""
    from test_proglanesim_host import random_trace
    steps, so, attr = [], [0], []
    per = []
    for t in range(n_traces):
        st, first, prio = random_trace(rng, n, max_phases=4 if not (long_every and t % long_every == 0) else 40)
        if huge_every and t % huge_every == 0:
            st = [(0, 0, 0xFFFFFFF0), (2, 0, 100)] + st   # app 0 runs past 2^32 - 2 ticks
            first = [0] + [f + 2 for f in first[1:]]
        base = len(steps)
        steps.extend(st)
        so.extend(base + f for f in first[1:])
        attr.append(prio)
        per.append((st, first, prio))
    steps_a = np.array(steps, dtype=B.STEP_DTYPE)
    return steps_a, np.array(so, np.uint32), np.array(attr, np.uint32), per


@pytest.mark.parametrize("n,long_every,huge_every", [(5, 0, 0), (12, 7, 0), (16, 0, 11), (17, 0, 0), (32, 5, 9)])
def test_program_batches_against_oracle(n, long_every, huge_every, cuda, engine):
    """Step-program batches on both engines (auto: the K1 v6 lane-per-
    simulation kernel, with its in-kernel warp fallback for traces longer
    than a slot and for time overflows; warp: K1 v3) against the oracle's
    program mode, every output bit-exact."""
    rng = np.random.default_rng(n * 7 + long_every)
    nt = 300
    steps, so, attr, per = _program_batch(rng, nt, n, long_every, huge_every)
    apps = np.zeros((nt, n, 4), np.uint32)
    apps[..., 3] = attr
    cap = 700
    res = B.simulate_batch(to_dev(apps, cuda), POLICIES, cap,
                           steps=torch.from_numpy(steps.view(np.int32).reshape(-1, 4).copy()).to(cuda),
                           step_offsets=torch.from_numpy(so.view(np.int32).copy()).to(cuda))
    torch.cuda.synchronize()
    st = res.stats()
    grant = res.ticks("grant").reshape(4, nt, n)
    end = res.ticks("end").reshape(4, nt, n)
    spd = res.speedup.cpu().numpy()
    for pi, pol in enumerate(POLICIES):
        for t, (s_, first, prio) in enumerate(per):
            if huge_every and t % huge_every == 0:
                # times past 2^32 - 2 ticks: flagged (the drop-in then raises)
                assert st[pi, t, 0]["status"] & 1, (pol, t)
                continue
            sa = np.array(s_, dtype=O.STEP_DTYPE) if s_ else np.zeros(0, O.STEP_DTYPE)
            g, e, s = O.simulate_program(sa, np.array(first, np.uint32), np.array(prio, np.uint32), cap, pol)
            np.testing.assert_array_equal(grant[pi, t], g, err_msg=f"grant {pol} {t}")
            np.testing.assert_array_equal(end[pi, t], e, err_msg=f"end {pol} {t}")
            assert st[pi, t, 0].tobytes() == s[0].tobytes(), (pol, t, st[pi, t, 0], s[0])
            seq = sum(d for op, _, d in s_ if op in (0, 2))
            want = O.speedup_from(np.array([seq]), s["makespan"][:1], np.array([n]))
            assert floats_equal(spd[pi, t, :1], want), (pol, t)
