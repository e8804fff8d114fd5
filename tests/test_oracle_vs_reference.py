"""Live cross-check of the oracle against the REAL reference simulator on
fresh random inputs (only where /root/reference exists, i.e. the build
container; the GPU box relies on the committed golden fixtures)."""

import dataclasses

import numpy as np
import pytest

import refsim
from oracle import oracle as O
from paper_1712_04495_b200.tracegen import CONFIGS, GenParams, as_u32x4, generate
from util import POLICIES

pytestmark = pytest.mark.skipif(not refsim.available(), reason="reference tree not present")


@pytest.mark.parametrize("pol", POLICIES)
def test_random_bursty_traces(pol):
    g = GenParams(seed=77, apps_per_trace=24, arr_hi=40, mem_lo=50, mem_hi=900, busy_lo=1,
                  busy_hi=12, prio_levels=3)
    apps = as_u32x4(generate(g, 0, 60))
    apps[::7, :, 2] = 0          # busy 0: free right after the grant
    apps[::5, ::3, 0] = 0        # arrival 0: request during the initial pops
    apps[::9, ::4, 1] = 0        # mem 0: no alloc / free
    apps[::11, 1, 1] = 5000      # larger than the device: stuck forever
    gg, ee, st = O.simulate_burst(apps, (2000,), pol)
    ms, mp, dp = O.pct_from_stats(st[:, 0], 2000)
    for t in range(len(apps)):
        r = refsim.run_burst(apps[t], 2000, pol)
        assert [None if x == 0xFFFFFFFF else int(x) for x in gg[t]] == r["grant"]
        assert [None if x == 0xFFFFFFFF else int(x) for x in ee[t]] == r["end"]
        assert st[t, 0]["makespan"] == r["T"]
        assert (ms[t], mp[t], dp[t]) == (r["makespan_ms"], r["mem_pct"], r["dev_pct"])
        assert st[t, 0]["max_holders"] == r["max_holders"]
        assert st[t, 0]["unfinished"] == r["unfinished"]


def test_config_shapes_fresh_seed():
    for cname, nt in (("C2", 10), ("C4", 6), ("C3", 2)):
        cfg = CONFIGS[cname]
        apps = as_u32x4(generate(dataclasses.replace(cfg.gen, seed=4242), 0, nt))
        for pol in cfg.policies:
            gg, ee, st = O.simulate_burst(apps, cfg.cap_mib, pol)
            for t in range(nt):
                r = refsim.run_burst(apps[t], cfg.cap_mib[0], pol)
                assert st[t, 0]["makespan"] == r["T"] and st[t, 0]["grants"] == r["grants"]
                assert [None if x == 0xFFFFFFFF else int(x) for x in ee[t]] == r["end"]
