"""The K1 v5 per-lane simulator (csrc/sgpu_lanesim.cuh, LaneSim) compiled
for the HOST with g++ (tests/lanesim_host.cpp) and checked against the
oracle: the exact decision logic the kernel runs (arrival stream, virtual
counters, 32- and 64-bit event keys, the two-level heap, wake FIFO drain,
incremental select_grants steps over the fit table, class sets) on CPU,
bit for bit, including edge shapes (zero fields, ties, stuck requests,
eight priority classes).  No GPU needed; the -m gpu tests run the same
logic inside the kernel."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate
from util import POLICIES

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lanesim_host.cpp")
HDR = os.path.join(os.path.dirname(HERE), "paper_1712_04495_b200", "csrc", "sgpu_lanesim.cuh")
CODES = {"fifo": 0, "mmu": 1, "pfifo": 2, "pmmu": 3}
STAT_FIELDS = ("makespan", "busy", "mem_integral", "grants", "pops", "max_holders", "unfinished")


@pytest.fixture(scope="module")
def lanesim(tmp_path_factory):
    cxx = shutil.which("g++") or shutil.which("c++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    exe = str(tmp_path_factory.mktemp("lanesim") / "lanesim_host")
    subprocess.run([cxx, "-O2", "-std=c++17", "-Wall", "-Wno-unknown-pragmas", "-o", exe, SRC],
                   check=True)
    return exe


def run_host(exe, apps, pol, cap, keys):
    """keys: 1 / True = 32-bit, 0 / False = 64-bit (main-pass heap),
    2 = 64-bit (retry-pass heap)."""
    lines = []
    for tr in apps:
        lines.append(f"{len(tr)} {CODES[pol]} {cap} {int(keys)}")
        lines.extend(" ".join(str(int(x)) for x in (r[0], r[1], r[2], r[3] & 0xFF)) for r in tr)
    out = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True).stdout.split("\n")
    return [list(map(int, o.split())) for o in out[:len(apps)]]


def check(exe, apps, pol, cap, narrow, min_checked):
    g, e, st = O.simulate_burst(apps, (cap,), pol)
    res = run_host(exe, apps, pol, cap, narrow)
    checked = 0
    for t, v in enumerate(res):
        if v[0] == 0:       # lane path declined (capacity): the kernel's warp fallback runs it
            continue
        checked += 1
        stats = v[1:8]
        ref = [int(st[t][0][f]) for f in STAT_FIELDS]
        assert stats == ref, (pol, narrow, t, stats, ref)
        ticks = np.array(v[8:], dtype=np.uint64)
        np.testing.assert_array_equal(ticks[0::2], g[t].astype(np.uint64), err_msg=f"grant {pol} {t}")
        np.testing.assert_array_equal(ticks[1::2], e[t].astype(np.uint64), err_msg=f"end {pol} {t}")
    assert checked >= min_checked, (checked, len(res))
    return checked


def narrow_lim(n):
    """LaneKey<K, true>::LIM: every event time of a 32-bit-key lane stays below it."""
    logn = 5 if n <= 32 else 6 if n <= 64 else 7 if n <= 128 else 8
    return (1 << (31 - 2 * logn)) - 1


def narrow_mask(apps, n):
    """Per trace, the kernel's staging rule for 32-bit keys (sgpu_lane.cu
    stage_trace): arrival max + busy sum below LaneKey::LIM."""
    a = apps.astype(np.uint64)
    return a[..., 0].max(axis=1) + a[..., 2].sum(axis=1) < narrow_lim(n)


def narrow_ok(apps, n):
    return bool(np.all(narrow_mask(apps, n)))


WIDE, NARROW, WIDE_RETRY = 0, 1, 2   # lanesim_host key modes


@pytest.mark.parametrize("pol", POLICIES)
def test_lanesim_c2_traces(lanesim, pol):
    cfg = CONFIGS["C2"]
    apps = as_u32x4(generate(cfg.gen, 123_456, 150))
    assert narrow_ok(apps, 64)
    check(lanesim, apps, pol, cfg.cap_mib[0], NARROW, 150)
    # 64-bit keys: the main pass's 10-slot heap declines the busiest traces
    # to the retry pass, whose 20-slot heap takes them all
    check(lanesim, apps, pol, cfg.cap_mib[0], WIDE, 1)
    check(lanesim, apps, pol, cfg.cap_mib[0], WIDE_RETRY, 150)


@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("n", [32, 64, 128])
def test_lanesim_narrow_limit_boundary(lanesim, pol, n):
    """A holder ending near LaneKey::LIM with a waiter behind it whose busy
    step is 0 or 1 (the waiter's wake-up is the last event): every trace the
    staging rule admits to 32-bit keys, up to the tightest one (arrival max
    + busy sum = LIM - 1), matches the oracle; 64-bit keys take them all."""
    lim = narrow_lim(n)
    traces = []
    for end in range(lim - 5, lim + 2):
        for wb in (0, 1):
            tr = np.zeros((n, 4), np.uint32)
            tr[0] = (1000, 10, end - 1000, 0)   # holder: the whole device (busy < 2^21)
            tr[1] = (1001, 10, wb, 0)           # waiter, granted at the holder's end
            traces.append(tr)
    apps = np.stack(traces)
    ok = narrow_mask(apps, n)
    a = apps.astype(np.int64)
    assert (a[ok, :, 0].max(axis=1) + a[ok, :, 2].sum(axis=1)).max() == lim - 1
    check(lanesim, apps[ok], pol, 10, NARROW, int(ok.sum()))
    check(lanesim, apps, pol, 10, WIDE, len(apps))


@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("n", [32, 64, 128])
def test_lanesim_wide_heap_overflow(lanesim, pol, n):
    """11..20 busy apps at once overflow the main pass's 64-bit heap (10
    events) but not the retry pass's (20); more overflow both (the kernel's
    warp fallback runs those)."""
    rng = np.random.default_rng(900 + n)
    nt = 120
    apps = np.zeros((nt, n, 4), np.uint32)
    apps[..., 0] = rng.integers(0, 64, (nt, n))
    conc = np.linspace(6, 26, nt).astype(int)                 # target concurrency per trace
    apps[..., 1] = (1000 // conc)[:, None]
    apps[..., 2] = rng.integers(500, 900, (nt, n))
    apps[..., 3] = rng.integers(0, 3, (nt, n))
    wide = run_host(lanesim, apps, pol, 1000, WIDE)
    retry = run_host(lanesim, apps, pol, 1000, WIDE_RETRY)
    d_wide = np.array([v[0] == 0 for v in wide])
    d_retry = np.array([v[0] == 0 for v in retry])
    assert not np.any(d_retry & ~d_wide)                      # a bigger heap never declines more
    assert np.sum(d_wide & ~d_retry) >= 10 and np.sum(~d_wide) >= 10
    check(lanesim, apps, pol, 1000, WIDE, int((~d_wide).sum()))
    check(lanesim, apps, pol, 1000, WIDE_RETRY, int((~d_retry).sum()))


def random_edge_traces(rng, n_traces, n, cap):
    apps = np.zeros((n_traces, n, 4), np.uint32)
    # arrivals: many ties and zeros
    apps[..., 0] = rng.integers(0, 12, (n_traces, n)) * rng.integers(0, 2, (n_traces, n)) * 7
    apps[..., 1] = rng.integers(0, cap // 3, (n_traces, n))
    apps[..., 1] *= rng.random((n_traces, n)) > 0.1            # some mem = 0
    apps[..., 2] = rng.integers(0, 25, (n_traces, n))            # some busy = 0
    apps[..., 3] = rng.integers(0, 8, (n_traces, n))             # up to 8 classes
    stuck = rng.random((n_traces, n)) < 0.02                     # requests above capacity
    apps[..., 1][stuck] = cap + 1
    return apps


@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("n", [7, 32, 45, 64, 65, 100, 128])
def test_lanesim_edge_shapes(lanesim, pol, n):
    rng = np.random.default_rng(1000 + n)
    cap = 1000
    apps = random_edge_traces(rng, 300, n, cap)
    check(lanesim, apps, pol, cap, NARROW, 250)
    check(lanesim, apps, pol, cap, WIDE, 10 if n <= 64 else 0)
    check(lanesim, apps, pol, cap, WIDE_RETRY, 250)


@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("n", [64, 128])
def test_lanesim_near_capacity(lanesim, pol, n):
    """C4-like: requests of 1/4..1x capacity, long queues, head-of-line blocking."""
    rng = np.random.default_rng(77 + n)
    cap = 184_320
    apps = np.zeros((100, n, 4), np.uint32)
    apps[..., 0] = rng.integers(0, 8192, (100, n))
    apps[..., 1] = rng.integers(46_080, cap + 1, (100, n))
    apps[..., 2] = rng.integers(1, 2049, (100, n))
    apps[..., 3] = rng.integers(0, 4, (100, n))
    ok = narrow_mask(apps, n)
    if ok.any():
        check(lanesim, apps[ok], pol, cap, NARROW, int(ok.sum()))
    check(lanesim, apps, pol, cap, WIDE, 100)
    check(lanesim, apps, pol, cap, WIDE_RETRY, 100)


@pytest.mark.parametrize("pol", POLICIES)
def test_lanesim_c4_traces(lanesim, pol):
    cfg = CONFIGS["C4"]
    apps = as_u32x4(generate(cfg.gen, 7_000, 40))
    ok = narrow_mask(apps, 128)
    assert 0 < ok.sum() < len(ok)   # C4 mixes 32- and 64-bit-key traces
    check(lanesim, apps[ok], pol, cfg.cap_mib[0], NARROW, int(ok.sum()))
    check(lanesim, apps, pol, cfg.cap_mib[0], WIDE, 40)
    check(lanesim, apps, pol, cfg.cap_mib[0], WIDE_RETRY, 40)


@pytest.mark.parametrize("pol", POLICIES)
def test_lanesim_256_apps(lanesim, pol):
    """The global-table lane kernel's simulator at 129..256 apps (fit table
    of four words, u16 rank tables, 32-key three-level heap): C3 traces and
    edge shapes, both key widths, against the oracle."""
    cfg = CONFIGS["C3"]
    apps = as_u32x4(generate(cfg.gen, 31_000, 24))
    ok = narrow_mask(apps, 256)
    if ok.any():
        check(lanesim, apps[ok], pol, cfg.cap_mib[0], NARROW, int(ok.sum()))
    check(lanesim, apps, pol, cfg.cap_mib[0], WIDE, 20)
    rng = np.random.default_rng(256)
    for n in (129, 200, 256):
        edge = random_edge_traces(rng, 40, n, 1000)
        check(lanesim, edge, pol, 1000, WIDE, 30)
        okn = narrow_mask(edge, n)
        check(lanesim, edge[okn], pol, 1000, NARROW, int(okn.sum()) * 3 // 4)


def test_header_is_shared_with_the_kernel():
    """The kernel includes the same header the host test compiles."""
    src = open(os.path.join(os.path.dirname(HDR), "sgpu_lane.cu")).read()
    assert '#include "sgpu_lanesim.cuh"' in src
    assert "struct LaneSim" in open(HDR).read()
