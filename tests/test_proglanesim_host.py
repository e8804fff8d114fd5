"""The K1 v6 step-program lane simulator (csrc/sgpu_proglanesim.cuh,
ProgLaneSim) compiled for the HOST with g++ (tests/proglanesim_host.cpp) and
checked against the oracle's program mode (oracle/sim_oracle.c): the
kernel's decision logic for multi-phase profiles (several allocs per app,
memory held across cpu steps, repeated waits, frees without allocs, zero
durations, priorities) on CPU, bit for bit.  No GPU needed; the -m gpu
tests run the same logic inside the kernel."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from util import POLICIES

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "proglanesim_host.cpp")
CODES = {"fifo": 0, "mmu": 1, "pfifo": 2, "pmmu": 3}
STAT_FIELDS = ("makespan", "busy", "mem_integral", "grants", "pops", "max_holders", "unfinished")


@pytest.fixture(scope="module")
def proglane(tmp_path_factory):
    cxx = shutil.which("g++") or shutil.which("c++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    exe = str(tmp_path_factory.mktemp("proglane") / "proglanesim_host")
    subprocess.run([cxx, "-O2", "-std=c++17", "-Wall", "-Wno-unknown-pragmas", "-o", exe, SRC],
                   check=True)
    return exe


def random_trace(rng, n, max_phases=4, free_prob=0.85):
    """Random multi-phase programs in the reference's flattening order
    (cpu, alloc, busy, free per phase, zero fields skipped), like the
    golden 'random programs' scenarios (tests/golden/make_golden.py)."""
    steps, first, prio = [], [], []
    for _ in range(n):
        first.append(len(steps))
        held = 0
        for _ in range(rng.integers(1, max_phases + 1)):
            cpu = int(rng.choice([0, 0, 1, 3, 7, 12]))
            alloc = int(rng.choice([0, 50, 120, 300]))
            busy = int(rng.choice([0, 2, 5, 9]))
            if cpu:
                steps.append((0, 0, cpu))
            if alloc:
                steps.append((1, alloc, 0))
                held += alloc
            if busy:
                steps.append((2, 0, busy))
        if held and rng.random() < free_prob:
            steps.append((3, held, 0))
        prio.append(int(rng.integers(0, 4)))
    first.append(len(steps))
    return steps, first, prio


def run_host(exe, cases, pol, cap):
    lines = []
    for steps, first, prio in cases:
        lines.append(f"{len(prio)} {CODES[pol]} {cap} {len(steps)}")
        lines.append(" ".join(map(str, first)))
        lines.append(" ".join(map(str, prio)) if prio else "")
        lines.extend(f"{op} {mib} {dur}" for op, mib, dur in steps)
    out = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True).stdout.split("\n")
    return [list(map(int, o.split())) for o in out[:len(cases)]]


def check(exe, cases, pol, cap):
    res = run_host(exe, cases, pol, cap)
    for (steps, first, prio), v in zip(cases, res):
        assert v[0] == 1, "lane declined a trace within its limits"
        st = np.array([(op, mib, dur) for op, mib, dur in steps] or [(0, 0, 0)], dtype=O.STEP_DTYPE)
        if not steps:
            st = st[:0]
        g, e, s = O.simulate_program(st, np.array(first, np.uint32), np.array(prio, np.uint32), cap, pol)
        assert v[1:8] == [int(s[0][f]) for f in STAT_FIELDS], (pol, v[1:8], s[0])
        ticks = np.array(v[8:], dtype=np.uint64)
        np.testing.assert_array_equal(ticks[0::2], g.astype(np.uint64), err_msg=f"grant {pol}")
        np.testing.assert_array_equal(ticks[1::2], e.astype(np.uint64), err_msg=f"end {pol}")


@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("n", [1, 5, 12, 16, 17, 32])
def test_random_programs(proglane, pol, n):
    rng = np.random.default_rng(100 + n)
    cases = [random_trace(rng, n) for _ in range(60)]
    for cap in (400, 1000):
        check(proglane, cases, pol, cap)


@pytest.mark.parametrize("pol", POLICIES)
def test_builtin_profiles_workload(proglane, pol):
    """The reference's builtin ara / mummer / blast profiles
    (memshare/harness.py:65-83) on tight and loose devices, with seeded
    start offsets, as step programs on the tick grid."""
    from paper_1712_04495_b200 import harness as H
    P = H.builtin_profiles()
    hi = H.AppProfile("mummer-like", P["mummer-like"].phases, priority=2)
    spec = H.WorkloadSpec(instances=[P["ara-like"]] * 4 + [hi] * 4 + [P["blast-like"]] * 4,
                          time_scale=1000.0 / 1024.0)
    enc = H.encode_spec(spec)
    rng = np.random.default_rng(3)
    cases = []
    for _ in range(20):
        steps, first = [], []
        for i in range(len(enc.attr)):
            first.append(len(steps))
            steps.append((0, 0, int(rng.integers(0, 2048))))
            for s in enc.steps[enc.step_offsets[i]:enc.step_offsets[i + 1]]:
                steps.append((int(s["op"]), int(s["mib"]), int(s["dur"])))
        first.append(len(steps))
        cases.append((steps, first, [int(a) for a in enc.attr]))
    for cap in (2400, 4799):
        check(proglane, cases, pol, cap)


@pytest.mark.parametrize("pol", POLICIES)
def test_edge_programs(proglane, pol):
    """Empty programs, a free without an alloc, an oversize request that
    waits forever, zero-length cpu / busy steps, an app that allocates twice
    and waits twice."""
    cases = [
        ([], [0, 0, 0], [0, 0]),
        ([(3, 100, 0)], [0, 1], [1]),
        ([(1, 5000, 0), (2, 0, 3), (3, 5000, 0), (1, 10, 0), (3, 10, 0)], [0, 3, 5], [0, 2]),
        ([(0, 0, 0), (1, 300, 0), (2, 0, 0), (3, 300, 0), (1, 800, 0), (2, 0, 4), (3, 800, 0),
          (1, 500, 0), (0, 0, 2), (1, 400, 0), (2, 0, 1), (3, 900, 0)], [0, 4, 7, 12], [1, 3, 3]),
    ]
    check(proglane, cases, pol, 1000)
