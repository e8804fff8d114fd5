"""Shared helpers for the parity tests."""

import os
import random

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
POLICIES = ("fifo", "mmu", "pfifo", "pmmu")
NEVER = 0xFFFFFFFF


_CACHE = {}


def golden(name):
    """All arrays of a golden .npz, decompressed once."""
    if name not in _CACHE:
        with np.load(os.path.join(GOLDEN, name)) as z:
            _CACHE[name] = {k: z[k] for k in z.files}
    return _CACHE[name]


def floats_equal(a, b):
    """Bit-exact float64 equality (NaN-free inputs)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def criterion5_queues(seed: int = 20260823, trials: int = 100_000):
    """The reference's acceptance criterion 5 queue stream, draw for draw
    (pkg/tests/test_acceptance.py:211-219): n U[0,8], sizes U[1,2000],
    prios U[0,3], free U[0,6000]; each queue is evaluated under the four
    policies (golden/ref_criterion5.npz holds the reference's answers)."""
    rng = random.Random(seed)
    out = []
    for _ in range(trials):
        n = rng.randint(0, 8)
        sizes = [rng.randint(1, 2000) for _ in range(n)]
        prios = [rng.randint(0, 3) for _ in range(n)]
        free = rng.randint(0, 6000)
        out.append((sizes, prios, free))
    return out


def criterion5_flags():
    """Reference select_grants flags of criterion 5, queue-major, then
    policy (fifo, mmu, pfifo, pmmu), then entry."""
    z = golden("ref_criterion5.npz")
    return np.unpackbits(z["granted_bits"])[:int(z["n_flags"][0])].astype(bool)


def brute_select(sizes, prios, free, code):
    """The reference test's brute-force oracle (test_acceptance.py:177-199):
    FIFO = longest fitting prefix; MMU = the feasible subset that is largest
    in earlier-index-dominates order; priority kinds = the same on the top
    class."""
    if code >= 2:
        if not sizes:
            return []
        top = max(prios)
        idx = [i for i, p in enumerate(prios) if p == top]
        sub = brute_select([sizes[i] for i in idx], [0] * len(idx), free, code - 2)
        return [idx[i] for i in sub]
    n = len(sizes)
    if n == 0:
        return []
    if code == 0:
        k = int(np.searchsorted(np.cumsum(sizes), free, side="right"))
        return list(range(k))
    masks = ((np.arange(1 << n)[:, None] >> np.arange(n)) & 1).astype(np.int64)
    pref = masks @ (1 << np.arange(n)[::-1])
    feasible = np.flatnonzero(masks @ np.asarray(sizes) <= free)
    win = int(feasible[np.argmax(pref[feasible])])
    return [i for i in range(n) if win >> i & 1]
