"""Shared helpers for the parity tests."""

import os

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
