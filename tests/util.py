"""Shared helpers for the parity tests."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
POLICIES = ("fifo", "mmu", "pfifo", "pmmu")
NEVER = 0xFFFFFFFF


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def floats_equal(a, b):
    """Bit-exact float64 equality (NaN-free inputs)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
