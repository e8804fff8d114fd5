"""The ctypes binding INTEGRATION.md shows a memshare maintainer (the
reference-side stub for the C ABI) is executed as written, against the
in-tree libsgpu.so, and its outputs checked against the oracle."""

import ctypes
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1712_04495_b200 import _lib
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source():
    s = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    a = s.index("# memshare/_sgpu.py")
    return s[a:s.index("```", a)].replace('ctypes.CDLL("libsgpu.so")', f'ctypes.CDLL({_lib.LIB_PATH!r})')


def test_stub_struct_layouts_match_the_abi():
    ns = {}
    exec(stub_source().split("lib.sg_simulate_batch_host.argtypes")[0].replace(
        f'ctypes.CDLL({_lib.LIB_PATH!r})', "None"), ns)
    assert ctypes.sizeof(ns["sg_batch"]) == ctypes.sizeof(_lib.SgBatch)
    assert ctypes.sizeof(ns["sg_out"]) == ctypes.sizeof(_lib.SgOut)
    for name, _ in _lib.SgBatch._fields_:
        assert getattr(ns["sg_batch"], name).offset == getattr(_lib.SgBatch, name).offset, name


@pytest.mark.gpu
def test_stub_runs_bit_exact(cuda):
    ns = {}
    exec(stub_source(), ns)
    cfg = CONFIGS["C2"]
    apps = np.ascontiguousarray(as_u32x4(generate(cfg.gen, 77, 400)))
    for code, pol in enumerate(("fifo", "mmu", "pfifo", "pmmu")):
        g, e, st, sp = ns["simulate_many"](apps, cfg.cap_mib[0], code)
        og, oe, os_ = O.simulate_burst(apps, cfg.cap_mib, pol)
        want = O.speedup_from(O.seq_ticks(apps)[:, 0], os_[:, 0]["makespan"], np.full(len(apps), apps.shape[1]))
        np.testing.assert_array_equal(sp.view(np.uint64), want.view(np.uint64))
        np.testing.assert_array_equal(g, og)
        np.testing.assert_array_equal(e, oe)
        np.testing.assert_array_equal(st.view(np.uint8).reshape(len(apps), -1), os_.view(np.uint8).reshape(len(apps), -1))
