"""The C ABI (include/sgpu.h) without a GPU: libsgpu.so loads, exports every
declared entry point, its ctypes mirror has the header's struct layouts, and
argument validation fails loudly before touching the device."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1712_04495_b200 import _lib, batch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgpu.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sg_\w+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_functions()
    assert set(decl) == set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(L, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", nm), name


def test_abi_version():
    assert _lib.lib().sg_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "sgpu.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\","
        "sizeof(sg_batch), sizeof(sg_out), sizeof(sg_gen_params), sizeof(sg_app),"
        "sizeof(sg_step), sizeof(sg_trace_stats), sizeof(sg_trace_stats_f64),"
        "sizeof(sg_event), sizeof(sg_aggr));"
        "printf(\"%zu %zu %zu\\n\", offsetof(sg_batch, cap_mib), offsetof(sg_batch, tick_log2),"
        "offsetof(sg_out, events_per_trace));return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(probe), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = list(map(int, out))
    assert sizes[0] == ctypes.sizeof(_lib.SgBatch)
    assert sizes[1] == ctypes.sizeof(_lib.SgOut)
    assert sizes[2] == ctypes.sizeof(_lib.SgGenParams)
    assert sizes[3] == 16 and sizes[4] == batch.STEP_DTYPE.itemsize == 16
    assert sizes[5] == batch.STATS_DTYPE.itemsize == 32
    assert sizes[6] == batch.STATS_F64_DTYPE.itemsize == 40
    assert sizes[7] == batch.EVENT_DTYPE.itemsize == 16
    assert sizes[8] == 8 * len(_lib.AGGR_FIELDS)
    assert sizes[9] == _lib.SgBatch.cap_mib.offset
    assert sizes[10] == _lib.SgBatch.tick_log2.offset
    assert sizes[11] == _lib.SgOut.events_per_trace.offset


def _batch(**kw):
    b = _lib.SgBatch()
    b.n_traces = 1
    b.apps_per_trace = 4
    b.max_apps = 4
    b.policy_mask = 1
    b.ndev = 1
    b.cap_mib[0] = 100
    for k, v in kw.items():
        setattr(b, k, v)
    return b


@pytest.mark.parametrize("bad,msg", [
    (dict(policy_mask=0), "policy_mask"),
    (dict(policy_mask=0x10), "policy_mask"),
    (dict(ndev=0), "ndev"),
    (dict(ndev=9), "ndev"),
    (dict(apps_per_trace=2000, max_apps=2000), "longer than"),
    (dict(time_mode=1), "SG_TIME_F64 requires"),
    (dict(time_mode=7), "time_mode"),
])
def test_validation_errors_without_gpu(bad, msg):
    L = _lib.lib()
    b = _batch(**bad)
    o = _lib.SgOut()
    rc = L.sg_simulate_batch(ctypes.byref(b), ctypes.byref(o), None)
    assert rc < 0
    assert msg in L.sg_last_error().decode()


def test_cap_range_checked():
    L = _lib.lib()
    b = _batch()
    b.cap_mib[0] = 0
    rc = L.sg_simulate_batch(ctypes.byref(b), ctypes.byref(_lib.SgOut()), None)
    assert rc < 0 and "cap_mib" in L.sg_last_error().decode()


def test_check_raises_with_message():
    L = _lib.lib()
    rc = L.sg_simulate_batch(ctypes.byref(_batch(policy_mask=0)), ctypes.byref(_lib.SgOut()), None)
    with pytest.raises(_lib.SgpuError, match="policy_mask"):
        _lib.check(rc, "sg_simulate_batch")


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.SgpuUnavailable, match="no CPU fallback"):
        _lib.lib()
