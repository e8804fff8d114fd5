"""bench.py's reference arm runs on CPU (the reference's own simulate() on
the host cores): its one JSON line must carry the contract's keys."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    ref = os.path.join(ROOT, "oracle", "_ref", "memshare")
    if not os.path.isdir(ref):
        import pytest
        pytest.skip("oracle/_ref not installed (python oracle/build_ref.sh)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-step-s", "0.5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, check=True).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


def test_k1_engine_and_launch_count(monkeypatch):
    """bench.py's gpu_launches and roofline kernel name follow the engine
    sg_simulate_batch picks (sgpu_abi.cu simulate_device)."""
    sys.path.insert(0, ROOT)
    from paper_1712_04495_b200 import batch as B
    from paper_1712_04495_b200.tracegen import CONFIGS
    monkeypatch.delenv("SGPU_K1", raising=False)
    want = {"C2": "lane", "C3": "lane256", "C4": "lane", "C5": "lane"}
    for c, eng in want.items():
        cfg = CONFIGS[c]
        assert B.k1_engine(cfg.gen.apps_per_trace, len(cfg.policies), cfg.ndev) == eng, c
        assert B.k1_launches(cfg.gen.apps_per_trace, len(cfg.policies), cfg.ndev) == (2 if eng == "lane" else 1)
    assert B.k1_engine(128, 1) == "warp"          # one policy at 128 apps: the warp kernel is faster
    assert B.k1_engine(20, 4, 9) == "warp"        # more than 32 simulations per trace
    monkeypatch.setenv("SGPU_K1", "warp")
    assert B.k1_engine(64, 4) == "warp" and B.k1_launches(64, 4) == 1
    assert B.k1_engine(300, 2) == "warp"          # beyond 256 apps
    monkeypatch.setenv("SGPU_K1", "lane")
    assert B.k1_engine(256, 2) == "lane"
    monkeypatch.setenv("SGPU_K1", "octet")
    assert B.k1_engine(256, 2) == "octet" and B.k1_launches(256, 2) == 1
    assert B.K1_KERNELS["lane256"] == "trace_sim_lane256_kernel"
