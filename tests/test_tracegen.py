"""Generator determinism and distribution (CPU; the CUDA twin is checked
bit-for-bit in test_gpu_parity.py::test_generator_bit_identical)."""

import dataclasses

import numpy as np

from paper_1712_04495_b200.tracegen import (APP_DTYPE, CONFIGS, GenParams, as_u32x4, generate,
                                            mix64_int)


def test_mix64_known_values():
    # SplitMix64 (Steele et al.) reference outputs for state 0, GOLDEN, ...
    assert mix64_int(0) == 0xE220A8397B1DCDAF
    assert mix64_int(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_shard_independence():
    g = CONFIGS["C2"].gen
    whole = generate(g, 0, 100)
    np.testing.assert_array_equal(whole[40:70], generate(g, 40, 30))


def test_layout_and_ranges():
    for name, cfg in CONFIGS.items():
        a = generate(cfg.gen, 0, 64)
        assert a.dtype == APP_DTYPE and a.dtype.itemsize == 16
        g = cfg.gen
        assert a["arrival"].min() >= g.arr_lo and a["arrival"].max() <= g.arr_hi
        assert a["mem_mib"].min() >= g.mem_lo and a["mem_mib"].max() <= g.mem_hi
        assert a["busy"].min() >= g.busy_lo and a["busy"].max() <= g.busy_hi
        prio = a["attr"] & 0xFF
        assert prio.max() < g.prio_levels
        dev = a["attr"] >> 8
        np.testing.assert_array_equal(dev, (np.arange(g.apps_per_trace) % g.ndev)[None, :]
                                      .repeat(64, 0))


def test_c1_is_readme_burst():
    a = as_u32x4(generate(CONFIGS["C1"].gen, 0, 1))[0]
    assert (a[:, 0] == 900).all() and (a[:, 1] == 700).all() and (a[:, 2] == 100).all()
    assert (a[:, 3] == 0).all() and a.shape == (8, 4)


def test_skewed_priorities_and_cubic_arrivals():
    a = generate(CONFIGS["C3"].gen, 0, 4000)
    p = np.bincount((a["attr"] & 0xFF).ravel(), minlength=4) / a.size
    np.testing.assert_allclose(p, [8 / 15, 4 / 15, 2 / 15, 1 / 15], atol=0.01)
    arr = a["arrival"].ravel()
    assert arr.max() < 16384 and np.median(arr) < 16384 / 4  # bursty near 0


def test_seed_changes_output():
    g = CONFIGS["C2"].gen
    assert not np.array_equal(generate(g, 0, 4), generate(dataclasses.replace(g, seed=2), 0, 4))
    assert np.array_equal(generate(GenParams(), 0, 3), generate(GenParams(), 0, 3))
