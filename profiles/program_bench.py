"""Step-program mode throughput: the reference's
multi-phase builtin profiles (memshare/harness.py:65-83: ara-like,
mummer-like, blast-like) as step programs, one batch of many traces on one
B200 through simulate_batch (default engine: K1 v6 lane-per-simulation
kernel; SGPU_K1=warp: the warp-per-trace kernel), checked bit-exactly
against the oracle on a sample.

Each trace is the acceptance workload shape (test_acceptance.py:229-246:
4 ara + 4 mummer (priority 2) + 4 blast on a 2400 MiB device) with a seeded
per-app start offset (a leading cpu step of 0..2047 ticks of the workload's
exact dyadic grid), so traces differ.

    python profiles/program_bench.py [n_traces]      (needs a GPU)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1712_04495_b200 import _lib, batch as B  # noqa: E402
from paper_1712_04495_b200 import harness as H  # noqa: E402
from oracle import oracle as O  # noqa: E402

POLICIES = ("fifo", "mmu", "pfifo", "pmmu")


def workload(n_traces: int, seed: int = 7):
    prof = H.builtin_profiles()
    apps = [prof["ara-like"]] * 4 + [H.AppProfile(prof["mummer-like"].name, prof["mummer-like"].phases,
                                                  priority=2)] * 4 + [prof["blast-like"]] * 4
    spec = H.WorkloadSpec(instances=apps, time_scale=1000.0 / 1024.0)
    enc = H.encode_spec(spec)
    assert enc.time_mode == _lib.TIME_TICKS  # exact dyadic tick grid (2^-tick_log2 s)
    n = len(enc.attr)
    body = enc.steps
    offs = enc.step_offsets.astype(np.int64)
    per_trace = len(body) + n          # + one leading cpu step per app
    rng = np.random.default_rng(seed)
    start = rng.integers(0, 2048, size=(n_traces, n))
    so = np.zeros(n_traces * n + 1, dtype=np.uint32)
    # one trace's layout: per app [cpu(start), its profile steps]
    lay = []
    for i in range(n):
        lay.append(-1)                  # placeholder for the start step
        lay.extend(range(offs[i], offs[i + 1]))
    lay = np.array(lay)
    app_first = np.zeros(n, dtype=np.int64)
    k = 0
    for i in range(n):
        app_first[i] = k
        k += 1 + int(offs[i + 1] - offs[i])
    tmpl = np.zeros(per_trace, dtype=B.STEP_DTYPE)
    tmpl[lay >= 0] = body[lay[lay >= 0]]
    steps = np.tile(tmpl, n_traces)
    cpu_pos = (np.arange(n_traces)[:, None] * per_trace + app_first[None, :]).reshape(-1)
    steps["op"][cpu_pos] = _lib.OP_CPU
    steps["mib"][cpu_pos] = 0
    steps["dur"][cpu_pos] = start.reshape(-1)
    so[:-1] = (np.arange(n_traces)[:, None] * per_trace + app_first[None, :]).reshape(-1)
    so[-1] = n_traces * per_trace
    attr = np.tile(enc.attr, n_traces).reshape(n_traces, n)
    return steps, so, attr, enc.cap_mib, n, enc.tick_log2


def main():
    n_traces = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    steps, so, attr, cap, n, tick_log2 = workload(n_traces)
    dev = torch.device("cuda", 0)
    apps = np.zeros((n_traces, n, 4), dtype=np.uint32)
    apps[..., 3] = attr
    apps_t = torch.from_numpy(apps.view(np.int32)).to(dev)
    steps_t = torch.from_numpy(steps.view(np.int32).reshape(-1, 4).copy()).to(dev)
    so_t = torch.from_numpy(so.view(np.int32).copy()).to(dev)
    run = lambda: B.simulate_batch(apps_t, POLICIES, cap, steps=steps_t, step_offsets=so_t,
                                   tick_log2=tick_log2)
    for _ in range(2):
        res = run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = 3
    for _ in range(reps):
        res = run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    # oracle on a sample of traces
    st = res.stats()
    grant = res.ticks("grant").reshape(len(POLICIES), n_traces, n)
    end = res.ticks("end").reshape(len(POLICIES), n_traces, n)
    sample = np.linspace(0, n_traces - 1, 64).astype(int)
    for pi, pol in enumerate(POLICIES):
        for t in sample:
            s0, s1 = int(so[t * n]), int(so[(t + 1) * n])
            g, e, s = O.simulate_program(steps[s0:s1], so[t * n:(t + 1) * n + 1] - s0, attr[t], cap, pol)
            assert np.array_equal(grant[pi, t], g) and np.array_equal(end[pi, t], e), (pol, t)
            assert np.array_equal(st[pi, t].view(np.uint8), s.view(np.uint8)), (pol, t)
    import os as _os
    eng = _os.environ.get("SGPU_K1", "auto")
    print(f"program mode [{eng}]: {n_traces} traces x {n} apps ({len(steps) // n_traces} steps/trace) x "
          f"{len(POLICIES)} policies: {ms:.1f} ms per launch = "
          f"{n_traces * len(POLICIES) / ms * 1e3:.3g} trace-sims/s; 64-trace oracle sample bit-exact")


if __name__ == "__main__":
    main()
