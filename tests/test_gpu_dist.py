"""Multi-rank runs of the real kernels (K1 trace simulation + K2 statistics
reduction + the one aggregate collective) with two ranks sharing cuda:0
over gloo — the only multi-process shape a one-GPU box offers.  The NCCL
path is the same code with backend "nccl" (one rank per GPU)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1712_04495_b200 import batch as B
from paper_1712_04495_b200.parallel import shard_range, sharded_run
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cname, n, q):
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = CONFIGS[cname]
    res, agg = sharded_run(cfg.gen, n, cfg.policies, cfg.cap_mib, rank, world, device=0)
    torch.cuda.synchronize()
    # this rank's outputs against the oracle on a sample of its shard
    b, e = shard_range(n, rank, world)
    k = min(64, e - b)
    apps = as_u32x4(generate(cfg.gen, b, k))
    st = res.stats()
    napp = cfg.gen.apps_per_trace
    ok = True
    for pi, pol in enumerate(res.policies):
        g, en, s = O.simulate_burst(apps, cfg.cap_mib, pol.value)
        ok &= np.array_equal(res.ticks("grant")[pi][:k * napp].reshape(g.shape), g)
        ok &= np.array_equal(res.ticks("end")[pi][:k * napp].reshape(en.shape), en)
        ok &= np.array_equal(st[pi][:k].view(np.uint8), s.view(np.uint8))
    q.put((rank, agg, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cname,n", [("C2", 20_011), ("C5", 6_001)])
def test_two_ranks_real_kernels(cname, n, cuda):
    """parallel.sharded_run on two ranks: each rank's K1 outputs match the
    oracle, and the all-gathered aggregate equals one process's K2 over the
    whole trace range [0, n)."""
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cname, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, agg, ok = q.get(timeout=600)
        got[r] = agg
        assert ok, f"rank {r} outputs differ from the oracle"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = CONFIGS[cname]
    apps = B.generate_traces(cfg.gen, 0, n, device=0)
    whole = B.aggr_to_dict(B.reduce_stats(B.simulate_batch(apps, cfg.policies, cfg.cap_mib).stats_raw))
    assert got[0] == got[1] == whole


def test_bench_launches_ranks_itself(cuda):
    """`bench.py --gpus 2` without a launcher re-executes under
    torch.distributed.run: two ranks (gloo on one GPU here), n_gpus 2, and
    the aggregate of both shards equals one process's K2 over [0, 2n)."""
    n = 8192
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dist-backend", "gloo", "--traces", str(n), "--steps", "2",
                          "--warmup", "3", "--no-cpu", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    cfg = CONFIGS["C2"]
    apps = B.generate_traces(cfg.gen, 0, 2 * n, device=0)
    whole = B.aggr_to_dict(B.reduce_stats(B.simulate_batch(apps, cfg.policies, cfg.cap_mib).stats_raw))
    assert line["aggregate"] == whole
    assert line["value"] > 0 and line["gpu_launches"] > 0
