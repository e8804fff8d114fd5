"""Multi-rank host logic on CPU with the gloo backend (world size 2): the
trace-shard partition and the aggregate all-reduce used by bench.py /
parallel.sharded_run.  Per-rank statistics come from the oracle here (the
checker), standing in for the GPU kernel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1712_04495_b200 import _lib
from paper_1712_04495_b200.parallel import allreduce_aggregate, shard_range
from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate


def np_aggregate(stats):
    """sg_aggr layout computed with numpy (what K2 computes on the GPU)."""
    s = stats.reshape(-1)
    u = lambda f: int(s[f].astype(np.uint64).sum())
    return np.array([s.size, u("makespan"), u("busy"), u("mem_integral"), u("grants"), u("pops"),
                     u("unfinished"), u("max_holders"), int((s["unfinished"] > 0).sum()),
                     int((s["status"] != 0).sum()), 0, 0, int(s["makespan"].max()),
                     int(s["max_holders"].max()), int(np.bitwise_or.reduce(s["status"])), 0],
                    dtype=np.int64)


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["C5"]
    b, e = shard_range(n, rank, world)
    apps = as_u32x4(generate(cfg.gen, b, e - b))
    aggs = []
    for pol in cfg.policies:
        _, _, st = O.simulate_burst(apps, cfg.cap_mib, pol)
        aggs.append(st)
    local = np_aggregate(np.stack(aggs))
    if rank == 1:
        local[14] |= 0x10  # a status bit only rank 1 sees must survive the OR
    out = allreduce_aggregate(torch.from_numpy(local))
    q.put((rank, out.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_aggregate_equals_single_process():
    from oracle import oracle as O
    world, n = 2, 301
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CONFIGS["C5"]
    apps = as_u32x4(generate(cfg.gen, 0, n))
    whole = np_aggregate(np.stack([O.simulate_burst(apps, cfg.cap_mib, pol)[2]
                                   for pol in cfg.policies]))
    whole[14] |= 0x10
    assert res[0] == res[1] == whole.tolist()
    assert len(whole) == len(_lib.AGGR_FIELDS)
