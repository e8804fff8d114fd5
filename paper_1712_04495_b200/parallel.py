"""Multi-GPU: contiguous trace-id shards, one process per GPU, and the only
collective of the path — the aggregate-statistics all-reduce.

Traces are independent: rank r of W simulates traces
[r*N/W, (r+1)*N/W) (or, for weak scaling, its own fixed-size shard), keeps
its per-trace outputs in its own HBM, and contributes its K2 aggregate
(16 x u64: 12 sums, 4 maxima) to one SUM and one MAX all-reduce over
NCCL/NVLink.  No data-path collective exists.
"""

from __future__ import annotations

from . import _lib


def shard_range(n_traces: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [begin, end) of rank in world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n_traces, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def allreduce_aggregate(agg, group=None):
    """Cross-rank reduction of a 16-entry int64 aggregate (sg_aggr layout):
    entries [0, 12) are summed; max_makespan / max_holders are maxed;
    status_or is OR-ed (as a MAX over its expanded bits)."""
    import torch
    import torch.distributed as dist

    nsum = _lib.AGGR_NSUM
    sums = agg[:nsum].clone()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    status = agg[nsum + 2]
    bits = torch.stack([(status >> b) & 1 for b in range(8)])
    mx = torch.cat([agg[nsum:nsum + 2], bits, agg[nsum + 3:nsum + 4]])
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    st = torch.zeros((), dtype=agg.dtype, device=agg.device)
    for b in range(8):
        st = st | (mx[2 + b] << b)
    return torch.cat([sums, mx[0:2], st.reshape(1), mx[10:11]])


def sharded_run(gen, n_traces: int, policies, cap_mib, rank: int, world: int, device=None,
                group=None, stream=None):
    """Generate this rank's shard on its GPU, simulate it, reduce its stats
    and all-reduce the aggregate.  Returns (BatchResult, global aggregate dict)."""
    from .batch import aggr_to_dict, generate_traces, reduce_stats, simulate_batch

    b, e = shard_range(n_traces, rank, world)
    apps = generate_traces(gen, b, e - b, device=device, stream=stream)
    res = simulate_batch(apps, policies, cap_mib, stream=stream)
    agg = reduce_stats(res.stats_raw, stream=stream)
    if world > 1:
        agg = allreduce_aggregate(agg, group)
    return res, aggr_to_dict(agg)
