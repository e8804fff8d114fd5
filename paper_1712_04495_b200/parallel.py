"""Multi-GPU: contiguous trace-id shards, one process per GPU, and the only
collective of the path — the aggregate-statistics all-reduce.

Traces are independent: rank r of W simulates traces
[r*N/W, (r+1)*N/W) (or, for weak scaling, its own fixed-size shard), keeps
its per-trace outputs in its own HBM, and contributes its K2 aggregate
(16 x u64: 12 sums, 3 maxima, a status OR) to one all-gather over
NCCL/NVLink, combined locally.  No data-path collective exists.
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


def combine_aggregates(parts):
    """Reduce a (world, 16) int64 stack of sg_aggr rows: entries [0, 12)
    summed, max_makespan / max_holders / reserved_max0 maxed, status_or
    OR-ed (include/sgpu.h sg_aggr)."""
    import torch

    nsum = _lib.AGGR_NSUM
    out = torch.empty(parts.shape[1], dtype=parts.dtype, device=parts.device)
    out[:nsum] = parts[:, :nsum].sum(dim=0)
    out[nsum:] = parts[:, nsum:].max(dim=0).values
    st = parts[0, nsum + 2].clone()
    for r in range(1, parts.shape[0]):
        st |= parts[r, nsum + 2]
    out[nsum + 2] = st
    return out


def allreduce_aggregate(agg, group=None):
    """Cross-rank reduction of a 16-entry int64 aggregate (sg_aggr layout) in
    ONE collective: an all-gather of every rank's 128 B row (NCCL over
    NVLink; gloo on CPU for the multi-process tests), then the sums, maxima
    and the status OR are combined locally on each rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = agg if dist.get_backend(group) == "nccl" else agg.cpu()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return combine_aggregates(torch.stack(parts)).to(agg.device)


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
