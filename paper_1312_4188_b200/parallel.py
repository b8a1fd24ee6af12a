"""Multi-GPU sharding of the paper's two parallel-firewall models.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:

* data-parallel (engines.py:302-314 at GPU granularity): the ruleset is
  replicated on every GPU and the global packet batch is split into
  contiguous balanced shards ``partition_bounds(N, world)[rank]``
  (engines.py:143-154).  Each GPU scans its shard against [0, R); results
  are positional within the shard.  There is NO collective on the data
  path (stats are reduced only when asked for).
* function-parallel (engines.py:316-321, 349-369 at GPU granularity): the
  ruleset is split into contiguous shards ``partition_bounds(R, world)`` and
  every GPU scans the whole (replicated) batch against its shard only,
  speculatively.  Per packet the global first match is the minimum of the
  shard-local first matches (engines.py:202-212): one int32 MIN all-reduce
  with PFW_NO_MATCH = INT32_MAX as the identity, over NCCL/NVLink.  Per-task
  comparison counts (engines.py:366) are SUM-reduced when requested.

The local scan is injectable so the rank logic can be exercised on CPU with
the gloo backend in tests (with the oracle standing in for the kernel).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from .engines import partition_bounds

NO_MATCH = 0x7FFFFFFF


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int


def rank_info(group=None) -> RankInfo:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return RankInfo(dist.get_rank(group), dist.get_world_size(group))
    return RankInfo(0, 1)


def packet_shard(total_packets: int, info: RankInfo) -> tuple[int, int]:
    """This rank's contiguous packet shard (data-parallel)."""
    return partition_bounds(total_packets, info.world)[info.rank]


def rule_shard(num_rules: int, info: RankInfo) -> tuple[int, int]:
    """This rank's contiguous rule shard (function-parallel)."""
    return partition_bounds(num_rules, info.world)[info.rank]


def function_parallel_combine(local_first, local_comps=None, local_stats=None, group=None,
                              async_op: bool = False):
    """Fold every rank's shard-local results into global ones, in place.

    local_first: int32 tensor (global rule indices, NO_MATCH = none)
    local_comps: optional int32 per-packet per-task comparisons -> SUM
    local_stats: optional int64 [sum, max] -> [SUM, MAX]
    """
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return None
    works = [dist.all_reduce(local_first, op=dist.ReduceOp.MIN, group=group, async_op=async_op)]
    if local_comps is not None:
        works.append(dist.all_reduce(local_comps, op=dist.ReduceOp.SUM, group=group, async_op=async_op))
    if local_stats is not None:
        s, m = local_stats[0:1].clone(), local_stats[1:2].clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        local_stats[0:1].copy_(s)
        local_stats[1:2].copy_(m)
    return works if async_op else None


def reduce_stats(stats, group=None) -> None:
    """Data-parallel stats: [SUM of comparisons, MAX of comparisons] over ranks."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    s, m = stats[0:1].clone(), stats[1:2].clone()
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    stats[0:1].copy_(s)
    stats[1:2].copy_(m)


ScanFn = Callable[[int, int], tuple]  # (lo, hi) -> (first, comps, stats) for this rank's packets


def run_function_parallel(scan: ScanFn, num_rules: int, group=None, with_comps: bool = True):
    """Scan this rank's rule shard with ``scan`` then combine across ranks.

    ``scan(lo, hi)`` must return (first int32 [global index or NO_MATCH],
    comps int32 per-task counts, stats int64 [sum, max]) for the replicated
    packet batch.  Returns the global (first, comps, stats)."""
    info = rank_info(group)
    lo, hi = rule_shard(num_rules, info)
    first, comps, stats = scan(lo, hi)
    function_parallel_combine(first, comps if with_comps else None, stats, group)
    return first, comps, stats


def run_data_parallel(scan: Callable[[int, int], tuple], total_packets: int, group=None,
                      reduce: bool = False):
    """Scan this rank's packet shard with ``scan(start, stop)`` -> (first,
    comps, stats); no collective unless ``reduce`` (stats only)."""
    info = rank_info(group)
    a, b = packet_shard(total_packets, info)
    first, comps, stats = scan(a, b)
    if reduce and stats is not None:
        reduce_stats(stats, group)
    return (a, b), first, comps, stats
