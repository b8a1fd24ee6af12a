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


def _active(group) -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def all_reduce(t, op, group=None) -> None:
    """In-place all-reduce.  NCCL reduces device tensors directly (NVLink /
    NVSwitch); the gloo backend (CPU tests, shared-GPU smoke runs) reduces a
    host copy."""
    import torch.distributed as dist
    if not _active(group):
        return
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def function_parallel_combine(local_first, local_comps=None, local_stats=None, group=None) -> None:
    """Fold every rank's shard-local results into global ones, in place
    (engines.py:202-212 and 359-369 across GPUs).

    local_first: int32 tensor (global rule indices, NO_MATCH = none) -> MIN
    local_comps: optional int32 per-packet per-task comparisons      -> SUM
    local_stats: optional int64 [sum, max]                           -> [SUM, MAX]
    """
    import torch.distributed as dist
    if not _active(group):
        return
    all_reduce(local_first, dist.ReduceOp.MIN, group)
    if local_comps is not None:
        all_reduce(local_comps, dist.ReduceOp.SUM, group)
    if local_stats is not None:
        reduce_stats(local_stats, group)


def reduce_stats(stats, group=None) -> None:
    """[SUM of comparisons, MAX of per-task comparisons] over ranks."""
    import torch.distributed as dist
    if not _active(group):
        return
    s, m = stats[0:1].clone(), stats[1:2].clone()
    all_reduce(s, dist.ReduceOp.SUM, group)
    all_reduce(m, dist.ReduceOp.MAX, group)
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


class FusedFunctionParallel:
    """Function-parallel across ranks with the MIN / SUM combine fused into the
    scan kernel's epilogue: every rank scans its rule shard
    of the replicated batch and writes resolved packets straight into the
    owner rank's result buffer with NVLink atomics (CUDA IPC mappings), so
    the exchange overlaps the scan tile by tile instead of following it as a
    separate all-reduce.

    scatter=True (default): rank t ends up holding packets
    ``packet_shard(n, t)`` (reduce-scatter result, one atomic per packet);
    scatter=False: every rank holds all n results (all-reduce result,
    world atomics per packet).
    """

    def __init__(self, compiled, n: int, scatter: bool = True, with_comps: bool = True, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _native
        self.compiled, self.n, self.scatter, self.group = compiled, n, scatter, group
        self.info = rank_info(group)
        self.device = compiled.device
        dev = f"cuda:{self.device}"
        self.own_range = packet_shard(n, self.info) if scatter else (0, n)
        m = self.own_range[1] - self.own_range[0]
        # two result buffer sets, used by alternate calls: a call writes one
        # set (reset during the previous call) and resets the other before its
        # completion barrier, so every call needs a single host barrier.
        # never allocate 0 bytes: IPC needs a real allocation on every rank
        self._first = [torch.full((max(m, 1),), NO_MATCH, dtype=torch.int32, device=dev) for _ in range(2)]
        self._comps = [torch.zeros(max(m, 1), dtype=torch.int32, device=dev) for _ in range(2)] \
            if with_comps else [None, None]
        self._k = 0
        torch.cuda.synchronize(self.device)
        lib = _native.lib()
        hs = lib.pfw_ipc_handle_size()

        def handle(t):
            buf = ctypes.create_string_buffer(hs)
            off = ctypes.c_uint64()
            _native.check(lib.pfw_ipc_get_handle(t.data_ptr(), buf, ctypes.byref(off)), "pfw_ipc_get_handle")
            return buf.raw, off.value

        mine = [(handle(self._first[k]), handle(self._comps[k]) if with_comps else None) for k in range(2)]
        world = self.info.world
        if world > 1:
            allh = [None] * world
            dist.all_gather_object(allh, mine, group=group)  # (also the initial barrier)
        else:
            allh = [mine]
        self._opened = []
        P = ctypes.c_void_p
        self._peer_first, self._peer_comps = [], []
        for k in range(2):
            firsts, comps = [], []
            for t, sets in enumerate(allh):
                hf, hc = sets[k]
                if t == self.info.rank:
                    firsts.append(self._first[k].data_ptr())
                    comps.append(self._comps[k].data_ptr() if with_comps else None)
                    continue
                for hnd, out in ((hf, firsts), (hc, comps)):
                    if hnd is None:
                        out.append(None)
                        continue
                    raw, off = hnd
                    base = ctypes.c_void_p()
                    _native.check(lib.pfw_ipc_open(self.device, raw, ctypes.byref(base)), "pfw_ipc_open")
                    self._opened.append(base.value)
                    out.append(base.value + off)
            self._peer_first.append((P * world)(*firsts))
            self._peer_comps.append((P * world)(*comps) if with_comps else None)
        # packets each rank's buffers hold (checked again by the C side)
        self._peer_cap = (ctypes.c_int64 * world)(*[
            (b - a if scatter else n) for a, b in partition_bounds(n, world)])

    @property
    def first(self):
        """This rank's first-match buffer of the latest call."""
        return self._first[(self._k - 1) % 2]

    @property
    def comps(self):
        return self._comps[(self._k - 1) % 2]

    def _barrier(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        if self.info.world > 1:
            dist.barrier(group=self.group)

    def run(self, pkts, stats=None, stream: int | None = None):
        """Scan this rank's rule shard with the fused combine and return this
        rank's (first, comps) once every rank's scan has completed.  The
        returned tensors are views of an internal buffer set: valid until
        the next call (which resets them for the call after it)."""
        import torch
        from . import _native
        if len(pkts) != self.n:
            raise ValueError(f"FusedFunctionParallel was set up for batches of {self.n} packets, got {len(pkts)}")
        k = self._k % 2
        # a rule-shard handle holds exactly this rank's rules (local window,
        # global indices); a whole-ruleset handle scans this rank's window
        if getattr(self.compiled, "is_shard", False):
            lo, hi = 0, self.compiled.num_rules
        else:
            lo, hi = rule_shard(self.compiled.num_rules, self.info)
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        _native.check(_native.lib().pfw_scan_fused_min(
            self.compiled.handle, lo, hi, pkts.data.data_ptr(), len(pkts), self._peer_first[k],
            self._peer_comps[k], self._peer_cap, self.info.world, 1 if self.scatter else 0,
            None if stats is None else stats.data_ptr(), st), "pfw_scan_fused_min")
        # reset the other set (the previous call's results) for the next call;
        # the barrier below orders it before any rank's next-call atomics
        with torch.cuda.stream(torch.cuda.ExternalStream(st, device=self.device)):
            self._first[k ^ 1].fill_(NO_MATCH)
            if self._comps[k ^ 1] is not None:
                self._comps[k ^ 1].zero_()
        self._barrier()  # every rank's atomics into set k have landed
        self._k += 1
        m = self.own_range[1] - self.own_range[0]
        return self._first[k][:m], (self._comps[k][:m] if self._comps[k] is not None else None)

    def close(self):
        from . import _native
        for ptr in self._opened:
            _native.lib().pfw_ipc_close(self.device, ptr)
        self._opened = []
