"""Parallel firewall execution models on the GPU (drop-in for ``parafw.engines``).

Public surface mirrors /root/reference/pkg/src/parafw/engines.py:40-57.
The reference runs every model as tasks on a CPU pool; here every model is
a sequence of scan launches (match-set or rule-by-rule scan) on one GPU, and the
multi-GPU layer (``parallel``) maps the models onto GPUs:

* data-parallel (engines.py:302-314): one scan of [0, R) over all packets.
  Packet chunks per logical node are invisible in results, so ``nodes`` only
  affects nothing but validation (as in the reference, results and counters
  are node-independent).
* function-parallel (engines.py:316-321, 349-357): one speculative scan per
  non-empty rule partition ``partition_bounds(R, nodes)``; each launch folds
  its partition-local first match into a running per-packet minimum and adds
  its per-task comparisons (engines.py:359-369) in the kernel epilogue.
* hybrid (engines.py:323-347): packet chunks x rule lanes.  Per packet the
  lanes are exactly the function-parallel partitions, and chunking is
  invisible, so results and counters equal function-parallel with the same
  ``nodes``; it runs the same launches.

``batch_size`` (engines.py:277-282) splits dispatches in the reference; it is
invisible in results and counters, so the GPU scans the whole batch at once.
``executor`` / ``max_workers`` are validated for compatibility only: there is
no CPU backend.
"""

from __future__ import annotations

import os
import time
import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Sequence

import numpy as np

from . import _native
from .classifier import (ClassifyStats, CompiledRuleset, PacketArrays, classify_batch_sequential,
                         compile_ruleset, first_to_host)
from .model import Action, MatchResult, Packet, Rule, Ruleset

__all__ = [
    "MAX_NODES", "ConfigError", "ExecutionModel", "EngineConfig", "RulePartition", "PartialMatch",
    "partition_bounds", "partition_rules", "scan_partition", "aggregate",
    "combine_partition_matches", "Engine", "EngineResult", "run", "run_data_parallel",
    "run_function_parallel", "run_hybrid",
]

MAX_NODES = 512  # engines.py:59-61
_EXECUTORS = ("process", "thread", "serial")


class ConfigError(ValueError):
    """Invalid engine configuration."""


class ExecutionModel(Enum):
    SEQUENTIAL = "sequential"
    DATA_PARALLEL = "data"
    FUNCTION_PARALLEL = "function"
    HYBRID = "hybrid"

    @property
    def key(self) -> str:
        return self.value

    @classmethod
    def from_key(cls, key: str) -> "ExecutionModel":
        for m in cls:
            if m.value == key:
                return m
        raise ConfigError(f"unknown execution model {key!r} (expected one of "
                          f"{', '.join(m.value for m in cls)})")


@dataclass(frozen=True)
class EngineConfig:
    """Model selector + logical node count (engines.py:89-114).

    ``nodes``: packet chunks (data), rule partitions (function) or rule lanes
    (hybrid); it defines the function/hybrid comparison counters.
    ``batch_size``/``executor``/``max_workers`` are validated as in the
    reference and otherwise ignored (the GPU replaces the pool).
    """

    model: ExecutionModel
    nodes: int = 1
    batch_size: int = 4096
    executor: str = "process"
    max_workers: int | None = None

    def __post_init__(self) -> None:
        if not 1 <= self.nodes <= MAX_NODES:
            raise ConfigError(f"nodes must be within 1..{MAX_NODES}, got {self.nodes}")
        if self.batch_size < 1:
            raise ConfigError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.executor not in _EXECUTORS:
            raise ConfigError(f"executor must be one of {_EXECUTORS}, got {self.executor!r}")
        if self.max_workers is not None and self.max_workers < 1:
            raise ConfigError(f"max_workers must be >= 1, got {self.max_workers}")


@dataclass(frozen=True)
class RulePartition:
    """Contiguous ruleset slice owned by one node."""

    part_index: int
    global_offset: int
    rules: tuple[Rule, ...] = field(repr=False)

    def __len__(self) -> int:
        return len(self.rules)


@dataclass(frozen=True)
class PartialMatch:
    """One node's earliest local match (global index, action) and its comparisons."""

    part_index: int
    local_match: tuple[int, Action] | None
    comparisons: int


def partition_bounds(total: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous [lo, hi): the first ``total % parts`` parts get one extra
    (engines.py:143-154).  These are also the GPU shard boundaries."""
    if parts < 1:
        raise ConfigError(f"parts must be >= 1, got {parts}")
    q, r = divmod(total, parts)
    bounds, lo = [], 0
    for i in range(parts):
        hi = lo + q + (i < r)
        bounds.append((lo, hi))
        lo = hi
    return bounds


def partition_rules(ruleset: Ruleset, nodes: int) -> list[RulePartition]:
    return [RulePartition(i, lo, ruleset.rules[lo:hi])
            for i, (lo, hi) in enumerate(partition_bounds(len(ruleset), nodes))]


_part_cache: dict[int, tuple] = {}


def _compiled_partition(partition: RulePartition) -> CompiledRuleset:
    hit = _part_cache.get(id(partition))
    if hit is not None and hit[0]() is partition:
        return hit[1]
    compiled = CompiledRuleset(Ruleset(partition.rules))
    key = id(partition)
    _part_cache[key] = (weakref.ref(partition, lambda _r, k=key: _part_cache.pop(k, None)), compiled)
    return compiled


def scan_partition(partition: RulePartition, packet: Packet) -> PartialMatch:
    """Early-exit scan of one partition (engines.py:165-174), on the GPU."""
    n = len(partition)
    if n == 0:
        return PartialMatch(partition.part_index, None, 0)
    compiled = _compiled_partition(partition)
    local = int(compiled.scan_range([packet], 0, n)[0])
    if local < 0:
        return PartialMatch(partition.part_index, None, n)
    return PartialMatch(partition.part_index, (partition.global_offset + local, partition.rules[local].action),
                        local + 1)


def aggregate(partials: Iterable[PartialMatch], num_rules: int) -> MatchResult:
    """Coordinator combine: minimum global index wins, comparisons add up
    (engines.py:177-199).  Duplicate part indices and out-of-range indices raise."""
    seen: set[int] = set()
    best: tuple[int, Action] | None = None
    total = 0
    for pm in partials:
        if pm.part_index in seen:
            raise ValueError(f"duplicate part_index {pm.part_index} in partials")
        seen.add(pm.part_index)
        total += pm.comparisons
        if pm.local_match is None:
            continue
        idx, action = pm.local_match
        if not 0 <= idx < num_rules:
            raise ValueError(f"match index {idx} outside ruleset of {num_rules} rules")
        if best is None or idx < best[0]:
            best = (idx, action)
    if best is None:
        return MatchResult(Action.DROP, None, total)
    return MatchResult(best[1], best[0], total)


def combine_partition_matches(local_first, num_rules: int):
    """Per-packet minimum global index over partition rows, -1 = none
    (engines.py:202-212).  numpy in -> numpy out; the min runs on the GPU."""
    import torch
    arr = np.asarray(local_first)
    if arr.size == 0:
        return np.full(arr.shape[-1] if arr.ndim > 1 else 0, -1, dtype=np.int64)
    rows = arr.reshape(-1, arr.shape[-1]) if arr.ndim > 1 else arr.reshape(1, -1)
    valid = (rows >= 0) & (rows < num_rules)
    enc = np.where(valid, rows, _native.NO_MATCH).astype(np.int32)
    _native.require_device()
    dev = torch.cuda.current_device()
    d_rows = torch.from_numpy(np.ascontiguousarray(enc)).to(f"cuda:{dev}")
    out = torch.empty(rows.shape[1], dtype=torch.int32, device=f"cuda:{dev}")
    _native.check(_native.lib().pfw_combine_min(d_rows.data_ptr(), rows.shape[0], rows.shape[1],
                                                out.data_ptr(),
                                                torch.cuda.current_stream(dev).cuda_stream),
                  "pfw_combine_min")
    return first_to_host(out)


@dataclass(frozen=True)
class EngineResult:
    """Array form of one run: no per-packet objects (the large-batch fast path)."""

    first: np.ndarray        # int64, -1 = default deny
    comparisons: np.ndarray  # int64 per packet
    verdict_accept: np.ndarray  # bool per packet
    stats: ClassifyStats


class Engine:
    """Reusable batch-synchronous runner for one EngineConfig on one GPU.

    Not reentrant (engines.py:221-228); rulesets are compiled once per object
    and cached, packets are shared read-only.
    """

    def __init__(self, config: EngineConfig, device: int | None = None) -> None:
        self.config = config
        self.device = device

    @property
    def pool_width(self) -> int:
        return self.config.max_workers or os.cpu_count() or 1

    def close(self) -> None:
        pass

    def __enter__(self) -> "Engine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    # ------------------------------------------------------------- device
    def run_device(self, compiled: CompiledRuleset, pkts: PacketArrays, stream: int | None = None):
        """Launch the configured model; returns device tensors
        (first int32 [NO_MATCH = none], comps int32, stats int64 [sum, max_worker])."""
        import torch
        n = len(pkts)
        dev = pkts.data.device
        comps = torch.empty(n, dtype=torch.int32, device=dev)
        stats = torch.zeros(2, dtype=torch.int64, device=dev)
        model = self.config.model
        R = compiled.num_rules
        if model in (ExecutionModel.SEQUENTIAL, ExecutionModel.DATA_PARALLEL):
            first = compiled.scan_range_device(pkts, 0, R, comps=comps, stats=stats, stream=stream)
            return first, comps, stats
        if model not in (ExecutionModel.FUNCTION_PARALLEL, ExecutionModel.HYBRID):
            raise ConfigError(f"unsupported model {model}")
        first = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        _native.check(_native.lib().pfw_accumulator_init(n, first.data_ptr(), comps.data_ptr(), st),
                      "pfw_accumulator_init")
        for lo, hi in partition_bounds(R, self.config.nodes):
            if hi > lo:
                compiled.scan_partition_accumulate(pkts, lo, hi, first, comps, stats, stream=st)
        return first, comps, stats

    # -------------------------------------------------------------- arrays
    def run_arrays(self, ruleset, packets) -> EngineResult:
        start = time.perf_counter_ns()
        compiled = ruleset if isinstance(ruleset, CompiledRuleset) else compile_ruleset(ruleset, self.device)
        if compiled.is_shard:
            raise ValueError("Engine.run_arrays needs a whole ruleset, not a rule shard "
                             "(shards are scanned through parallel.run_function_parallel)")
        pkts = compiled._packets(packets)
        n = len(pkts)
        if n == 0:
            z = np.zeros(0, np.int64)
            return EngineResult(z, z, np.zeros(0, np.bool_),
                                ClassifyStats(0, 0, time.perf_counter_ns() - start, 0))
        first, comps, stats = self.run_device(compiled, pkts)
        first_h = first_to_host(first)
        comps_h = comps.cpu().numpy().astype(np.int64)
        st = stats.cpu().numpy()
        acc = np.zeros(n, dtype=np.bool_)
        hit = first_h >= 0
        acc[hit] = compiled.action_accept[first_h[hit]]
        return EngineResult(first_h, comps_h, acc,
                            ClassifyStats(int(st[0]), n, time.perf_counter_ns() - start, int(st[1])))

    # ----------------------------------------------------------- drop-in
    def run(self, ruleset: Ruleset, packets: Sequence[Packet]) -> tuple[list[MatchResult], ClassifyStats]:
        """Classify packets under the configured model (engines.py:260-290).
        results[i] belongs to packets[i]."""
        if self.config.model is ExecutionModel.SEQUENTIAL:
            return classify_batch_sequential(ruleset, packets)
        start = time.perf_counter_ns()
        compiled = compile_ruleset(ruleset, self.device)
        res = self.run_arrays(compiled, packets)
        results = compiled.build_results(res.first, res.comparisons) if len(res.first) else []
        s = res.stats
        return results, ClassifyStats(s.total_comparisons, s.packets_processed,
                                      time.perf_counter_ns() - start, s.max_worker_comparisons)


def run(ruleset: Ruleset, packets: Sequence[Packet], config: EngineConfig):
    """One-shot dispatch to the configured model (engines.py:372-375)."""
    with Engine(config) as engine:
        return engine.run(ruleset, packets)


def _run_checked(ruleset, packets, config: EngineConfig, expected: ExecutionModel):
    if config.model is not expected:
        raise ConfigError(f"config.model is {config.model.key!r}, expected {expected.key!r}")
    return run(ruleset, packets, config)


def run_data_parallel(ruleset, packets, config: EngineConfig):
    return _run_checked(ruleset, packets, config, ExecutionModel.DATA_PARALLEL)


def run_function_parallel(ruleset, packets, config: EngineConfig):
    return _run_checked(ruleset, packets, config, ExecutionModel.FUNCTION_PARALLEL)


def run_hybrid(ruleset, packets, config: EngineConfig):
    return _run_checked(ruleset, packets, config, ExecutionModel.HYBRID)
