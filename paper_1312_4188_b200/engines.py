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
from .classifier import (NO_MATCH, ClassifyStats, CompiledRuleset, MatchResults, PacketArrays,
                         classify_batch_sequential, compile_ruleset, first_to_host)
from .model import Action, MatchResult, Packet, Rule, Ruleset

__all__ = [
    "MAX_NODES", "ConfigError", "ExecutionModel", "EngineConfig", "RulePartition", "PartialMatch",
    "partition_bounds", "partition_rules", "scan_partition", "aggregate",
    "combine_partition_matches", "Engine", "EngineResult", "run", "run_data_parallel",
    "run_function_parallel", "run_hybrid",
]

MAX_NODES = 512  # engines.py:59-61
_EXECUTORS = ("process", "thread", "serial")
_SHARDS = ("auto", "packets", "rules")


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
    ``gpus``: how many GPUs the Engine shards over (results and counters do
    not depend on it).  ``shard``: how the function-parallel / hybrid models
    use them -- "rules" gives each GPU a contiguous run of the ``nodes``
    partitions (the model's own decomposition, combined by the fused NVLink
    MIN / SUM), "packets" gives each GPU a packet shard and the whole
    partition loop (no combine; the model's speculative per-partition work
    then stays per GPU instead of growing with the GPU count); "auto" picks
    packets.  Results and counters are identical.
    ``batch_size``/``executor``/``max_workers`` are validated as in the
    reference and otherwise ignored (the GPU replaces the pool).
    """

    model: ExecutionModel
    nodes: int = 1
    batch_size: int = 4096
    executor: str = "process"
    max_workers: int | None = None
    gpus: int = 1  # GPUs one Engine drives (packet shards / rule shards; see Engine)
    shard: str = "auto"  # function / hybrid over several GPUs: "rules", "packets" or "auto" (= packets)

    def __post_init__(self) -> None:
        if not 1 <= self.gpus <= 64:
            raise ConfigError(f"gpus must be within 1..64, got {self.gpus}")
        if self.shard not in _SHARDS:
            raise ConfigError(f"shard must be one of {_SHARDS}, got {self.shard!r}")
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


class EngineResult:
    """Array form of one run: no per-packet objects (the large-batch fast path).

    ``first``: matched rule index per packet, -1 = default deny (int32 from
    the host path, int64 otherwise); ``verdict_accept``: bool per packet;
    ``comparisons``: per-packet comparison counts -- given by the kernels for
    the function-parallel / hybrid models, derived on first access for the
    sequential / data-parallel ones (``first + 1`` or R, classifier.py:200);
    ``stats``: ClassifyStats."""

    __slots__ = ("first", "verdict_accept", "stats", "_comps", "_num_rules")

    def __init__(self, first, comparisons, verdict_accept, stats: ClassifyStats, num_rules: int | None = None):
        self.first = first
        self.verdict_accept = verdict_accept
        self.stats = stats
        self._comps = comparisons
        self._num_rules = num_rules
        if comparisons is None and num_rules is None:
            raise ValueError("EngineResult needs comparisons or num_rules")

    @property
    def comparisons(self) -> np.ndarray:
        if self._comps is None:
            f = np.asarray(self.first, dtype=np.int64)
            self._comps = np.where(f >= 0, f + 1, self._num_rules)
        return self._comps

    def __len__(self) -> int:
        return len(self.first)


def _is_host_batch(packets) -> bool:
    """Host packet batch for the e2e path: the reference's PacketArrays
    columns as a dict of arrays, or (n, 4) uint32 records."""
    if isinstance(packets, dict):
        return True
    return isinstance(packets, np.ndarray) and packets.ndim == 2 and packets.shape[1] == 4


def _host_len(packets) -> int:
    return len(packets["proto"]) if isinstance(packets, dict) else int(packets.shape[0])


def _host_slice(packets, a: int, b: int):
    if isinstance(packets, dict):
        return {f: np.asarray(packets[f])[a:b] for f in ("proto", "src_ip", "src_port", "dst_ip", "dst_port")}
    return packets[a:b]


def _nvtx(name: str):
    import torch
    return torch.cuda.nvtx.range(name)


class Engine:
    """Reusable batch-synchronous runner for one EngineConfig (engines.py:221-290).

    Not reentrant (engines.py:221-228); rulesets are compiled once per
    device and cached, packets are shared read-only.

    GPUs: ``devices`` (or ``EngineConfig.gpus``, devices 0..gpus-1) -- one
    process drives all of them, one stream per device:

    * sequential / data-parallel: packets split into contiguous
      ``partition_bounds(N, G)`` shards (engines.py:307), the ruleset
      replicated on every device, no collective; host batches run the e2e
      pipeline on every device at once (one host thread each).
    * function-parallel / hybrid, shard="rules": the ``nodes`` rule
      partitions are grouped into G contiguous runs, each device uploads
      only its run (a rule shard) and scans the replicated packets against
      its partitions, combining straight into the packet owners' result
      buffers with NVLink atomics (the fused MIN / SUM epilogue, peer access
      within the process) -- engines.py:349-369 across devices with no
      separate collective.  shard="packets" (and "auto"): packet shards as
      for data-parallel, each device running all partitions.
    """

    def __init__(self, config: EngineConfig, device: int | None = None, devices=None) -> None:
        self.config = config
        if devices is None:
            if config.gpus > 1:
                devices = list(range(config.gpus))
            else:
                devices = [device]
        devices = list(devices)
        if not devices:
            raise ConfigError("devices must name at least one GPU")
        if any(d is not None for d in devices):
            _native.require_device()
            have = _native.device_count()
            for d in devices:
                if d is not None and not 0 <= int(d) < have:
                    raise ConfigError(f"GPU {d} requested but only {have} CUDA devices are visible")
        self.devices = devices
        self.device = devices[0]
        self._copies: dict = {}

    @property
    def pool_width(self) -> int:
        return self.config.max_workers or os.cpu_count() or 1

    @property
    def gpus(self) -> int:
        return len(self.devices)

    def close(self) -> None:
        self._copies.clear()

    def __enter__(self) -> "Engine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def _dev(self, g: int) -> int:
        d = self.devices[g]
        if d is None:
            import torch
            _native.require_device()
            return torch.cuda.current_device()
        return int(d)

    def _copy(self, compiled: CompiledRuleset, device: int, lo: int | None = None, hi: int | None = None,
              slot: int = 0):
        """``compiled`` (or its rule shard [lo, hi)) uploaded on ``device``, cached.
        ``slot`` > 0 asks for a separate handle (handles are not reentrant: host
        threads driving the same device concurrently each need their own)."""
        if lo is None and compiled.device == device and slot == 0:
            return compiled
        key = (id(compiled), device, lo, hi, slot)
        hit = self._copies.get(key)
        if hit is not None and hit[0]() is compiled:
            return hit[1]
        if lo is None:
            c = CompiledRuleset.from_columns(compiled.columns(), device=device)
        else:
            cols = {f: v[lo:hi] for f, v in compiled.columns().items()}
            c = CompiledRuleset.from_columns(cols, device=device, shard=(lo, compiled.num_rules))
        self._copies[key] = (weakref.ref(compiled), c)
        return c

    def _whole_table(self, model: ExecutionModel) -> bool:
        """One scan of [0, R) gives the model's exact results: sequential /
        data-parallel, and function-parallel / hybrid with one node (a single
        partition holding every rule: the same first match, per-task
        comparisons first + 1 or R, and per-task maximum, engines.py:349-369)."""
        return model in (ExecutionModel.SEQUENTIAL, ExecutionModel.DATA_PARALLEL) or self.config.nodes == 1

    # ------------------------------------------------------------- device
    def run_device(self, compiled: CompiledRuleset, pkts: PacketArrays, stream: int | None = None):
        """Launch the configured model on one device; returns device tensors
        (first int32 [NO_MATCH = none], comps int32, stats int64 [sum, max_worker])."""
        import torch
        n = len(pkts)
        dev = pkts.data.device
        comps = torch.empty(n, dtype=torch.int32, device=dev)
        stats = torch.zeros(2, dtype=torch.int64, device=dev)
        model = self.config.model
        R = compiled.num_rules
        if self._whole_table(model):
            first = compiled.scan_range_device(pkts, 0, R, comps=comps, stats=stats, stream=stream)
            return first, comps, stats
        if model not in (ExecutionModel.FUNCTION_PARALLEL, ExecutionModel.HYBRID):
            raise ConfigError(f"unsupported model {model}")
        first = torch.empty(n, dtype=torch.int32, device=dev)
        # every non-empty partition of partition_bounds(R, nodes), folded on the device
        compiled.scan_partitions(pkts, self.config.nodes, first, comps, stats, stream=stream)
        return first, comps, stats

    # -------------------------------------------------------------- arrays
    def run_arrays(self, ruleset, packets) -> EngineResult:
        """The configured model over a packet batch, results as arrays.

        ``packets``: a device ``PacketArrays``, a host batch (dict of the
        reference's PacketArrays columns, or (n, 4) uint32 records -- pinned or
        pageable numpy; the e2e pipeline copies, scans and returns results in
        overlapped chunks) or a sequence of ``Packet``."""
        start = time.perf_counter_ns()
        compiled = ruleset if isinstance(ruleset, CompiledRuleset) else compile_ruleset(ruleset, self._dev(0))
        if compiled.is_shard:
            raise ValueError("Engine.run_arrays needs a whole ruleset, not a rule shard "
                             "(shards are scanned through parallel.run_function_parallel)")
        R = compiled.num_rules
        host = _is_host_batch(packets)
        n = _host_len(packets) if host else len(packets)
        if n == 0:
            z = np.zeros(0, np.int64)
            return EngineResult(z, z, np.zeros(0, np.bool_), ClassifyStats(0, 0, time.perf_counter_ns() - start, 0))
        model = self.config.model
        seq = self._whole_table(model)
        if seq and host:
            with _nvtx("Engine.run_arrays: e2e (host batch)"):
                first, verdict, st = self._data_host(compiled, packets, n)
            return EngineResult(first, None, verdict, ClassifyStats(int(st[0]), n, time.perf_counter_ns() - start,
                                                                    int(st[1])), num_rules=R)
        if host and self.gpus == 1:
            # function-parallel / hybrid: the same H2D / scan / D2H pipeline,
            # every node partition per chunk folded on the device
            with _nvtx(f"Engine.run_arrays: e2e {model.value} (host batch)"):
                comp = self._copy(compiled, self._dev(0))
                first_h, comps_h, verdict, st = comp.classify_host_partitions(packets, self.config.nodes)
            return EngineResult(first_h, comps_h, verdict, ClassifyStats(int(st[0]), n, time.perf_counter_ns() - start,
                                                                        int(st[1])), num_rules=R)
        if host:
            with _nvtx("Engine.run_arrays: upload"):
                pk = packets if isinstance(packets, dict) else PacketArrays.unpack_host(packets)
                pkts = PacketArrays.from_columns(*[pk[f] for f in ("proto", "src_ip", "src_port", "dst_ip",
                                                                  "dst_port")], device=self._dev(0))
        else:
            with _nvtx("Engine.run_arrays: pack + upload"):
                pkts = compiled._packets(packets) if self.gpus == 1 else (
                    packets if isinstance(packets, PacketArrays) else PacketArrays.from_packets(packets, self._dev(0)))
        if self.gpus > 1:
            with _nvtx(f"Engine.run_arrays: {model.value} on {self.gpus} GPUs"):
                by_rules = not seq and self.config.shard == "rules"
                first_h, comps_h, st = (self._function_multi(compiled, pkts) if by_rules
                                        else self._data_multi(compiled, pkts, with_comps=not seq))
        else:
            if compiled.device != pkts.device:
                compiled = self._copy(compiled, pkts.device)
            with _nvtx(f"Engine.run_arrays: {model.value} scan"):
                first, comps, stats = self.run_device(compiled, pkts)
            first_h = first_to_host(first)
            comps_h = None if seq else comps.cpu().numpy().astype(np.int64)
            st = stats.cpu().numpy()
        acc = np.zeros(n, dtype=np.bool_)
        hit = first_h >= 0
        acc[hit] = compiled.action_accept[first_h[hit]]
        return EngineResult(first_h, comps_h, acc,
                            ClassifyStats(int(st[0]), n, time.perf_counter_ns() - start, int(st[1])), num_rules=R)

    def _data_host(self, compiled, packets, n):
        """Host batch, sequential / data-parallel: the e2e pipeline on every
        device over its packet shard, outputs written in place."""
        if self.gpus == 1:
            dev = self._dev(0)
            return self._copy(compiled, dev).classify_host(packets)
        import torch
        from concurrent.futures import ThreadPoolExecutor
        first = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        verdict = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy().view(np.bool_)
        bounds = partition_bounds(n, self.gpus)
        devs = [self._dev(g) for g in range(self.gpus)]
        reps = [self._copy(compiled, d, slot=devs[:g].count(d)) for g, d in enumerate(devs)]

        def shard(g):  # ctypes drops the GIL: the devices' pipelines run concurrently
            a, b = bounds[g]
            if b == a:
                return np.zeros(2, np.int64)
            return reps[g].classify_host(_host_slice(packets, a, b), out=(first[a:b], verdict[a:b]))[2]
        with ThreadPoolExecutor(max_workers=self.gpus) as ex:
            sts = list(ex.map(shard, range(self.gpus)))
        return first, verdict, np.array([sum(int(x[0]) for x in sts), max(int(x[1]) for x in sts)], np.int64)

    def _data_multi(self, compiled, pkts, with_comps: bool = False):
        """Device batch over G devices as contiguous packet shards
        (engines.py:307), replicated rules, no collective: the data-parallel
        model, or any model with shard="packets" (each device runs the
        model's whole launch sequence on its shard)."""
        import torch
        bounds = partition_bounds(len(pkts), self.gpus)
        outs = []
        for g, (a, b) in enumerate(bounds):  # launches are asynchronous: the devices run concurrently
            if b == a:
                continue
            dev = self._dev(g)
            rep = self._copy(compiled, dev)
            with torch.cuda.device(dev):
                sub = PacketArrays(pkts.data[a:b].to(f"cuda:{dev}", non_blocking=True))
                outs.append(self.run_device(rep, sub))
        first = np.concatenate([first_to_host(f) for f, _, _ in outs])
        comps = np.concatenate([c.cpu().numpy() for _, c, _ in outs]).astype(np.int64) if with_comps else None
        st = [s.cpu().numpy() for _, _, s in outs]
        return first, comps, np.array([sum(int(x[0]) for x in st), max(int(x[1]) for x in st)], np.int64)

    def _function_multi(self, compiled, pkts):
        """Function-parallel / hybrid over G devices: device g owns a
        contiguous run of the ``nodes`` rule partitions (its rule shard) and
        scans the replicated packets against each of them; every scan's
        epilogue folds its per-packet first match (atomicMin) and per-task
        comparisons (atomicAdd) straight into the owner device's result
        buffers over NVLink (packet owners: partition_bounds(N, G))."""
        import ctypes
        import torch
        n, G, R = len(pkts), self.gpus, compiled.num_rules
        parts = [(lo, hi) for lo, hi in partition_bounds(R, self.config.nodes) if hi > lo]
        groups = partition_bounds(len(parts), G)
        owners = partition_bounds(n, G)
        devs = [self._dev(g) for g in range(G)]
        lib = _native.lib()
        for d in set(devs):
            for q in set(devs):
                if d != q:
                    _native.check(lib.pfw_peer_enable(d, q), "pfw_peer_enable")
        firsts = [torch.full((max(b - a, 1),), NO_MATCH, dtype=torch.int32, device=f"cuda:{d}")
                  for (a, b), d in zip(owners, devs)]
        comps = [torch.zeros(max(b - a, 1), dtype=torch.int32, device=f"cuda:{d}") for (a, b), d in zip(owners, devs)]
        stats = [torch.zeros(2, dtype=torch.int64, device=f"cuda:{d}") for d in devs]
        replicas = {}
        for d in set(devs):
            replicas[d] = pkts if pkts.device == d else PacketArrays(pkts.data.to(f"cuda:{d}"))
        for d in set(devs):
            torch.cuda.synchronize(d)  # every owner buffer is initialised before any scan writes into it
        P = ctypes.c_void_p
        tf = (P * G)(*[t.data_ptr() for t in firsts])
        tc = (P * G)(*[t.data_ptr() for t in comps])
        caps = (ctypes.c_int64 * G)(*[b - a for a, b in owners])
        for g, (ga, gb) in enumerate(groups):
            if gb == ga:
                continue
            lo_g, hi_g = parts[ga][0], parts[gb - 1][1]
            shard = self._copy(compiled, devs[g], lo_g, hi_g)
            st = torch.cuda.current_stream(devs[g]).cuda_stream
            for lo, hi in parts[ga:gb]:
                _native.check(lib.pfw_scan_fused_min(shard.handle, lo - lo_g, hi - lo_g, replicas[devs[g]].data.data_ptr(),
                                                     n, tf, tc, caps, G, 1, stats[g].data_ptr(), st),
                              "pfw_scan_fused_min")
        for d in set(devs):
            torch.cuda.synchronize(d)
        first = np.concatenate([first_to_host(f[:b - a]) for f, (a, b) in zip(firsts, owners)])
        comp = np.concatenate([c[:b - a].cpu().numpy() for c, (a, b) in zip(comps, owners)]).astype(np.int64)
        st = [s.cpu().numpy() for s in stats]
        return first, comp, np.array([sum(int(x[0]) for x in st), max(int(x[1]) for x in st)], np.int64)

    # ----------------------------------------------------------- drop-in
    def run(self, ruleset: Ruleset, packets: Sequence[Packet]) -> tuple[MatchResults, ClassifyStats]:
        """Classify packets under the configured model (engines.py:260-290).
        results[i] belongs to packets[i]; the results are an array-backed lazy
        sequence of MatchResult (equal to the reference's list)."""
        if self.config.model is ExecutionModel.SEQUENTIAL and self.gpus == 1:
            return classify_batch_sequential(ruleset, packets)
        start = time.perf_counter_ns()
        compiled = compile_ruleset(ruleset, self._dev(0))
        res = self.run_arrays(compiled, packets)
        results = compiled.build_results(res.first, res._comps) if len(res.first) else []
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
