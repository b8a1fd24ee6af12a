"""First-match classification on the GPU (drop-in for ``parafw.classifier``).

Public surface mirrors /root/reference/pkg/src/parafw/classifier.py:
``ClassifyStats``, ``CompiledRuleset``, ``PacketArrays``, ``classify``,
``classify_batch_sequential``, ``compile_ruleset``.  The difference is where
the data lives and who scans it:

* ``CompiledRuleset`` keeps the reference's ten SoA columns on the host
  (classifier.py:120-134) and builds the device forms once
  (``pfw_ruleset_create``): the per-field match sets (interval bitmaps, plain
  or compressed rows) and the range-test table of the rule-by-rule scan.
  ``CompiledRuleset.shard`` uploads one rule partition on its own
  (function-parallel across GPUs: local windows, global indices).
* ``PacketArrays`` is a device-resident batch of 16-byte packet records
  {src_ip, dst_ip, sport<<16|dport, proto} (the packet-batch layout that
  replaces the five numpy columns of classifier.py:62-95).
* ``CompiledRuleset.scan_range`` (classifier.py:146-162) is one launch of the
  match-set scan (or, with tuning ``algo=1``, the multi-pass packet x rule
  grid); comparison counts and stats are produced in the kernel epilogue
  (classifier.py:200-208), bit-exact either way.

There is no CPU fallback: without libpfw.so or a CUDA device every scan
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from collections.abc import Sequence as _SequenceABC
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from ._native import NO_MATCH, check
from .model import Action, MatchResult, Packet, Protocol, Ruleset

__all__ = [
    "ClassifyStats",
    "CompiledRuleset",
    "MatchResults",
    "PacketArrays",
    "classify",
    "classify_batch_sequential",
    "compile_ruleset",
    "NO_MATCH",
]

RULE_COLUMNS = ("proto", "src_base", "src_mask", "sport_lo", "sport_hi",
                "dst_base", "dst_mask", "dport_lo", "dport_hi", "action_accept")
_RULE_DTYPES = (np.uint8, np.uint32, np.uint32, np.uint16, np.uint16,
                np.uint32, np.uint32, np.uint16, np.uint16, np.bool_)
PACKET_COLUMNS = ("proto", "src_ip", "src_port", "dst_ip", "dst_port")
_PACKET_DTYPES = (np.uint8, np.uint32, np.uint16, np.uint32, np.uint16)


def _torch():
    import torch
    return torch


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def _default_device() -> int:
    _native.require_device()
    torch = _torch()
    return torch.cuda.current_device()


def _stream(device: int) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


@dataclass(frozen=True)
class ClassifyStats:
    """Aggregate counters of one run (classifier.py:38-51)."""

    total_comparisons: int
    packets_processed: int
    wall_time_ns: int
    max_worker_comparisons: int


def classify(ruleset: Ruleset, packet: Packet) -> MatchResult:
    """First match with early exit, default deny (classifier.py:54-59), on the GPU."""
    compiled = compile_ruleset(ruleset)
    # one packet through the host pipeline's packed tiny-batch path (one copy each way)
    cols = {"proto": np.array([int(packet.proto)], np.uint8), "src_ip": np.array([packet.src_ip], np.uint32),
            "src_port": np.array([packet.src_port], np.uint16), "dst_ip": np.array([packet.dst_ip], np.uint32),
            "dst_port": np.array([packet.dst_port], np.uint16)}
    first, _, _ = compiled.classify_host(cols)
    idx = int(first[0])
    if idx < 0:
        return MatchResult(Action.DROP, None, compiled.num_rules)
    return MatchResult(Action.ACCEPT if compiled.action_accept[idx] else Action.DROP, idx, idx + 1)


class MatchResults(_SequenceABC):
    """Array-backed, lazy ``list[MatchResult]`` (classifier.py:175-185 without
    building N objects): ``results[i]`` is a MatchResult made on access from
    the first-match index array (-1 = default deny), the per-packet
    comparison counts and the ruleset's action column.  Compares equal to a
    list of the same MatchResults (the reference returns a list), so
    ``results == expected`` and ``results == []`` behave as in the reference.

    ``comparisons=None`` means the sequential / data-parallel count
    ``first + 1`` or ``num_rules`` (classifier.py:200), derived on access."""

    __slots__ = ("first", "_comps", "_accept", "_num_rules")

    def __init__(self, first, comparisons, action_accept, num_rules: int) -> None:
        self.first = np.asarray(first)
        self._comps = None if comparisons is None else np.asarray(comparisons)
        self._accept = action_accept
        self._num_rules = int(num_rules)

    @property
    def comparisons(self) -> np.ndarray:
        if self._comps is None:
            f = self.first.astype(np.int64)
            self._comps = np.where(f >= 0, f + 1, self._num_rules)
        return self._comps

    @property
    def verdict_accept(self) -> np.ndarray:
        f = self.first
        hit = f >= 0
        out = np.zeros(len(f), dtype=np.bool_)
        out[hit] = np.asarray(self._accept)[f[hit]]
        return out

    def __len__(self) -> int:
        return int(self.first.shape[0])

    def _make(self, idx: int, comps: int) -> MatchResult:
        if idx < 0:
            return MatchResult(Action.DROP, None, comps)
        return MatchResult(Action.ACCEPT if self._accept[idx] else Action.DROP, idx, comps)

    def __getitem__(self, i):
        if isinstance(i, slice):
            c = None if self._comps is None else self._comps[i]
            return MatchResults(self.first[i], c, self._accept, self._num_rules)
        n = len(self)
        i = int(i)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("MatchResults index out of range")
        f = int(self.first[i])
        c = int(self._comps[i]) if self._comps is not None else (f + 1 if f >= 0 else self._num_rules)
        return self._make(f, c)

    def __iter__(self):
        step = 1 << 16
        for a in range(0, len(self), step):
            fs = self.first[a:a + step].tolist()
            cs = self.comparisons[a:a + step].tolist()
            for f, c in zip(fs, cs):
                yield self._make(f, c)

    def tolist(self) -> list[MatchResult]:
        return list(iter(self))

    def __eq__(self, other) -> bool:
        if isinstance(other, MatchResults):
            return (len(self) == len(other) and np.array_equal(self.first, other.first)
                    and np.array_equal(self.comparisons, other.comparisons)
                    and np.array_equal(self.verdict_accept, other.verdict_accept))
        if isinstance(other, (list, tuple)):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    __hash__ = None

    def __repr__(self) -> str:
        head = ", ".join(repr(r) for r in self[:3])
        return f"MatchResults([{head}{', ...' if len(self) > 3 else ''}], n={len(self)})"


# ----------------------------------------------------------------- packets

class PacketArrays:
    """Device-resident packet batch: ``data`` is an int32 CUDA tensor [n, 4]
    holding {src_ip, dst_ip, sport<<16|dport, proto} per packet.

    Column attributes (``proto``, ``src_ip`` ...) are host numpy views
    decoded on demand, for compatibility with classifier.py:62-95.
    """

    __slots__ = ("data",)

    def __init__(self, data) -> None:
        torch = _torch()
        if not isinstance(data, torch.Tensor) or data.dtype != torch.int32 or data.dim() != 2 \
                or data.shape[1] != 4:
            raise TypeError("PacketArrays wraps an int32 tensor of shape [n, 4]")
        if not data.is_cuda:
            raise _native.NativeUnavailable("PacketArrays must live on a CUDA device")
        if not data.is_contiguous():
            data = data.contiguous()
        self.data = data

    # --- constructors
    @staticmethod
    def pack_host(proto, src_ip, src_port, dst_ip, dst_port) -> np.ndarray:
        """Host [n, 4] uint32 records from the five reference columns."""
        n = len(proto)
        out = np.empty((n, 4), dtype=np.uint32)
        out[:, 0] = np.asarray(src_ip, dtype=np.uint32)
        out[:, 1] = np.asarray(dst_ip, dtype=np.uint32)
        out[:, 2] = (np.asarray(src_port, dtype=np.uint32) << 16) | np.asarray(dst_port, dtype=np.uint32)
        out[:, 3] = np.asarray(proto, dtype=np.uint32)
        return out

    @staticmethod
    def unpack_host(records: np.ndarray) -> dict:
        """Inverse of pack_host: the five reference columns of [n, 4] records."""
        rec = np.asarray(records, dtype=np.uint32).reshape(-1, 4)
        return {"proto": rec[:, 3].astype(np.uint8), "src_ip": rec[:, 0].copy(),
                "src_port": (rec[:, 2] >> 16).astype(np.uint16), "dst_ip": rec[:, 1].copy(),
                "dst_port": (rec[:, 2] & 0xFFFF).astype(np.uint16)}

    @classmethod
    def from_host_records(cls, records: np.ndarray, device: int | None = None) -> "PacketArrays":
        torch = _torch()
        device = _default_device() if device is None else device
        rec = np.ascontiguousarray(records, dtype=np.uint32).reshape(-1, 4)
        t = torch.from_numpy(rec.view(np.int32))
        if rec.shape[0] >= (1 << 16):
            t = t.pin_memory()
        return cls(t.to(f"cuda:{device}", non_blocking=True))

    @classmethod
    def from_columns(cls, proto, src_ip, src_port, dst_ip, dst_port,
                     device: int | None = None) -> "PacketArrays":
        return cls.from_host_records(cls.pack_host(proto, src_ip, src_port, dst_ip, dst_port), device)

    @classmethod
    def from_packets(cls, packets: Sequence[Packet], device: int | None = None) -> "PacketArrays":
        """classifier.py:75-83, packed straight into 16-byte records."""
        n = len(packets)
        rec = np.empty((n, 4), dtype=np.uint32)
        if n:
            rec[:, 0] = np.fromiter((p.src_ip for p in packets), dtype=np.uint32, count=n)
            rec[:, 1] = np.fromiter((p.dst_ip for p in packets), dtype=np.uint32, count=n)
            rec[:, 2] = np.fromiter(((p.src_port << 16) | p.dst_port for p in packets), dtype=np.uint32,
                                    count=n)
            rec[:, 3] = np.fromiter((int(p.proto) for p in packets), dtype=np.uint32, count=n)
        return cls.from_host_records(rec, device)

    @classmethod
    def empty(cls, n: int, device: int | None = None) -> "PacketArrays":
        torch = _torch()
        device = _default_device() if device is None else device
        return cls(torch.empty((n, 4), dtype=torch.int32, device=f"cuda:{device}"))

    # --- views
    def __len__(self) -> int:
        return int(self.data.shape[0])

    @property
    def device(self) -> int:
        return int(self.data.device.index)

    def slice(self, start: int, stop: int) -> "PacketArrays":
        return PacketArrays(self.data[start:stop])

    def host_records(self) -> np.ndarray:
        return self.data.cpu().numpy().view(np.uint32)

    def columns(self) -> dict:
        rec = self.host_records()
        return {
            "proto": rec[:, 3].astype(np.uint8),
            "src_ip": rec[:, 0].copy(),
            "src_port": (rec[:, 2] >> 16).astype(np.uint16),
            "dst_ip": rec[:, 1].copy(),
            "dst_port": (rec[:, 2] & 0xFFFF).astype(np.uint16),
        }

    def to_packets(self) -> list[Packet]:
        c = self.columns()
        return [Packet(i, Protocol(int(pr)), int(s), int(sp), int(d), int(dp))
                for i, (pr, s, sp, d, dp) in enumerate(zip(c["proto"].tolist(), c["src_ip"].tolist(),
                                                          c["src_port"].tolist(), c["dst_ip"].tolist(),
                                                          c["dst_port"].tolist()))]

    def __getattr__(self, name):
        if name in PACKET_COLUMNS:
            return self.columns()[name]
        raise AttributeError(name)


# ------------------------------------------------------------------- rules

def _rule_columns(ruleset: Ruleset) -> dict:
    """classifier.py:120-134 column form of a Ruleset."""
    n = len(ruleset)
    rs = ruleset.rules
    return {
        "proto": np.fromiter((int(r.proto) for r in rs), dtype=np.uint8, count=n),
        "src_base": np.fromiter((r.src.base for r in rs), dtype=np.uint32, count=n),
        "src_mask": np.fromiter((r.src.mask for r in rs), dtype=np.uint32, count=n),
        "sport_lo": np.fromiter((r.sport.lo for r in rs), dtype=np.uint16, count=n),
        "sport_hi": np.fromiter((r.sport.hi for r in rs), dtype=np.uint16, count=n),
        "dst_base": np.fromiter((r.dst.base for r in rs), dtype=np.uint32, count=n),
        "dst_mask": np.fromiter((r.dst.mask for r in rs), dtype=np.uint32, count=n),
        "dport_lo": np.fromiter((r.dport.lo for r in rs), dtype=np.uint16, count=n),
        "dport_hi": np.fromiter((r.dport.hi for r in rs), dtype=np.uint16, count=n),
        "action_accept": np.fromiter((r.action is Action.ACCEPT for r in rs), dtype=np.bool_, count=n),
    }


def _host_packet_ptrs(packets):
    """Host packet batch -> (arrays kept alive, n, record pointer, 5 column
    pointers): a dict of the reference's PacketArrays columns or (n, 4)
    uint32 16-byte records."""
    if isinstance(packets, dict):
        arrs = [np.ascontiguousarray(packets[f], dtype=d) for f, d in zip(PACKET_COLUMNS, _PACKET_DTYPES)]
        n = len(arrs[0])
        for f, a in zip(PACKET_COLUMNS, arrs):
            if len(a) != n:
                raise ValueError(f"packet column {f} has {len(a)} entries, expected {n}")
        return arrs, n, None, [a.ctypes.data for a in arrs]
    rec = np.ascontiguousarray(packets, dtype=np.uint32).reshape(-1, 4)
    return [rec], rec.shape[0], rec.ctypes.data, [None] * 5


class CompiledRuleset:
    """Ruleset uploaded to one GPU (drop-in for classifier.py:98-185)."""

    def __init__(self, ruleset: Ruleset | None = None, device: int | None = None, *,
                 columns: dict | None = None, shard: tuple[int, int] | None = None) -> None:
        if (ruleset is None) == (columns is None):
            raise TypeError("pass exactly one of ruleset or columns")
        if columns is not None:
            cols = {f: np.ascontiguousarray(columns[f], dtype=d) for f, d in zip(RULE_COLUMNS, _RULE_DTYPES)}
        else:
            cols = _rule_columns(ruleset)
        n = len(cols["proto"])
        for f in RULE_COLUMNS:
            if len(cols[f]) != n:
                raise ValueError(f"rule column {f} has {len(cols[f])} entries, expected {n}")
            setattr(self, f, cols[f])
        self.num_rules = n
        self.device = _default_device() if device is None else int(device)
        acc_u8 = cols["action_accept"].astype(np.uint8)
        self._keep = [cols[f] for f in RULE_COLUMNS[:-1]] + [acc_u8]
        h = ctypes.c_void_p()
        check(_native.lib().pfw_ruleset_create(self.device, n, *[a.ctypes.data for a in self._keep],
                                                ctypes.byref(h)), "pfw_ruleset_create")
        self._h = h
        self._finalizer = weakref.finalize(self, _native.lib().pfw_ruleset_destroy, h)
        # rule shard (function-parallel, engines.py:316-321): these rules are
        # positions [index_base, index_base + n) of a ruleset of total_rules;
        # windows are local, reported indices global
        self.index_base, self.total_rules = 0, n
        if shard is not None:
            base, total = int(shard[0]), int(shard[1])
            check(_native.lib().pfw_ruleset_set_shard(h, base, total), "pfw_ruleset_set_shard")
            self.index_base, self.total_rules = base, total

    @classmethod
    def from_columns(cls, columns: dict, device: int | None = None,
                     shard: tuple[int, int] | None = None) -> "CompiledRuleset":
        return cls(None, device, columns=columns, shard=shard)

    def shard(self, lo: int, hi: int) -> "CompiledRuleset":
        """Rules [lo, hi) uploaded on their own (their own match sets): scans of
        the shard take local windows and report global rule indices."""
        lo, hi = int(lo), int(hi)
        if not 0 <= lo <= hi <= self.num_rules:
            raise ValueError(f"shard [{lo}, {hi}) outside a ruleset of {self.num_rules} rules")
        cols = {f: getattr(self, f)[lo:hi] for f in RULE_COLUMNS}
        return CompiledRuleset.from_columns(cols, self.device,
                                            shard=(self.index_base + lo, self.total_rules))

    @property
    def is_shard(self) -> bool:
        return self.total_rules != self.num_rules

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def close(self) -> None:
        self._finalizer()

    def columns(self) -> dict:
        return {f: getattr(self, f) for f in RULE_COLUMNS}

    # --- device scans -----------------------------------------------------
    def _packets(self, pkts) -> PacketArrays:
        if isinstance(pkts, PacketArrays):
            if pkts.device != self.device:
                return PacketArrays(pkts.data.to(f"cuda:{self.device}"))
            return pkts
        return PacketArrays.from_packets(pkts, self.device)

    def scan_range_device(self, pkts: PacketArrays, lo: int, hi: int, *, first=None, comps=None,
                          verdict=None, stats=None, stream: int | None = None):
        """One kernel launch: int32 first-match tensor (NO_MATCH = none) on the device.
        Optional device outputs: ``comps`` (int32), ``verdict`` (uint8), ``stats``
        (int64 [2]: += sum of comps, max= max comps)."""
        torch = _torch()
        pkts = self._packets(pkts)
        n = len(pkts)
        if first is None:
            first = torch.empty(n, dtype=torch.int32, device=pkts.data.device)
        lo, hi = int(lo), int(hi)
        if lo > hi:
            lo = hi
        st = _stream(self.device) if stream is None else stream
        check(_native.lib().pfw_scan_range(self._h, lo, hi, _ptr(pkts.data), n, _ptr(first),
                                           _ptr(comps), _ptr(verdict), _ptr(stats), st),
              "pfw_scan_range")
        return first

    def scan_range_columns_device(self, cols: dict, lo: int, hi: int, *, first=None, comps=None,
                                  verdict=None, stats=None, stream: int | None = None):
        """scan_range over the reference's own column layout on the device:
        ``cols`` maps proto / src_ip / src_port / dst_ip / dst_port to CUDA
        tensors (uint8, int32/uint32, int16/uint16 bit patterns) -- no packing."""
        torch = _torch()
        n = int(cols["proto"].numel())
        if first is None:
            first = torch.empty(n, dtype=torch.int32, device=cols["proto"].device)
        lo, hi = int(lo), int(hi)
        if lo > hi:
            lo = hi
        st = _stream(self.device) if stream is None else stream
        check(_native.lib().pfw_scan_range_columns(
            self._h, lo, hi, _ptr(cols["proto"]), _ptr(cols["src_ip"]), _ptr(cols["src_port"]),
            _ptr(cols["dst_ip"]), _ptr(cols["dst_port"]), n, _ptr(first), _ptr(comps), _ptr(verdict),
            _ptr(stats), st), "pfw_scan_range_columns")
        return first

    def classify_host(self, packets, chunk: int = 1 << 23, out=None):
        """End-to-end first match over HOST packets, returned in host memory.

        ``packets``: a dict of the reference's PacketArrays columns (numpy:
        proto, src_ip, src_port, dst_ip, dst_port; classifier.py:62-95), or an
        (n, 4) uint32 array of 16-byte records.  Pinned inputs are copied by
        DMA directly; pageable ones are staged chunk by chunk through the
        handle's pinned ring by the native host thread pool -- either way
        host copies, device copies and scans overlap (pfw_classify_host_ex).

        Returns (first int32 [-1 = default deny], verdict bool, stats int64
        [sum, max] of the sequential comparison counts).  The outputs live in
        pinned memory from torch's caching host allocator (reused across
        calls), so results land by DMA with no staging copy; ``out`` = (first
        int32, verdict uint8 or bool) host arrays to write instead."""
        torch = _torch()
        arrs, n, rec_ptr, col_ptrs = _host_packet_ptrs(packets)
        if out is None:
            first = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
            verdict = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy().view(np.bool_)
        else:
            first, verdict = out
            if first.dtype != np.int32 or verdict.dtype.itemsize != 1 or len(first) != n or len(verdict) != n \
                    or not first.flags.c_contiguous or not verdict.flags.c_contiguous:
                raise ValueError("out must be contiguous (int32[n], uint8/bool[n]) host arrays")
        stats = np.zeros(2, dtype=np.uint64)
        check(_native.lib().pfw_classify_host_ex(self._h, rec_ptr, *col_ptrs, n, first.ctypes.data,
                                                 verdict.ctypes.data, stats.ctypes.data, chunk,
                                                 _native.HOST_FIRST_MINUS1), "pfw_classify_host_ex")
        return first, verdict, stats.astype(np.int64)

    def classify_host_partitions(self, packets, nodes: int, chunk: int = 1 << 23):
        """classify_host for the function-parallel / hybrid models over
        partition_bounds(R, nodes) (engines.py:316-369): the same chunked
        H2D / scan / D2H pipeline, each chunk scanned by every node partition
        and folded on the device.  Returns (first int32 [-1 = default deny],
        comparisons int32 [sum over nodes], verdict bool, stats int64 [sum,
        largest per-node count])."""
        torch = _torch()
        arrs, n, rec_ptr, col_ptrs = _host_packet_ptrs(packets)
        first = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        comps = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        verdict = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy().view(np.bool_)
        stats = np.zeros(2, dtype=np.uint64)
        check(_native.lib().pfw_classify_host_partitions(self._h, int(nodes), rec_ptr, *col_ptrs, n,
                                                         first.ctypes.data, comps.ctypes.data, verdict.ctypes.data,
                                                         stats.ctypes.data, chunk, _native.HOST_FIRST_MINUS1),
              "pfw_classify_host_partitions")
        del arrs
        return first, comps, verdict, stats.astype(np.int64)

    def classify_host_columns(self, cols: dict, chunk: int = 1 << 23):
        """classify_host over the five columns, first as int64 (scan_range's dtype)."""
        f, v, st = self.classify_host(cols, chunk)
        return f.astype(np.int64), v.copy(), st

    def scan_partition_accumulate(self, pkts: PacketArrays, lo: int, hi: int, first, comps, stats=None,
                                  stream: int | None = None) -> None:
        """Function-parallel / hybrid partition task folded into running min / sums."""
        st = _stream(self.device) if stream is None else stream
        check(_native.lib().pfw_scan_partition_accumulate(self._h, int(lo), int(hi), _ptr(pkts.data),
                                                          len(pkts), _ptr(first), _ptr(comps),
                                                          _ptr(stats), st),
              "pfw_scan_partition_accumulate")

    def scan_partitions(self, pkts: PacketArrays, nodes: int, first, comps, stats=None,
                        stream: int | None = None) -> None:
        """Every node of the function-parallel / hybrid models over
        partition_bounds(R, nodes) (engines.py:349-369) in one call: first =
        the lowest node's match, comps = the sum over nodes, stats += [sum,
        largest per-node count]."""
        st = _stream(self.device) if stream is None else stream
        check(_native.lib().pfw_scan_partitions(self._h, int(nodes), _ptr(pkts.data), len(pkts), _ptr(first),
                                                _ptr(comps), _ptr(stats), st),
              "pfw_scan_partitions")

    def verdicts_device(self, first, verdict=None, stream: int | None = None):
        torch = _torch()
        if verdict is None:
            verdict = torch.empty(first.numel(), dtype=torch.uint8, device=first.device)
        st = _stream(self.device) if stream is None else stream
        check(_native.lib().pfw_verdicts(self._h, _ptr(first), first.numel(), _ptr(verdict), st),
              "pfw_verdicts")
        return verdict

    # --- reference-shaped API ---------------------------------------------
    def scan_range(self, pkts, lo: int, hi: int) -> np.ndarray:
        """Earliest matching rule index in [lo, hi) per packet, or -1 (int64, host)."""
        pkts = self._packets(pkts)
        if len(pkts) == 0:
            return np.full(0, -1, dtype=np.int64)
        first = self.scan_range_device(pkts, lo, hi)
        return first_to_host(first)

    def first_match(self, packet: Packet) -> int:
        return int(self.scan_range([packet], 0, self.num_rules)[0])

    def build_results(self, first: np.ndarray, comparisons) -> MatchResults:
        """MatchResults from first-match indices and counts (classifier.py:175-185),
        array-backed: MatchResult objects are made only when accessed."""
        return MatchResults(first, comparisons, self.action_accept, self.num_rules)


def first_to_host(first) -> np.ndarray:
    """int32 device first-match tensor -> int64 host array with -1 for no match."""
    f = first.cpu().numpy().astype(np.int64)
    f[f == NO_MATCH] = -1
    return f


# one compiled copy per live Ruleset object (the reference recompiles per
# call; uploading 100K rules per call would dominate small batches)
_cache: dict[tuple[int, int], tuple] = {}


def compile_ruleset(ruleset: Ruleset, device: int | None = None) -> CompiledRuleset:
    device = _default_device() if device is None else int(device)
    key = (id(ruleset), device)
    hit = _cache.get(key)
    if hit is not None and hit[0]() is ruleset:
        return hit[1]
    compiled = CompiledRuleset(ruleset, device)
    try:
        ref = weakref.ref(ruleset, lambda _r, k=key: _cache.pop(k, None))
    except TypeError:
        return compiled
    _cache[key] = (ref, compiled)
    return compiled


def classify_batch_sequential(ruleset: Ruleset, packets) -> tuple[list[MatchResult], ClassifyStats]:
    """Classify a batch in packet order (classifier.py:192-209) on the GPU.

    ``packets`` may be a sequence of Packet (drop-in) or a PacketArrays."""
    torch = _torch()
    start = time.perf_counter_ns()
    compiled = compile_ruleset(ruleset)
    pkts = compiled._packets(packets)
    n = len(pkts)
    R = compiled.num_rules
    if n == 0:
        return [], ClassifyStats(0, 0, time.perf_counter_ns() - start, 0)
    dev = pkts.data.device
    comps = torch.empty(n, dtype=torch.int32, device=dev)
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    first = compiled.scan_range_device(pkts, 0, R, comps=comps, stats=stats)
    first_h = first_to_host(first)
    comps_h = comps.cpu().numpy().astype(np.int64)
    st = stats.cpu().numpy()
    results = compiled.build_results(first_h, comps_h)
    wall = time.perf_counter_ns() - start
    return results, ClassifyStats(int(st[0]), n, wall, int(st[1]))
