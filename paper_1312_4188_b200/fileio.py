"""Array readers / writers for the on-disk formats.

``load_ruleset_columns`` and ``load_traffic_arrays`` read the reference's
ruleset text and traffic CSV formats natively (hostio.cpp) straight into the
CompiledRuleset columns / the 16-byte device packet layout, so file-driven
runs at scale never build Rule / Packet objects.  A file the strict native
parser does not accept is re-read by the reference-compatible Python parser
(model.load_ruleset / traffic.load_traffic): the result is identical to the
reference's for every input, including its exact errors.
``format_results`` writes the CLI's ``id,VERDICT,index`` lines natively.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native

__all__ = ["load_ruleset_columns", "parse_traffic", "load_traffic_arrays", "format_results"]

_RULE_DTYPES = (np.uint8, np.uint32, np.uint32, np.uint16, np.uint16, np.uint32, np.uint32, np.uint16,
                np.uint16, np.uint8)
_RULE_COLUMNS = ("proto", "src_base", "src_mask", "sport_lo", "sport_hi", "dst_base", "dst_mask",
                 "dport_lo", "dport_hi", "action_accept")


def _read(path) -> bytes:
    with open(path, "rb") as fh:
        return fh.read()


def load_ruleset_columns(path) -> dict:
    """Ruleset file -> CompiledRuleset columns (model.py:319-331 semantics)."""
    data = _read(path)
    cap = data.count(b"\n") + 1
    cols = [np.empty(cap, dtype=d) for d in _RULE_DTYPES]
    n = ctypes.c_int64()
    rc = _native.lib().pfw_parse_rules(data, len(data), cap, *[c.ctypes.data for c in cols], ctypes.byref(n))
    if rc == _native.PFW_OK:
        out = {f: c[: n.value].copy() for f, c in zip(_RULE_COLUMNS, cols)}
        out["action_accept"] = out["action_accept"].astype(np.bool_)
        return out
    from .classifier import _rule_columns
    from .model import load_ruleset
    return _rule_columns(load_ruleset(path))  # exact reference behaviour / errors


def parse_traffic(path):
    """Traffic CSV -> (ids int64 [n], host records uint32 [n, 4]) (traffic.py:259-297)."""
    from .classifier import PacketArrays
    data = _read(path)
    cap = data.count(b"\n") + 1
    ids = np.empty(cap, dtype=np.int64)
    rec = np.empty((cap, 4), dtype=np.uint32)
    n = ctypes.c_int64()
    rc = _native.lib().pfw_parse_traffic(data, len(data), cap, ids.ctypes.data, rec.ctypes.data,
                                         ctypes.byref(n))
    if rc == _native.PFW_OK:
        return ids[: n.value].copy(), rec[: n.value].copy()
    from .traffic import load_traffic
    packets = load_traffic(path)  # exact reference behaviour / errors
    ids = np.fromiter((p.id for p in packets), dtype=np.int64, count=len(packets))
    rec = PacketArrays.pack_host([int(p.proto) for p in packets], [p.src_ip for p in packets],
                                 [p.src_port for p in packets], [p.dst_ip for p in packets],
                                 [p.dst_port for p in packets])
    return ids, rec


def load_traffic_arrays(path, device: int | None = None):
    """Traffic CSV -> (ids int64, device PacketArrays)."""
    from .classifier import PacketArrays
    ids, rec = parse_traffic(path)
    return ids, PacketArrays.from_host_records(rec, device)


def format_results(ids: np.ndarray, first_raw: np.ndarray, verdict: np.ndarray) -> bytes:
    """``id,VERDICT,index|-`` lines (cli.py:62-65); first_raw holds uint32
    indices with PFW_NO_MATCH for default deny."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    first = np.ascontiguousarray(first_raw, dtype=np.uint32)
    verd = np.ascontiguousarray(verdict, dtype=np.uint8)
    n = len(ids)
    buf = ctypes.create_string_buffer(n * 48 + 64)
    w = ctypes.c_int64()
    _native.check(_native.lib().pfw_format_results(ids.ctypes.data, first.ctypes.data, verd.ctypes.data,
                                                   n, buf, len(buf), ctypes.byref(w)), "pfw_format_results")
    return buf.raw[: w.value]
