"""CPU oracle for the packet-filter hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference ``parafw`` algorithm (/root/reference/pkg/src/parafw)
in numpy (small cases, combine/partition logic) and in C (``fw_oracle.c``,
loaded through ctypes, for full-size parity and the CPU baseline).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this module, and only as the checker / the CPU arm -- never as the product
path.  Parity is pinned: ``tests/test_oracle.py`` checks every function here
against the golden vectors that the unmodified reference produced
(``tests/golden/make_golden.py``).

Citations are ``parafw/<file>:<line>``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

RULE_FIELDS = ("proto", "src_base", "src_mask", "sport_lo", "sport_hi",
               "dst_base", "dst_mask", "dport_lo", "dport_hi", "action_accept")
RULE_DTYPES = (np.uint8, np.uint32, np.uint32, np.uint16, np.uint16,
               np.uint32, np.uint32, np.uint16, np.uint16, np.bool_)
PKT_FIELDS = ("proto", "src_ip", "src_port", "dst_ip", "dst_port")
PKT_DTYPES = (np.uint8, np.uint32, np.uint16, np.uint32, np.uint16)

_lib = None


def build() -> str:
    """Compile fw_oracle.c (gcc, no external deps) into oracle/liboracle.so."""
    subprocess.run(["make", "-s", "-C", HERE, "CC=gcc"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, u64, i32, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_derive_seed.restype = u64
        L.orc_derive_seed.argtypes = [u64, u64]
        L.orc_xs_stream.argtypes = [u64, i64, P]
        L.orc_gen_traffic_uniform.argtypes = [u64, i64, i32, ctypes.c_uint32, i32, ctypes.c_uint32,
                                              i32, i32, i32, i32, i32, P, P, P, P, P]
        L.orc_gen_ruleset.argtypes = [i64, u64, dbl, dbl] + [P] * 10
        L.orc_scan_range.argtypes = [P] * 9 + [i64] + [P] * 5 + [i64, i64, P, i32]
        L.orc_max_threads.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------- rng

def xs_stream(seed: int, n: int) -> np.ndarray:
    """First n outputs of Xorshift64Star(seed) (rng.py:38-52)."""
    out = np.empty(n, dtype=np.uint64)
    lib().orc_xs_stream(seed & (2**64 - 1), n, _ptr(out))
    return out


def derive_seed(seed: int, stream: int) -> int:
    """rng.py:79-81"""
    return int(lib().orc_derive_seed(seed & (2**64 - 1), stream & (2**64 - 1)))


# ------------------------------------------------------------- generators

def gen_traffic_uniform(count, seed, proto=6, src_base=0, src_plen=0, dst_base=0, dst_plen=0,
                        sport_lo=0, sport_hi=65535, dport_lo=0, dport_hi=65535) -> dict:
    """generate_traffic(TrafficProfile(...UNIFORM)) as PacketArrays columns
    (traffic.py:117-130, 148-160; classifier.py:75-83)."""
    out = {f: np.empty(count, dtype=d) for f, d in zip(PKT_FIELDS, PKT_DTYPES)}
    lib().orc_gen_traffic_uniform(seed & (2**64 - 1), count, proto, src_base, src_plen, dst_base,
                                  dst_plen, sport_lo, sport_hi, dport_lo, dport_hi,
                                  *[_ptr(out[f]) for f in PKT_FIELDS])
    return out


def gen_ruleset(count, seed, wp=0.1, action_split=0.5) -> dict:
    """generate_ruleset(RulesetGenParams(...)) as CompiledRuleset columns
    (traffic.py:194-229; classifier.py:120-134)."""
    out = {f: np.empty(count, dtype=d) for f, d in zip(RULE_FIELDS, RULE_DTYPES)}
    acc = np.empty(count, dtype=np.uint8)
    ptrs = [_ptr(out[f]) for f in RULE_FIELDS[:-1]] + [_ptr(acc)]
    lib().orc_gen_ruleset(count, seed & (2**64 - 1), wp, action_split, *ptrs)
    out["action_accept"] = acc.astype(np.bool_)
    return out


# ------------------------------------------------------------------- scan

def scan_range(rules: dict, pkts: dict, lo: int, hi: int, threads: int = 0) -> np.ndarray:
    """CompiledRuleset.scan_range (classifier.py:146-162) in C: earliest match
    in [lo, hi) per packet, int64, -1 for none."""
    n = len(pkts["proto"])
    first = np.empty(n, dtype=np.int64)
    if n == 0:
        return first
    r = [np.ascontiguousarray(rules[f], dtype=d) for f, d in zip(RULE_FIELDS[:-1], RULE_DTYPES[:-1])]
    p = [np.ascontiguousarray(pkts[f], dtype=d) for f, d in zip(PKT_FIELDS, PKT_DTYPES)]
    lib().orc_scan_range(*[_ptr(a) for a in r], n, *[_ptr(a) for a in p], lo, hi, _ptr(first),
                         threads)
    return first


def match_block_np(rules: dict, pkts: dict, b0: int, b1: int) -> np.ndarray:
    """CompiledRuleset._match_block (classifier.py:136-144), numpy."""
    sl = slice(b0, b1)
    rp = rules["proto"][sl][:, None]
    m = (rp == 0) | (rp == pkts["proto"])
    m &= (pkts["src_ip"] & rules["src_mask"][sl][:, None]) == rules["src_base"][sl][:, None]
    m &= (pkts["src_port"] >= rules["sport_lo"][sl][:, None]) & (pkts["src_port"] <= rules["sport_hi"][sl][:, None])
    m &= (pkts["dst_ip"] & rules["dst_mask"][sl][:, None]) == rules["dst_base"][sl][:, None]
    m &= (pkts["dst_port"] >= rules["dport_lo"][sl][:, None]) & (pkts["dst_port"] <= rules["dport_hi"][sl][:, None])
    return m


def scan_range_np(rules: dict, pkts: dict, lo: int, hi: int, block: int = 128) -> np.ndarray:
    """scan_range (classifier.py:146-162), numpy block form, for small cases."""
    n = len(pkts["proto"])
    first = np.full(n, -1, dtype=np.int64)
    if lo >= hi or n == 0:
        return first
    unmatched = np.ones(n, dtype=np.bool_)
    for b0 in range(lo, hi, block):
        b1 = min(b0 + block, hi)
        m = match_block_np(rules, pkts, b0, b1)
        hit = m.any(axis=0)
        new = hit & unmatched
        if new.any():
            first[new] = b0 + m.argmax(axis=0)[new]
            unmatched &= ~hit
            if not unmatched.any():
                break
    return first


# ------------------------------------------------------ engine-level logic

def partition_bounds(total: int, parts: int) -> list[tuple[int, int]]:
    """engines.py:143-154"""
    base, extra = divmod(total, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def combine_partition_matches(local_first: np.ndarray, num_rules: int) -> np.ndarray:
    """engines.py:202-212"""
    if local_first.size == 0:
        return np.full(local_first.shape[-1] if local_first.ndim > 1 else 0, -1, dtype=np.int64)
    masked = np.where(local_first >= 0, local_first, num_rules)
    best = masked.min(axis=0)
    return np.where(best < num_rules, best, -1)


def sequential_comparisons(first: np.ndarray, num_rules: int) -> np.ndarray:
    """classifier.py:200 / engines.py:312: first+1, or R on a miss."""
    return np.where(first >= 0, first + 1, num_rules)


def engine_run(rules: dict, pkts: dict, model: str, nodes: int, threads: int = 0):
    """Engine.run (engines.py:260-369) result arrays: (first, comps, total, max_worker).
    Batching (engines.py:277-282) is invisible in results, so it is not restated."""
    R = len(rules["proto"])
    n = len(pkts["proto"])
    if model in ("sequential", "data"):
        first = scan_range(rules, pkts, 0, R, threads) if n else np.zeros(0, np.int64)
        comps = sequential_comparisons(first, R)
        return first, comps, int(comps.sum()), int(comps.max()) if n else 0
    parts = [(lo, hi) for lo, hi in partition_bounds(R, nodes) if hi > lo]
    if not parts:
        return np.full(n, -1, np.int64), np.zeros(n, np.int64), 0, 0
    local = np.stack([scan_range(rules, pkts, lo, hi, threads) for lo, hi in parts])
    first = combine_partition_matches(local, R)
    lows = np.array([lo for lo, _ in parts], dtype=np.int64)[:, None]
    sizes = np.array([hi - lo for lo, hi in parts], dtype=np.int64)[:, None]
    per_task = np.where(local >= 0, local - lows + 1, sizes)          # engines.py:366
    comps = per_task.sum(axis=0)
    return first, comps, int(comps.sum()), int(per_task.max()) if n else 0


def max_threads() -> int:
    return int(lib().orc_max_threads())


# --------------------------------------------------- adversarial recipe

def adversarial_rules(total: int = 50_000) -> dict:
    """SURVEY 8(d) adversarial ruleset (rule 0 ACCEPT any->192.0.0.0/2, 45K
    decoys forced into 128.0.0.0/1, 5K random tail), column form."""
    n_decoy = int(total * 0.9)
    head = {f: np.zeros(1, dtype=d) for f, d in zip(RULE_FIELDS, RULE_DTYPES)}
    head["dst_base"][0] = 0xC0000000
    head["dst_mask"][0] = 0xC0000000
    head["sport_hi"][0] = 65535
    head["dport_hi"][0] = 65535
    head["action_accept"][0] = True
    dec = gen_ruleset(n_decoy, 2)
    wild = dec["dst_mask"] == 0
    dec["dst_base"] = np.where(wild, np.uint32(0x80000000), dec["dst_base"] | np.uint32(0x80000000)).astype(np.uint32)
    dec["dst_mask"] = np.where(wild, np.uint32(0x80000000), dec["dst_mask"]).astype(np.uint32)
    tail = gen_ruleset(total - 1 - n_decoy, 1)
    return {f: np.concatenate([head[f], dec[f], tail[f]]) for f in RULE_FIELDS}


def adversarial_traffic(n: int) -> dict:
    n_late = int(n * 0.9)
    late = gen_traffic_uniform(n_late, 7, dst_base=0, dst_plen=1)
    early = gen_traffic_uniform(n - n_late, 8, dst_base=0xC0000000, dst_plen=2)
    return {f: np.concatenate([late[f], early[f]]) for f in PKT_FIELDS}
