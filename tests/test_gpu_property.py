"""Property-based parity (hypothesis): random small rulesets / packet batches
drawn with heavy weight on boundary values -- ports 0 / 65535 / range ends,
prefixes /0, /1, /31, /32, bases with host bits (never-match under the
reference predicate), inverted port ranges, protocol 0 (ANY) and unusual
protocol numbers -- scanned over random windows under every layout option,
bit-exact against the oracle (classifier.py:146-162, model.py:222-230)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

import paper_1312_4188_b200 as pfw  # noqa: E402
from paper_1312_4188_b200 import _native  # noqa: E402
from oracle import oracle  # noqa: E402
from oracle.oracle import PKT_FIELDS, RULE_DTYPES, RULE_FIELDS  # noqa: E402

PORT = st.one_of(st.sampled_from([0, 1, 79, 80, 81, 1023, 1024, 65534, 65535]), st.integers(0, 65535))
IP = st.one_of(st.sampled_from([0, 1, 0x7FFFFFFF, 0x80000000, 0xC0000000, 0xFFFFFFFE, 0xFFFFFFFF,
                                0x0A000000, 0x0A0000FF]), st.integers(0, 0xFFFFFFFF))
PLEN = st.one_of(st.sampled_from([0, 1, 8, 16, 24, 31, 32]), st.integers(0, 32))
PROTO_RULE = st.sampled_from([0, 0, 1, 6, 17, 47, 255])
PROTO_PKT = st.sampled_from([1, 6, 17, 47, 255, 0])
EXAMPLES = int(os.environ.get("PFW_HYP_EXAMPLES", "90"))


@st.composite
def rules_and_packets(draw):
    R = draw(st.integers(1, 300))
    n = draw(st.integers(1, 400))
    cols = {f: np.zeros(R, dtype=d) for f, d in zip(RULE_FIELDS, RULE_DTYPES)}
    for i in range(R):
        cols["proto"][i] = draw(PROTO_RULE)
        for side in ("src", "dst"):
            plen = draw(PLEN)
            mask = 0 if plen == 0 else (0xFFFFFFFF << (32 - plen)) & 0xFFFFFFFF
            base = draw(IP)
            if not draw(st.booleans().filter(lambda _: True)) or draw(st.integers(0, 9)) > 0:
                base &= mask  # mostly normalised; sometimes host bits set (never matches)
            cols[f"{side}_base"][i], cols[f"{side}_mask"][i] = base, mask
        for side in ("sport", "dport"):
            a, b = draw(PORT), draw(PORT)
            if draw(st.integers(0, 19)) > 0:
                a, b = min(a, b), max(a, b)  # mostly well-formed; sometimes inverted
            cols[f"{side}_lo"][i], cols[f"{side}_hi"][i] = a, b
        cols["action_accept"][i] = draw(st.booleans())
    pk = {f: np.zeros(n, dtype=d) for f, d in zip(PKT_FIELDS, oracle.PKT_DTYPES)}
    for i in range(n):
        if draw(st.integers(0, 3)) == 0 and R:
            # aim at a rule's boundary: its base / range ends
            r = draw(st.integers(0, R - 1))
            pk["src_ip"][i] = cols["src_base"][r] | (draw(IP) & ~cols["src_mask"][r] & 0xFFFFFFFF)
            pk["dst_ip"][i] = cols["dst_base"][r] | (draw(IP) & ~cols["dst_mask"][r] & 0xFFFFFFFF)
            pk["src_port"][i] = draw(st.sampled_from([int(cols["sport_lo"][r]), int(cols["sport_hi"][r])]))
            pk["dst_port"][i] = draw(st.sampled_from([int(cols["dport_lo"][r]), int(cols["dport_hi"][r])]))
            pk["proto"][i] = cols["proto"][r] or draw(PROTO_PKT)
        else:
            pk["src_ip"][i], pk["dst_ip"][i] = draw(IP), draw(IP)
            pk["src_port"][i], pk["dst_port"][i] = draw(PORT), draw(PORT)
            pk["proto"][i] = draw(PROTO_PKT)
    lo = draw(st.integers(0, R))
    hi = draw(st.integers(lo, R))
    return cols, pk, lo, hi


@pytest.fixture(autouse=True)
def _reset():
    yield
    for k, v in (("proto_split", 0), ("first_pass", 1024), ("ks", 8), ("algo", 0), ("ms_group", 0), ("ms_words", 4),
                 ("ms_summary", 2), ("ms_compress", 2)):
        _native.set_tuning(k, v)


@settings(max_examples=EXAMPLES, deadline=None, suppress_health_check=list(HealthCheck))
@given(case=rules_and_packets(), mode=st.sampled_from(["matchset", "compressed", "rule", "split"]),
       fp=st.sampled_from([32, 64, 1024]),
       shape=st.sampled_from([(8, 4), (8, 2), (16, 4), (16, 2), (32, 2), (32, 1)]),
       summary=st.sampled_from([0, 1]))
def test_random_boundary_cases_bit_exact(case, mode, fp, shape, summary):
    """Match-set scan, rule-by-rule scan and protocol-split chains on the same
    boundary-heavy random cases."""
    cols, pk, lo, hi = case
    _native.set_tuning("algo", {"matchset": 2, "compressed": 2, "rule": 1, "split": 1}[mode])
    _native.set_tuning("ms_compress", 1 if mode == "compressed" else 2)
    _native.set_tuning("proto_split", int(mode == "split"))
    _native.set_tuning("first_pass", fp)
    _native.set_tuning("ms_summary", summary)
    _native.set_tuning("ms_group", shape[0])
    _native.set_tuning("ms_words", shape[1])
    c = pfw.CompiledRuleset.from_columns(cols, device=0)
    p = pfw.PacketArrays.from_columns(*[pk[f] for f in PKT_FIELDS], device=0)
    np.testing.assert_array_equal(c.scan_range(p, lo, hi), oracle.scan_range(cols, pk, lo, hi))
    np.testing.assert_array_equal(c.scan_range(p, 0, len(cols["proto"])),
                                  oracle.scan_range(cols, pk, 0, len(cols["proto"])))


@settings(max_examples=max(EXAMPLES // 3, 10), deadline=None, suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2**31 - 1), R=st.integers(1025, 12000), wp=st.floats(0.02, 0.6),
       cluster=st.floats(0.0, 0.95), mode=st.sampled_from(["plain", "compressed"]),
       summary=st.sampled_from([0, 1]), lo_f=st.floats(0.0, 1.0), len_f=st.floats(0.0, 1.0))
def test_multi_block_rulesets_bit_exact(seed, R, wp, cluster, mode, summary, lo_f, len_f):
    """Rulesets spanning several 1024-rule blocks (summaries, compressed rows,
    windows across blocks): a fraction of the rules is clustered into one dst
    half so block summaries can skip blocks; packets partly aimed at rule
    boundaries."""
    rng = np.random.default_rng(seed)
    cols = oracle.gen_ruleset(R, seed % 100_000 + 1, wp=wp)
    k = rng.random(R) < cluster
    cols["dst_mask"][k] = np.maximum(cols["dst_mask"][k], np.uint32(0x80000000))
    cols["dst_base"][k] = (cols["dst_base"][k] | np.uint32(0x80000000)) & cols["dst_mask"][k]
    pk = oracle.gen_traffic_uniform(3000, seed % 100_000 + 7)
    pk["dst_ip"][:2000] &= np.uint32(0x7FFFFFFF)          # mostly outside the clustered half
    r = rng.integers(0, R, 600)
    pk["src_ip"][2000:2600] = cols["src_base"][r]
    pk["dst_port"][2000:2600] = cols["dport_hi"][r]
    pk["src_port"][2600:] = cols["sport_lo"][rng.integers(0, R, 400)]
    lo = int(lo_f * R)
    hi = min(R, lo + int(len_f * R) + 1)
    _native.set_tuning("ms_compress", 1 if mode == "compressed" else 0)
    _native.set_tuning("ms_summary", summary)
    _native.set_tuning("algo", 2)
    c = pfw.CompiledRuleset.from_columns(cols, device=0)
    p = pfw.PacketArrays.from_columns(*[pk[f] for f in PKT_FIELDS], device=0)
    np.testing.assert_array_equal(c.scan_range(p, lo, hi), oracle.scan_range(cols, pk, lo, hi))
    np.testing.assert_array_equal(c.scan_range(p, 0, R), oracle.scan_range(cols, pk, 0, R))
