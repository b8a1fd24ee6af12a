"""Pin the CPU oracle (oracle/) to the reference's golden vectors.

The golden fixtures were produced by the unmodified reference
(tests/golden/make_golden.py); every oracle function must reproduce them
bit-exactly before it is trusted as the checker for the CUDA path.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_rules, golden_traffic
from oracle import oracle
from oracle.oracle import PKT_FIELDS, RULE_FIELDS


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_rng_streams():
    g = golden("rng.npz")
    for seed, stream in zip(g["seeds"].tolist(), g["streams"]):
        np.testing.assert_array_equal(oracle.xs_stream(seed, 64), stream)
    for seed, row in zip(g["seeds"].tolist(), g["derive"]):
        assert [oracle.derive_seed(seed, k) for k in range(8)] == row.tolist()


RULESETS = ["r1000_s1", "r2048_s21_w15", "r300_s40_w30", "r100_s60_w35", "r503_s24_w30",
            "r64_s30_w40", "r4096_s1", "r10000_s1", "r100000_s1"]


@pytest.mark.parametrize("name", RULESETS)
def test_gen_ruleset_matches_reference(name):
    g = golden(f"rules_{name}.npz")
    rules = oracle.gen_ruleset(int(g["count"]), int(g["seed"]), float(g["wp"]))
    assert digest(*[rules[f] for f in RULE_FIELDS]) == str(g["sha256"])
    if "proto" in g:
        for f in RULE_FIELDS:
            np.testing.assert_array_equal(rules[f], g[f])


TRAFFIC = ["t100000_s2", "t1000_s22", "t10000_s41", "t150_s61", "t600_s25", "t2000_s7_dst0_1",
           "t2000_s8_dst192_2", "t5000_s9_ports", "t3000_s11_icmp"]


@pytest.mark.parametrize("name", TRAFFIC)
def test_gen_traffic_matches_reference(name):
    g = golden(f"traffic_{name}.npz")
    pk = golden_traffic(name)
    assert digest(*[pk[f] for f in PKT_FIELDS]) == str(g["sha256"])
    if "head_proto" in g:
        for f in PKT_FIELDS:
            np.testing.assert_array_equal(pk[f][: len(g[f"head_{f}"])], g[f"head_{f}"])


SCANS = [("oracle_r1000_t100000", "r1000_s1", "t100000_s2"),
         ("r2048_t1000", "r2048_s21_w15", "t1000_s22"),
         ("r300_t10000", "r300_s40_w30", "t10000_s41"),
         ("r64_t600", "r64_s30_w40", "t600_s25"),
         ("r1000_t5000ports", "r1000_s1", "t5000_s9_ports"),
         ("r1000_t3000icmp", "r1000_s1", "t3000_s11_icmp")]


@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_scan_matches_reference(name, rn, tn):
    g = golden(f"scan_{name}.npz")
    rules, pk = golden_rules(rn), golden_traffic(tn)
    R = len(rules["proto"])
    first = oracle.scan_range(rules, pk, 0, R)
    np.testing.assert_array_equal(first, g["first"])
    comps = oracle.sequential_comparisons(first, R)
    assert int(comps.sum()) == int(g["total_comparisons"])
    assert int(comps.max()) == int(g["max_worker_comparisons"])
    verdict = np.where(first >= 0, rules["action_accept"][np.maximum(first, 0)], False)
    np.testing.assert_array_equal(verdict, g["verdict"])


def test_oracle_config_total_comparisons():
    # 1,000 rules x 100K packets -> 69,698,223 comparisons
    assert int(golden("scan_oracle_r1000_t100000.npz")["total_comparisons"]) == 69_698_223


@pytest.mark.parametrize("rn", ["r4096_s1", "r10000_s1", "r100000_s1"])
def test_scan_config_samples(rn):
    g = golden(f"scan_{rn}_t20000.npz")
    rules = golden_rules(rn)
    pk = oracle.gen_traffic_uniform(20_000, 2)
    first = oracle.scan_range(rules, pk, 0, len(rules["proto"]))
    np.testing.assert_array_equal(first, g["first"])


def test_numpy_block_scan_equals_c_scan():
    rules, pk = golden_rules("r300_s40_w30"), golden_traffic("t10000_s41")
    for lo, hi in ((0, 300), (17, 53), (128, 300), (299, 300), (5, 5)):
        np.testing.assert_array_equal(oracle.scan_range_np(rules, pk, lo, hi),
                                      oracle.scan_range(rules, pk, lo, hi))


def test_scan_windows():
    g = golden("scan_windows_r100_t150.npz")
    rules, pk = golden_rules("r100_s60_w35"), golden_traffic("t150_s61")
    for (lo, hi), want in zip(g["windows"].tolist(), g["first"]):
        np.testing.assert_array_equal(oracle.scan_range(rules, pk, lo, hi), want)


@pytest.mark.parametrize("model", ["data", "function", "hybrid"])
def test_engine_models_r503(model):
    g = golden("engine_r503_t600.npz")
    rules, pk = golden_rules("r503_s24_w30"), golden_traffic("t600_s25")
    for nodes in (1, 2, 3, 4, 8, 16, 64, 512):
        first, comps, total, mx = oracle.engine_run(rules, pk, model, nodes)
        key = f"{model}_{nodes}"
        np.testing.assert_array_equal(first, g[f"{key}_first"])
        np.testing.assert_array_equal(comps, g[f"{key}_comps"])
        assert [total, mx, len(first)] == g[f"{key}_stats"].tolist()


def test_engine_function_parallel_100k():
    g = golden("engine_r100000_t2000.npz")
    rules = golden_rules("r100000_s1")
    pk = oracle.gen_traffic_uniform(2000, 2)
    for nodes in (1, 2, 4, 8):
        first, comps, total, mx = oracle.engine_run(rules, pk, "function", nodes)
        np.testing.assert_array_equal(first, g[f"function_{nodes}_first"])
        np.testing.assert_array_equal(comps, g[f"function_{nodes}_comps"])
        assert [total, mx, len(first)] == g[f"function_{nodes}_stats"].tolist()


def test_adversarial_recipe():
    g = golden("adversarial.npz")
    rules = oracle.adversarial_rules(50_000)
    pk = oracle.adversarial_traffic(20_000)
    assert digest(*[rules[f] for f in RULE_FIELDS]) == str(g["rules_sha256"])
    assert digest(*[pk[f] for f in PKT_FIELDS]) == str(g["traffic_sha256"])
    first = oracle.scan_range(rules, pk, 0, 50_000)
    np.testing.assert_array_equal(first, g["first"])
    comps = oracle.sequential_comparisons(first, 50_000)
    assert int(comps.sum()) == int(g["total_comparisons"])


def test_partition_bounds_kats():
    # test_engines.py:50-66
    assert [lo for lo, _ in oracle.partition_bounds(2048, 4)] == [0, 512, 1024, 1536]
    assert oracle.partition_bounds(5, 2) == [(0, 3), (3, 5)]
    assert [hi - lo for lo, hi in oracle.partition_bounds(3, 8)] == [1, 1, 1, 0, 0, 0, 0, 0]
