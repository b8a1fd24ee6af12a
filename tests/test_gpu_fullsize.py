"""Full-size parity: every BASELINE.json configuration at its full size, the
CUDA path against the C oracle (all host threads), bit-exact on every packet:
first-match index, verdict, and the comparison counters -- for both scans
(the match-set scan and the rule-by-rule scan) against one oracle answer.

    data-parallel 10K rules x 64Mi packets, grid 4096 x 16Mi, function-parallel
    100K rules x 16Mi (G = 1 and the 8-way partitioned model on a subsample),
    adversarial 50K rules x 4Mi, oracle config 1000 x 100K.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1312_4188_b200 as pfw  # noqa: E402
from paper_1312_4188_b200 import _native, workloads  # noqa: E402
from paper_1312_4188_b200.classifier import NO_MATCH  # noqa: E402
from oracle import oracle  # noqa: E402


def gpu_scan(c, p):
    import torch
    n = len(p)
    verdict = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    first = c.scan_range_device(p, 0, c.num_rules, verdict=verdict, stats=stats)
    f = first.cpu().numpy().astype(np.int64)
    f[f == NO_MATCH] = -1
    return f, verdict.cpu().numpy(), stats.cpu().tolist()


@pytest.mark.parametrize("name", ["oracle", "grid", "data", "adversarial", "function"])
def test_baseline_config_full_size_bit_exact(name):
    w = workloads.WORKLOADS[name]
    cols = workloads.rule_columns(w)
    c = pfw.CompiledRuleset.from_columns(cols, device=0)
    assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) > 0
    p = workloads.packets(w, 0, w.packets, 0)
    host = p.columns()
    # the device generator reproduces the reference stream (oracle C generator)
    if name == "adversarial":
        ref_pk = oracle.adversarial_traffic(w.packets)
    else:
        ref_pk = oracle.gen_traffic_uniform(w.packets, 2)
    for f in oracle.PKT_FIELDS:
        np.testing.assert_array_equal(host[f], ref_pk[f])
    want = oracle.scan_range(cols, ref_pk, 0, w.rules)
    acc = np.zeros(len(want), np.uint8)
    hit = want >= 0
    acc[hit] = cols["action_accept"][want[hit]]
    comps = oracle.sequential_comparisons(want, w.rules)
    try:
        for algo in (0, 1):  # match-set scan, rule-by-rule scan
            _native.set_tuning("algo", algo)
            got, verdict, stats = gpu_scan(c, p)
            np.testing.assert_array_equal(got, want)
            np.testing.assert_array_equal(verdict, acc)
            assert stats == [int(comps.sum()), int(comps.max())]
    finally:
        _native.set_tuning("algo", 0)


def test_function_parallel_8_partitions_full_rules():
    """100K rules split 8 ways (the 8-GPU function-parallel model) on 1Mi packets:
    the partitioned scan + min/sum combine equals the oracle's engine model."""
    w = workloads.WORKLOADS["function"]
    cols = workloads.rule_columns(w)
    c = pfw.CompiledRuleset.from_columns(cols, device=0)
    n = 1 << 20
    p = workloads.packets(w, 0, n, 0)
    res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=8)).run_arrays(c, p)
    ref_pk = oracle.gen_traffic_uniform(n, 2)
    first, comps, total, mx = oracle.engine_run(cols, ref_pk, "function", 8)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.comparisons, comps)
    assert (res.stats.total_comparisons, res.stats.max_worker_comparisons) == (total, mx)


def test_more_than_2g_packets():
    """A batch of 2^31 + 5 packets (32 GB of records): packet ids past INT32_MAX
    through the match-set scan; a strided subsample against the oracle plus
    the comparison checksum on every packet."""
    import torch
    n = (1 << 31) + 5
    free, _ = torch.cuda.mem_get_info(0)
    if free < n * 16 + n * 4 + (8 << 30):
        pytest.skip("not enough device memory")
    rules = oracle.gen_ruleset(1000, 1)
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    first = c.scan_range_device(p, 0, 1000, stats=stats)
    idx = np.concatenate([np.arange(0, n, 1 << 20), np.arange(n - 4097, n)])
    sub = pfw.PacketArrays(p.data[torch.as_tensor(idx, device="cuda:0")]).columns()
    got = first[torch.as_tensor(idx, device="cuda:0")].cpu().numpy().astype(np.int64)
    got[got == NO_MATCH] = -1
    np.testing.assert_array_equal(got, oracle.scan_range(rules, sub, 0, 1000))
    f = first.to(torch.int64)
    comps = torch.where(f == NO_MATCH, torch.full_like(f, 1000), f + 1)
    assert stats.cpu().tolist() == [int(comps.sum().item()), int(comps.max().item())]
