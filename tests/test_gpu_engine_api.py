"""The drop-in Engine API beyond one device and one layout:
host batches through the e2e pipeline (pinned and pageable numpy, columns and
records), the lazy MatchResult sequence, and one Engine driving several
devices (``devices=`` / ``EngineConfig.gpus``) -- all bit-exact against the
reference's golden results.

Several-device runs use the same device listed more than once where only
one GPU is visible: the shard / owner / fused-combine logic is identical
(peer pointers are then local), so this checks it on any box; the
``device_count() >= 2`` tests (tests/test_gpu_multidevice.py) cover real
NVLink peers."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_rules, golden_traffic

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1312_4188_b200 as pfw  # noqa: E402
from paper_1312_4188_b200 import _native  # noqa: E402
from paper_1312_4188_b200.classifier import MatchResults, first_to_host  # noqa: E402
from oracle import oracle  # noqa: E402
from oracle.oracle import PKT_FIELDS  # noqa: E402


def _pinned(cols):
    out = {}
    for f in PKT_FIELDS:
        a = np.ascontiguousarray(cols[f])
        t = torch.empty(a.shape, dtype={1: torch.uint8, 2: torch.int16, 4: torch.int32}[a.itemsize], pin_memory=True)
        t.numpy().view(a.dtype)[:] = a
        out[f] = t.numpy().view(a.dtype)
    return out


@pytest.mark.parametrize("layout", ["pageable", "pinned", "records"])
def test_run_arrays_host_batch_equals_golden(layout):
    g = golden("scan_oracle_r1000_t100000.npz")
    c = pfw.CompiledRuleset.from_columns(golden_rules("r1000_s1"), device=0)
    pk = golden_traffic("t100000_s2")
    if layout == "pinned":
        pk = _pinned(pk)
    elif layout == "records":
        pk = pfw.PacketArrays.pack_host(*[pk[f] for f in PKT_FIELDS])
    eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.DATA_PARALLEL))
    for _ in range(2):  # second call reuses the staging ring and pinned outputs
        res = eng.run_arrays(c, pk)
        np.testing.assert_array_equal(res.first, g["first"])
        np.testing.assert_array_equal(res.verdict_accept, g["verdict"])
        assert res.stats.total_comparisons == int(g["total_comparisons"]) == int(res.comparisons.sum())
        assert res.stats.max_worker_comparisons == int(g["max_worker_comparisons"])


@pytest.mark.parametrize("model", ["function", "hybrid"])
@pytest.mark.parametrize("layout", ["pageable", "pinned", "records"])
def test_run_arrays_host_batch_partitioned_models(model, layout):
    """Function-parallel / hybrid with a host batch: the chunked H2D / scan /
    D2H pipeline with every node partition folded on the device per chunk
    (pfw_classify_host_partitions) -- first, per-packet comparisons, verdicts
    and stats equal the reference's goldens for every node count."""
    g = golden("engine_r503_t600.npz")
    rules, traffic = golden_rules("r503_s24_w30"), golden_traffic("t600_s25")
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    pk = traffic
    if layout == "pinned":
        pk = _pinned(pk)
    elif layout == "records":
        pk = pfw.PacketArrays.pack_host(*[pk[f] for f in PKT_FIELDS])
    for nodes in (1, 2, 3, 8, 64, 512):
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=nodes)).run_arrays(c, pk)
        key = f"{model}_{nodes}"
        np.testing.assert_array_equal(res.first, g[f"{key}_first"])
        np.testing.assert_array_equal(res.comparisons, g[f"{key}_comps"])
        want_v = np.where(g[f"{key}_first"] >= 0, rules["action_accept"][np.maximum(g[f"{key}_first"], 0)], False)
        np.testing.assert_array_equal(res.verdict_accept, want_v)
        s = res.stats
        assert [s.total_comparisons, s.max_worker_comparisons, s.packets_processed] == g[f"{key}_stats"].tolist()


def test_partitioned_host_pipeline_many_chunks_vs_device():
    """Several chunks (ramped schedule), pageable in and out, compressed rows
    and a 7-node split: identical to the device-resident partition scans."""
    rules = oracle.gen_ruleset(30_000, 3, wp=0.2)
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    n = 3_000_001
    pk = oracle.gen_traffic_uniform(n, 78)
    first, comps, verdict, st = c.classify_host_partitions(pk, 7, chunk=1 << 18)
    p = pfw.PacketArrays.from_columns(*[pk[f] for f in PKT_FIELDS], device=0)
    df = torch.empty(n, dtype=torch.int32, device="cuda:0")
    dc = torch.empty(n, dtype=torch.int32, device="cuda:0")
    ds = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    c.scan_partitions(p, 7, df, dc, ds)
    want_f = first_to_host(df)
    np.testing.assert_array_equal(first, want_f)
    np.testing.assert_array_equal(comps, dc.cpu().numpy())
    np.testing.assert_array_equal(verdict, np.where(want_f >= 0, rules["action_accept"][np.maximum(want_f, 0)], False))
    assert st.tolist() == ds.cpu().numpy().tolist()
    idx = np.arange(0, n, 9973)
    sub = {f: v[idx] for f, v in pk.items()}
    f2, c2, _, _ = oracle.engine_run(rules, sub, "function", 7)
    np.testing.assert_array_equal(first[idx], f2)
    np.testing.assert_array_equal(comps[idx], c2)


def test_host_batch_staging_large_pageable():
    # several chunks, pageable in and out: staged through the pinned ring
    rules = oracle.gen_ruleset(1000, 1)
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    n = 3 << 20
    pk = oracle.gen_traffic_uniform(n, 77)
    want = oracle.scan_range(rules, pk, 0, 1000)
    f, v, st = c.classify_host(pk, chunk=1 << 18)
    np.testing.assert_array_equal(f, want)
    np.testing.assert_array_equal(v, np.where(want >= 0, rules["action_accept"][np.maximum(want, 0)], False))
    out_f = np.empty(n, np.int32)  # pageable outputs too
    out_v = np.empty(n, np.uint8)
    c.classify_host(pk, chunk=1 << 18, out=(out_f, out_v))
    np.testing.assert_array_equal(out_f, want)


def test_lazy_match_results_equal_reference_list():
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(170, seed=29, wildcard_probability=0.3))
    packets = pfw.generate_traffic(pfw.TrafficProfile(count=350, seed=30))
    for model in ("sequential", "data", "function", "hybrid"):
        results, _ = pfw.run(rs, packets, pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=3))
        assert isinstance(results, MatchResults)
        eager = [pfw.classify(rs, p) for p in packets[:20]]
        if model in ("sequential", "data"):
            assert results[:20] == eager  # MatchResult objects made on access
        assert len(results) == 350 and results[-1] == list(results)[-1]
        assert results == results.tolist()


@pytest.mark.parametrize("model", ["data", "function", "hybrid"])
def test_engine_on_several_devices_equals_golden(model):
    g = golden("engine_r503_t600.npz")
    c = pfw.CompiledRuleset.from_columns(golden_rules("r503_s24_w30"), device=0)
    cols = golden_traffic("t600_s25")
    p = pfw.PacketArrays.from_columns(*[cols[f] for f in PKT_FIELDS], device=0)
    for nodes in (1, 3, 8, 64):
        for devices, shard in (([0, 0], "rules"), ([0, 0, 0], "rules"), ([0, 0], "packets"), ([0, 0, 0], "auto")):
            eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=nodes, shard=shard),
                             devices=devices)
            for batch in (p, cols):
                res = eng.run_arrays(c, batch)
                key = f"{model}_{nodes}"
                np.testing.assert_array_equal(res.first, g[f"{key}_first"])
                np.testing.assert_array_equal(res.comparisons, g[f"{key}_comps"])
                s = res.stats
                assert [s.total_comparisons, s.max_worker_comparisons, s.packets_processed] == \
                    g[f"{key}_stats"].tolist()


def test_function_parallel_100k_rules_on_several_devices():
    g = golden("engine_r100000_t2000.npz")
    c = pfw.CompiledRuleset.from_columns(golden_rules("r100000_s1"), device=0)
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=2000, seed=2), device=0)
    for nodes, shard in ((2, "rules"), (8, "rules"), (8, "packets")):
        eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=nodes, shard=shard),
                         devices=[0, 0])
        res = eng.run_arrays(c, p)
        np.testing.assert_array_equal(res.first, g[f"function_{nodes}_first"])
        np.testing.assert_array_equal(res.comparisons, g[f"function_{nodes}_comps"])


def test_gpus_beyond_visible_devices_is_config_error():
    have = _native.device_count()
    with pytest.raises(pfw.ConfigError, match="CUDA devices are visible"):
        pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.DATA_PARALLEL, gpus=have + 1))


def test_partitioned_host_pipeline_pageable_outputs_c_abi():
    """pfw_classify_host_partitions called directly with ordinary numpy
    output arrays (first, comparisons, verdicts staged out through the pinned
    ring) and 16-byte records in: equal to the pinned-output call."""
    rules = oracle.gen_ruleset(5000, 11, wp=0.2)
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    n = 2_500_003
    pk = oracle.gen_traffic_uniform(n, 12)
    rec = pfw.PacketArrays.pack_host(*[pk[f] for f in PKT_FIELDS])
    want_f, want_c, want_v, want_st = c.classify_host_partitions(pk, 5, chunk=1 << 18)
    f = np.empty(n, np.int32)
    cm = np.empty(n, np.int32)
    v = np.empty(n, np.uint8)
    st = np.zeros(2, np.uint64)
    _native.check(_native.lib().pfw_classify_host_partitions(
        c.handle, 5, rec.ctypes.data, None, None, None, None, None, n, f.ctypes.data, cm.ctypes.data,
        v.ctypes.data, st.ctypes.data, 1 << 18, _native.HOST_FIRST_MINUS1), "pfw_classify_host_partitions")
    np.testing.assert_array_equal(f, want_f)
    np.testing.assert_array_equal(cm, want_c)
    np.testing.assert_array_equal(v.view(np.bool_), want_v)
    assert st.astype(np.int64).tolist() == want_st.tolist()
    with pytest.raises(ValueError):   # comparisons buffer required; nodes >= 1
        _native.check(_native.lib().pfw_classify_host_partitions(
            c.handle, 0, rec.ctypes.data, None, None, None, None, None, n, f.ctypes.data, cm.ctypes.data,
            None, None, 0, 0), "pfw_classify_host_partitions")


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 100, 65_535, 262_143, 262_145, 524_289])
def test_host_pipeline_tiny_and_odd_batches(n):
    """Host batches of every awkward size through the e2e pipeline (chunks
    smaller than the ramp, one-packet batches, just past a chunk boundary),
    both the whole-table and the partitioned models -- against the oracle."""
    rules = oracle.gen_ruleset(3000, 21, wp=0.3)
    c = pfw.CompiledRuleset.from_columns(rules, device=0)
    pk = oracle.gen_traffic_uniform(n, 22 + n)
    f, v, st = c.classify_host(pk)
    want = oracle.scan_range(rules, pk, 0, 3000)
    np.testing.assert_array_equal(f, want)
    np.testing.assert_array_equal(v, np.where(want >= 0, rules["action_accept"][np.maximum(want, 0)], False))
    comps = oracle.sequential_comparisons(want, 3000)
    assert st.tolist() == [int(comps.sum()), int(comps.max())]
    f2, c2, v2, st2 = c.classify_host_partitions(pk, 3)
    wf, wc, total, mx = oracle.engine_run(rules, pk, "function", 3)
    np.testing.assert_array_equal(f2, wf)
    np.testing.assert_array_equal(c2, wc)
    assert st2.tolist() == [total, mx]
    res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.DATA_PARALLEL)).run_arrays(c, pk)
    np.testing.assert_array_equal(res.first, want)


@pytest.mark.parametrize("model", ["data", "function", "hybrid"])
def test_host_pipeline_empty_ruleset_and_batch(model):
    """Empty ruleset (every packet default-denied after 0 comparisons) and
    empty batches through the host pipelines, every model."""
    empty = pfw.Ruleset()
    pk = oracle.gen_traffic_uniform(1000, 5)
    eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=4))
    res = eng.run_arrays(empty, pk)
    assert (np.asarray(res.first) == -1).all() and not np.asarray(res.verdict_accept).any()
    assert (np.asarray(res.comparisons) == 0).all()
    assert (res.stats.total_comparisons, res.stats.max_worker_comparisons) == (0, 0)
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(100, seed=3))
    res0 = eng.run_arrays(rs, {f: v[:0] for f, v in pk.items()})
    assert len(res0) == 0
