"""GPU parity: the CUDA path (through libpfw.so's C-ABI) against the oracle and
the reference's golden vectors.  Integer work: every comparison is bit-exact.

Mirrors the reference's own KATs (pkg/tests/test_classifier.py,
test_engines.py) and adds full-size properties that the oracle cannot
enumerate.
"""
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
from paper_1312_4188_b200.classifier import NO_MATCH, first_to_host  # noqa: E402
from oracle import oracle  # noqa: E402
from oracle.oracle import PKT_FIELDS  # noqa: E402


def dev_pkts(cols: dict) -> pfw.PacketArrays:
    return pfw.PacketArrays.from_columns(*[cols[f] for f in PKT_FIELDS], device=0)


def compiled(rules: dict) -> pfw.CompiledRuleset:
    return pfw.CompiledRuleset.from_columns(rules, device=0)


@pytest.fixture(autouse=True)
def _reset_tuning():
    yield
    for k, v in (("ks", 8), ("tile", 2048), ("ctas_per_sm", 0), ("force_imad", 1), ("first_pass", 1024),
                 ("proto_split", 0), ("short_circuit", 0), ("bucket", 1), ("bucket_min", 1 << 20),
                 ("algo", 0), ("ms_group", 0), ("ms_words", 4), ("matchset", 1), ("matchset_budget_mb", 0),
                 ("ms_summary", 2), ("count_blocks", 0), ("ms_compress", 2), ("ms_lean", 3), ("ms_lean_cmp", 3), ("ms_lean_sum", 2)):
        _native.set_tuning(k, v)


def mk_rule(action, proto, src="*", sport=None, dst="*", dport=None):
    import ipaddress

    def cidr(spec):
        if spec == "*":
            return pfw.CidrMatcher(0, 0)
        b, _, p = spec.partition("/")
        return pfw.CidrMatcher(int(ipaddress.IPv4Address(b)), int(p))
    ports = lambda s: pfw.PortRange(0, 65535) if s is None else pfw.PortRange(*s)  # noqa: E731
    return pfw.Rule(action, proto, cidr(src), ports(sport), cidr(dst), ports(dport))


def mk_packet(pid=0, proto=pfw.Protocol.TCP, sport=5555, dport=80):
    return pfw.Packet(pid, proto, 0x0A010203, sport, 0x08080808, dport)


# ----------------------------------------------------------------- reference KATs

def test_empty_ruleset_default_deny():
    r = pfw.classify(pfw.Ruleset(), mk_packet())
    assert (r.verdict, r.matched_index, r.comparisons) == (pfw.Action.DROP, None, 0)


def test_first_match_shadows_later_rules():
    rs = pfw.Ruleset((mk_rule(pfw.Action.DROP, pfw.Protocol.TCP),
                      mk_rule(pfw.Action.ACCEPT, pfw.Protocol.TCP, dport=(80, 80))))
    r = pfw.classify(rs, mk_packet(dport=80))
    assert (r.verdict, r.matched_index, r.comparisons) == (pfw.Action.DROP, 0, 1)


def test_no_match_scans_everything():
    rs = pfw.Ruleset((mk_rule(pfw.Action.ACCEPT, pfw.Protocol.UDP),) * 37)
    results, stats = pfw.classify_batch_sequential(rs, [mk_packet(i) for i in range(25)])
    assert all(r.comparisons == 37 and r.matched_index is None for r in results)
    assert stats.total_comparisons == 25 * 37


def test_batch_empty():
    results, stats = pfw.classify_batch_sequential(pfw.Ruleset(), [])
    assert results == [] and stats.total_comparisons == 0 and stats.max_worker_comparisons == 0


SCANS = [("oracle_r1000_t100000", "r1000_s1", "t100000_s2"),
         ("r2048_t1000", "r2048_s21_w15", "t1000_s22"),
         ("r300_t10000", "r300_s40_w30", "t10000_s41"),
         ("r64_t600", "r64_s30_w40", "t600_s25"),
         ("r1000_t5000ports", "r1000_s1", "t5000_s9_ports"),
         ("r1000_t3000icmp", "r1000_s1", "t3000_s11_icmp")]


@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_scan_matches_reference_golden(name, rn, tn):
    g = golden(f"scan_{name}.npz")
    rules, pk = golden_rules(rn), golden_traffic(tn)
    c = compiled(rules)
    R = c.num_rules
    p = dev_pkts(pk)
    n = len(p)
    comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
    verdict = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    first = c.scan_range_device(p, 0, R, comps=comps, verdict=verdict, stats=stats)
    np.testing.assert_array_equal(first_to_host(first), g["first"])
    np.testing.assert_array_equal(verdict.cpu().numpy().astype(bool), g["verdict"])
    want = oracle.sequential_comparisons(g["first"].astype(np.int64), R)
    np.testing.assert_array_equal(comps.cpu().numpy(), want)
    assert stats.cpu().tolist() == [int(g["total_comparisons"]), int(g["max_worker_comparisons"])]


def test_oracle_config_through_drop_in_api():
    g = golden("scan_oracle_r1000_t100000.npz")
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(1000, seed=1))
    packets = pfw.generate_traffic(pfw.TrafficProfile(count=100_000, seed=2))
    results, stats = pfw.classify_batch_sequential(rs, packets)
    assert stats.total_comparisons == 69_698_223
    got = np.array([-1 if r.matched_index is None else r.matched_index for r in results])
    np.testing.assert_array_equal(got, g["first"])
    assert [r.verdict is pfw.Action.ACCEPT for r in results] == g["verdict"].tolist()


def test_scan_windows():
    g = golden("scan_windows_r100_t150.npz")
    c = compiled(golden_rules("r100_s60_w35"))
    p = dev_pkts(golden_traffic("t150_s61"))
    for (lo, hi), want in zip(g["windows"].tolist(), g["first"]):
        np.testing.assert_array_equal(c.scan_range(p, lo, hi), want)


def test_windows_every_alignment_vs_oracle():
    rules = golden_rules("r300_s40_w30")
    pk = golden_traffic("t10000_s41")
    c, p = compiled(rules), dev_pkts(pk)
    for lo, hi in [(0, 300), (1, 300), (31, 33), (32, 64), (33, 290), (255, 257), (256, 300),
                   (299, 300), (5, 5), (7, 3), (0, 1)]:
        np.testing.assert_array_equal(c.scan_range(p, lo, hi), oracle.scan_range(rules, pk, lo, hi))


@pytest.mark.parametrize("rn", ["r4096_s1", "r10000_s1", "r100000_s1"])
def test_config_rulesets_sample(rn):
    g = golden(f"scan_{rn}_t20000.npz")
    c = compiled(golden_rules(rn))
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=20_000, seed=2), device=0)
    np.testing.assert_array_equal(c.scan_range(p, 0, c.num_rules), g["first"])


def test_adversarial_recipe_sample():
    g = golden("adversarial.npz")
    c = compiled(oracle.adversarial_rules(50_000))
    pk = oracle.adversarial_traffic(20_000)
    np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), 0, 50_000), g["first"])


# ------------------------------------------------------------------- engine models

@pytest.mark.parametrize("model", ["data", "function", "hybrid"])
def test_engine_models_match_reference_golden(model):
    g = golden("engine_r503_t600.npz")
    c = compiled(golden_rules("r503_s24_w30"))
    p = dev_pkts(golden_traffic("t600_s25"))
    for nodes in (1, 2, 3, 4, 8, 16, 64, 512):
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=nodes)).run_arrays(c, p)
        key = f"{model}_{nodes}"
        np.testing.assert_array_equal(res.first, g[f"{key}_first"])
        np.testing.assert_array_equal(res.comparisons, g[f"{key}_comps"])
        s = res.stats
        assert [s.total_comparisons, s.max_worker_comparisons, s.packets_processed] == g[f"{key}_stats"].tolist()


def test_function_parallel_100k_rules():
    g = golden("engine_r100000_t2000.npz")
    c = compiled(golden_rules("r100000_s1"))
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=2000, seed=2), device=0)
    for nodes in (1, 2, 4, 8):
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=nodes)).run_arrays(c, p)
        np.testing.assert_array_equal(res.first, g[f"function_{nodes}_first"])
        np.testing.assert_array_equal(res.comparisons, g[f"function_{nodes}_comps"])
        assert [res.stats.total_comparisons, res.stats.max_worker_comparisons, 2000] == \
            g[f"function_{nodes}_stats"].tolist()


def test_scan_partitions_oracle_small():
    """The one-launch partition walk against the oracle's per-node scan
    (oracle.engine_run: engines.py:349-369), stats included."""
    import torch
    from oracle import oracle as orc
    from paper_1312_4188_b200.classifier import first_to_host
    rules, traffic = golden_rules("r503_s24_w30"), golden_traffic("t600_s25")
    c = compiled(rules)
    p = dev_pkts(traffic)
    n = len(p)
    for nodes in (2, 7, 100, 503, 600):
        first = torch.empty(n, dtype=torch.int32, device="cuda:0")
        comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
        stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
        c.scan_partitions(p, nodes, first, comps, stats)
        want_first, want_comps, total, mx = orc.engine_run(rules, traffic, "function", nodes)
        np.testing.assert_array_equal(first_to_host(first), want_first)
        np.testing.assert_array_equal(comps.cpu().numpy(), want_comps)
        assert stats.cpu().numpy().tolist() == [total, mx]


def test_engine_drop_in_run_all_models():
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(170, seed=29, wildcard_probability=0.3))
    packets = pfw.generate_traffic(pfw.TrafficProfile(count=350, seed=30))
    outs = []
    for model in ("sequential", "data", "function", "hybrid"):
        results, _ = pfw.run(rs, packets, pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=3))
        outs.append([(r.verdict, r.matched_index) for r in results])
    assert all(o == outs[0] for o in outs)
    # empty batch / empty ruleset under every model (test_engines.py:249-263)
    for model in ("sequential", "data", "function", "hybrid"):
        cfg = pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=4)
        results, stats = pfw.run(rs, [], cfg)
        assert results == [] and stats.packets_processed == 0 and stats.total_comparisons == 0
        results, stats = pfw.run(pfw.Ruleset(), packets[:50], cfg)
        assert all(r.verdict is pfw.Action.DROP and r.matched_index is None for r in results)
        assert stats.total_comparisons == 0
    with pytest.raises(pfw.ConfigError, match="expected"):
        pfw.run_data_parallel(rs, packets, pfw.EngineConfig(pfw.ExecutionModel.HYBRID))


def test_function_parallel_speculative_scan_bounds():
    rs = pfw.Ruleset((mk_rule(pfw.Action.ACCEPT, pfw.Protocol.TCP),)
                     + tuple(mk_rule(pfw.Action.DROP, pfw.Protocol.UDP) for _ in range(2047)))
    parts = pfw.partition_rules(rs, 4)
    partials = [pfw.scan_partition(p, mk_packet()) for p in parts]
    assert partials[0].comparisons == 1 and all(p.comparisons == 512 for p in partials[1:])
    results, stats = pfw.run_function_parallel(rs, [mk_packet()], pfw.EngineConfig(
        pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=4))
    assert results[0].comparisons == 1 + 3 * 512 and stats.max_worker_comparisons == 512
    combined = pfw.aggregate(partials, len(rs))
    assert (combined.verdict, combined.matched_index) == (pfw.Action.ACCEPT, 0)


def test_combine_partition_matches():
    rows = np.array([[-1, 5, 7, -1], [3, -1, 2, -1], [4, 9, -1, 11]], dtype=np.int64)
    np.testing.assert_array_equal(pfw.combine_partition_matches(rows, 12), [3, 5, 2, 11])
    np.testing.assert_array_equal(pfw.combine_partition_matches(rows, 10), [3, 5, 2, -1])
    assert pfw.combine_partition_matches(np.zeros((0, 0), np.int64), 5).shape == (0,)


# --------------------------------------------------------------------- generator

@pytest.mark.parametrize("name", ["t100000_s2", "t2000_s7_dst0_1", "t2000_s8_dst192_2", "t5000_s9_ports",
                                  "t3000_s11_icmp", "t150_s61"])
def test_device_generator_matches_reference(name):
    g = golden(f"traffic_{name}.npz")
    prof = pfw.TrafficProfile(
        count=int(g["count"]), seed=int(g["seed"]), proto=pfw.Protocol(int(g["p_proto"])),
        src_subnet=pfw.CidrMatcher(int(g["p_src_base"]), int(g["p_src_plen"])),
        dst_subnet=pfw.CidrMatcher(int(g["p_dst_base"]), int(g["p_dst_plen"])),
        sport_range=pfw.PortRange(int(g["p_sport_lo"]), int(g["p_sport_hi"])),
        dport_range=pfw.PortRange(int(g["p_dport_lo"]), int(g["p_dport_hi"])))
    cols = pfw.generate_traffic_device(prof, device=0).columns()
    want = golden_traffic(name)
    for f in PKT_FIELDS:
        np.testing.assert_array_equal(cols[f], want[f])


def test_device_generator_large_jump_ahead():
    # 5M packets: the device stream must equal the sequential C oracle everywhere
    n = 5_000_123
    got = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=12345), device=0).columns()
    want = oracle.gen_traffic_uniform(n, 12345)
    for f in PKT_FIELDS:
        np.testing.assert_array_equal(got[f], want[f])


def test_worst_case_generation():
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(64, seed=3, wildcard_probability=0.3))
    prof = pfw.TrafficProfile(count=300, seed=4, match_mode=pfw.MatchMode.WORST_CASE)
    packets = pfw.generate_traffic(prof, rs)
    assert [p.id for p in packets] == list(range(300))
    results, _ = pfw.classify_batch_sequential(rs, packets)
    assert all(r.matched_index is None for r in results)


# ------------------------------------------------------------------ edge cases / tuning

def test_ragged_sizes_and_empty():
    rules = oracle.gen_ruleset(777, 5, wp=0.4)
    c = compiled(rules)
    for n in (0, 1, 31, 33, 255, 257, 2047, 2049, 4097):
        pk = oracle.gen_traffic_uniform(n, 100 + n)
        if n == 0:
            assert c.scan_range(pfw.PacketArrays.empty(0, 0), 0, 777).shape == (0,)
            continue
        np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), 0, 777), oracle.scan_range(rules, pk, 0, 777))


def test_unnormalised_and_inverted_rules_never_match():
    # raw C-ABI columns outside the Rule invariants follow the reference
    # predicate literally: (ip & mask) == base can never hold with host bits
    # in base, and lo <= p <= hi never holds for an inverted range.
    rules = {f: np.zeros(4, dtype=d) for f, d in zip(oracle.RULE_FIELDS, oracle.RULE_DTYPES)}
    rules["sport_hi"][:] = 65535
    rules["dport_hi"][:] = 65535
    rules["src_base"][0], rules["src_mask"][0] = 0x0A000001, 0xFF000000  # host bit set
    rules["sport_lo"][1], rules["sport_hi"][1] = 100, 50                 # inverted
    rules["proto"][2] = 99                                               # unusual concrete proto
    pk = oracle.gen_traffic_uniform(1000, 9, src_base=0x0A000000, src_plen=8)
    pk["proto"][:500] = 99
    want = oracle.scan_range(rules, pk, 0, 4)
    np.testing.assert_array_equal(compiled(rules).scan_range(dev_pkts(pk), 0, 4), want)
    assert (want[:500] == 2).all() and (want[500:] == 3).all()


@pytest.mark.parametrize("sc", [0, 1])
@pytest.mark.parametrize("ks,tile,imad,fp", [(2, 256, 1, 64), (4, 1024, 0, 0), (8, 4096, 1, 256),
                                             (8, 6144, 0, 1024), (4, 2048, 1, 100), (8, 2048, 1, 32),
                                             (6, 2048, 1, 1024)])
def test_tuning_variants_identical(ks, tile, imad, fp, sc):
    _native.set_tuning("algo", 1)
    _native.set_tuning("short_circuit", sc)
    _native.set_tuning("ks", ks)
    _native.set_tuning("tile", tile)
    _native.set_tuning("force_imad", imad)
    _native.set_tuning("first_pass", fp)
    rules = golden_rules("r2048_s21_w15")
    pk = golden_traffic("t10000_s41")
    c = compiled(rules)
    np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), 0, 2048), oracle.scan_range(rules, pk, 0, 2048))
    np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), 100, 1500), oracle.scan_range(rules, pk, 100, 1500))
    # multi-pass accumulate (function-parallel partitions) under the same tuning
    g = golden("engine_r503_t600.npz")
    c5 = compiled(golden_rules("r503_s24_w30"))
    p5 = dev_pkts(golden_traffic("t600_s25"))
    for nodes in (1, 3, 64):
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=nodes)).run_arrays(c5, p5)
        np.testing.assert_array_equal(res.first, g[f"function_{nodes}_first"])
        np.testing.assert_array_equal(res.comparisons, g[f"function_{nodes}_comps"])


def test_tile_too_large_is_rejected_loudly():
    _native.set_tuning("algo", 1)
    _native.set_tuning("tile", 8192)
    c = compiled(golden_rules("r64_s30_w40"))
    with pytest.raises(ValueError, match="shared memory"):
        c.scan_range(dev_pkts(golden_traffic("t600_s25")), 0, 64)


def test_classify_host_e2e_matches_device():
    rules = oracle.gen_ruleset(4096, 1)
    c = compiled(rules)
    n = 1_000_003
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    dev_first = c.scan_range_device(p, 0, 4096)
    host_pk = p.data.cpu().pin_memory()
    h_first = torch.empty(n, dtype=torch.int32).pin_memory()
    h_verd = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_stats = torch.zeros(2, dtype=torch.int64)
    _native.check(_native.lib().pfw_classify_host(c.handle, host_pk.data_ptr(), n, h_first.data_ptr(),
                                                  h_verd.data_ptr(), h_stats.data_ptr(), 300_000),
                  "pfw_classify_host")
    np.testing.assert_array_equal(h_first.numpy(), dev_first.cpu().numpy())
    f = first_to_host(dev_first)
    comps = oracle.sequential_comparisons(f, 4096)
    assert h_stats.tolist() == [int(comps.sum()), int(comps.max())]
    acc = np.where(f >= 0, rules["action_accept"][np.maximum(f, 0)], False)
    np.testing.assert_array_equal(h_verd.numpy().astype(bool), acc)


def test_full_size_properties_data_parallel():
    """10K rules x 16Mi packets: oracle on a strided subsample, plus
    size-independent properties on every packet (index range, verdict
    consistency, comparison checksum = sum of per-packet counts)."""
    R, n = 10_000, 1 << 24
    rules = oracle.gen_ruleset(R, 1)
    c = compiled(rules)
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
    verdict = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    first = c.scan_range_device(p, 0, R, comps=comps, verdict=verdict, stats=stats)
    f = first.cpu().numpy()
    hit = f != NO_MATCH
    assert ((f[hit] >= 0) & (f[hit] < R)).all()
    cm = comps.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(cm, np.where(hit, f.astype(np.int64) + 1, R))
    assert stats.cpu().tolist() == [int(cm.sum()), int(cm.max())]
    acc = np.zeros(n, np.uint8)
    acc[hit] = rules["action_accept"][f[hit]]
    np.testing.assert_array_equal(verdict.cpu().numpy(), acc)
    idx = np.arange(0, n, 797)
    sub = {k: v[idx] for k, v in p.columns().items()}
    want = oracle.scan_range(rules, sub, 0, R)
    got = np.where(hit[idx], f[idx].astype(np.int64), -1)
    np.testing.assert_array_equal(got, want)


# ------------------------------------------------------ fused function-parallel

@pytest.mark.parametrize("scatter", [0, 1])
def test_fused_min_combine_virtual_ranks(scatter):
    """G virtual ranks on one GPU: each scans its rule shard with the fused
    epilogue into the G result buffers (local memory stands in for the IPC
    peer mappings) -- equals the function-parallel model with nodes = G."""
    import ctypes
    g = golden("engine_r503_t600.npz")
    c = compiled(golden_rules("r503_s24_w30"))
    p = dev_pkts(golden_traffic("t600_s25"))
    n = len(p)
    for G in (1, 2, 3, 8):
        bounds = pfw.partition_bounds(n, G)
        if scatter:
            first = torch.full((n,), NO_MATCH, dtype=torch.int32, device="cuda:0")
            comps = torch.zeros(n, dtype=torch.int32, device="cuda:0")
            fptr = [first.data_ptr() + 4 * a for a, _ in bounds]
            cptr = [comps.data_ptr() + 4 * a for a, _ in bounds]
            caps = [b - a for a, b in bounds]
            bufs = [(first, comps)]
        else:
            bufs = [(torch.full((n,), NO_MATCH, dtype=torch.int32, device="cuda:0"),
                     torch.zeros(n, dtype=torch.int32, device="cuda:0")) for _ in range(G)]
            fptr = [b[0].data_ptr() for b in bufs]
            cptr = [b[1].data_ptr() for b in bufs]
            caps = [n] * G
        P = ctypes.c_void_p
        stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
        for lo, hi in pfw.partition_bounds(c.num_rules, G):
            _native.check(_native.lib().pfw_scan_fused_min(
                c.handle, lo, hi, p.data.data_ptr(), n, (P * G)(*fptr), (P * G)(*cptr), (ctypes.c_int64 * G)(*caps),
                G, scatter,
                stats.data_ptr(), torch.cuda.current_stream().cuda_stream), "fused")
        torch.cuda.synchronize()
        if G > 1:  # a batch larger than the buffers is refused before any launch
            with pytest.raises(ValueError, match="buffer holds"):
                _native.check(_native.lib().pfw_scan_fused_min(
                    c.handle, 0, c.num_rules, p.data.data_ptr(), n + G, (P * G)(*fptr), (P * G)(*cptr),
                    (ctypes.c_int64 * G)(*caps), G, scatter, None, torch.cuda.current_stream().cuda_stream),
                    "fused")
        for first, comps in bufs:
            np.testing.assert_array_equal(first_to_host(first), g[f"function_{G}_first"])
            np.testing.assert_array_equal(comps.cpu().numpy(), g[f"function_{G}_comps"])
        total, mx, _ = g[f"function_{G}_stats"].tolist()
        assert stats.cpu().tolist() == [total, mx]


def test_fused_function_parallel_single_rank_class():
    from paper_1312_4188_b200.parallel import FusedFunctionParallel
    g = golden("engine_r100000_t2000.npz")
    c = compiled(golden_rules("r100000_s1"))
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=2000, seed=2), device=0)
    fused = FusedFunctionParallel(c, len(p))
    for _ in range(3):  # alternate buffer sets: each call's set was reset by the previous call
        first, comps = fused.run(p)
        np.testing.assert_array_equal(first_to_host(first), g["function_1_first"])
        np.testing.assert_array_equal(comps.cpu().numpy(), g["function_1_comps"])
    with pytest.raises(ValueError, match="batches of"):
        fused.run(p.slice(0, 100))
    fused.close()


# ------------------------------------------------------ protocol-split chains

@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_proto_split_scan_matches_reference_golden(name, rn, tn):
    _native.set_tuning("algo", 1)
    _native.set_tuning("proto_split", 1)
    test_scan_matches_reference_golden(name, rn, tn)


def test_proto_split_windows_engines_and_mixed_protocols():
    _native.set_tuning("algo", 1)
    _native.set_tuning("proto_split", 1)
    test_scan_windows()
    test_windows_every_alignment_vs_oracle()
    for model in ("data", "function", "hybrid"):
        test_engine_models_match_reference_golden(model)
    test_function_parallel_100k_rules()
    test_unnormalised_and_inverted_rules_never_match()
    test_fused_min_combine_virtual_ranks(1)
    # mixed-protocol traffic (TCP / UDP / ICMP / an unnamed protocol) against
    # a ruleset with every protocol class
    rules = oracle.gen_ruleset(3000, 17, wp=0.3)
    rules["proto"][::97] = 47  # a protocol only a few rules name
    parts = [oracle.gen_traffic_uniform(5000, 20 + k, proto=pr) for k, pr in enumerate((6, 17, 1, 47, 99))]
    pk = {f: np.concatenate([pt[f] for pt in parts]) for f in PKT_FIELDS}
    perm = np.random.default_rng(0).permutation(len(pk["proto"]))
    pk = {f: v[perm] for f, v in pk.items()}
    c = compiled(rules)
    for lo, hi in ((0, 3000), (5, 2900), (1000, 1001)):
        np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))


@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_short_circuit_scan_matches_reference_golden(name, rn, tn):
    _native.set_tuning("algo", 1)
    _native.set_tuning("short_circuit", 1)
    test_scan_matches_reference_golden(name, rn, tn)


# --------------------------------------------------- reference column layout

def test_scan_range_columns_device_and_host():
    rules = golden_rules("r2048_s21_w15")
    pk = golden_traffic("t10000_s41")
    c = compiled(rules)
    dev = {f: torch.from_numpy(np.ascontiguousarray(pk[f]).view(
        {np.uint8: np.uint8, np.uint16: np.int16, np.uint32: np.int32}[pk[f].dtype.type])).to("cuda:0")
        for f in PKT_FIELDS}
    for algo, split in ((0, 0), (1, 0), (1, 1)):
        _native.set_tuning("algo", algo)
        _native.set_tuning("proto_split", split)
        for lo, hi in ((0, 2048), (100, 1500)):
            first = c.scan_range_columns_device(dev, lo, hi)
            np.testing.assert_array_equal(first_to_host(first), oracle.scan_range(rules, pk, lo, hi))
    f, v, st = c.classify_host_columns(pk, chunk=3001)
    want = oracle.scan_range(rules, pk, 0, 2048)
    np.testing.assert_array_equal(f, want)
    np.testing.assert_array_equal(v, np.where(want >= 0, rules["action_accept"][np.maximum(want, 0)], False))
    comps = oracle.sequential_comparisons(want, 2048)
    assert st.tolist() == [int(comps.sum()), int(comps.max())]


def test_e2e_mixed_protocol_rule_scan_large_chunks():
    """The e2e pipeline runs consecutive chunks on two compute streams; with
    the rule-by-rule scan each chunk >= bucket_min is grouped by protocol
    first.  Each stream has its own bucket scratch, so mixed-protocol chunks
    scanned concurrently never see each other's buckets (9Mi packets,
    protocols shuffled)."""
    _native.set_tuning("algo", 1)
    rules = oracle.gen_ruleset(1000, 1)
    n = 9 << 20
    parts = [oracle.gen_traffic_uniform(n // 3, 31 + k, proto=pr) for k, pr in enumerate((6, 17, 1))]
    perm = np.random.default_rng(5).permutation(n)
    pk = {f: np.concatenate([q[f] for q in parts])[perm] for f in PKT_FIELDS}
    c = compiled(rules)
    want = oracle.scan_range(rules, pk, 0, 1000)
    for split in (0, 1):
        _native.set_tuning("proto_split", split)
        f, v, st = c.classify_host_columns(pk)
        np.testing.assert_array_equal(f, want)
    comps = oracle.sequential_comparisons(want, 1000)
    assert st.tolist() == [int(comps.sum()), int(comps.max())]


# --------------------------------------------- protocol-uniform tile fast path

@pytest.mark.parametrize("proto", [1, 6, 17, 47, 0, 255])
def test_protocol_uniform_tiles(proto):
    """Every packet of a tile has the same protocol -> ANY rules are rewritten
    into the protocol-major form for it at stage load (no rule skipped)."""
    _native.set_tuning("algo", 1)
    rules = oracle.gen_ruleset(1500, 23, wp=0.35)
    rules["proto"][::13] = 47
    rules["proto"][::29] = 255
    pk = oracle.gen_traffic_uniform(6000, 24, proto=max(proto, 1))
    pk["proto"][:] = proto
    c = compiled(rules)
    for lo, hi in ((0, 1500), (77, 1400)):
        np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))


def test_mixed_and_uniform_tiles_in_one_batch():
    _native.set_tuning("algo", 1)
    _native.set_tuning("tile", 256)
    rules = oracle.gen_ruleset(900, 25, wp=0.35)
    pk = oracle.gen_traffic_uniform(256 * 12, 26)
    pk["proto"][256 * 3:256 * 4] = 17          # a whole UDP tile
    pk["proto"][256 * 6 + 5] = 1               # one ICMP packet in a TCP tile
    pk["proto"][256 * 9:256 * 10:2] = 17       # an interleaved tile
    np.testing.assert_array_equal(compiled(rules).scan_range(dev_pkts(pk), 0, 900),
                                  oracle.scan_range(rules, pk, 0, 900))


@pytest.mark.parametrize("bucket_min", [0, 1 << 20])
def test_protocol_bucketing_mixed_traffic(bucket_min):
    """Mixed-protocol batches are grouped by protocol on the device so tiles are
    protocol-uniform; results identical, with or without the grouping."""
    _native.set_tuning("algo", 1)
    _native.set_tuning("bucket_min", bucket_min)
    rules = oracle.gen_ruleset(2500, 31, wp=0.3)
    rules["proto"][::17] = 47
    n = 1_200_000 if bucket_min else 40_000
    parts = [oracle.gen_traffic_uniform(n // 5, 40 + k, proto=pr) for k, pr in enumerate((6, 17, 1, 47, 99))]
    pk = {f: np.concatenate([pt[f] for pt in parts]) for f in PKT_FIELDS}
    perm = np.random.default_rng(1).permutation(len(pk["proto"]))
    pk = {f: v[perm] for f, v in pk.items()}
    c = compiled(rules)
    p = dev_pkts(pk)
    want = oracle.scan_range(rules, pk, 0, 2500)
    np.testing.assert_array_equal(c.scan_range(p, 0, 2500), want)
    _native.set_tuning("bucket", 0)
    np.testing.assert_array_equal(c.scan_range(p, 0, 2500), want)
    _native.set_tuning("bucket", 1)
    # function-parallel accumulate through the bucketed path
    res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=3)).run_arrays(c, p)
    first, comps, total, mx = oracle.engine_run(rules, pk, "function", 3)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.comparisons, comps)


@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_bucketed_scan_matches_reference_golden(name, rn, tn):
    _native.set_tuning("algo", 1)
    _native.set_tuning("bucket_min", 0)
    test_scan_matches_reference_golden(name, rn, tn)


# ------------------------------------------------- rule-by-rule vs match sets

@pytest.mark.parametrize("name,rn,tn", SCANS)
def test_rule_scan_matches_reference_golden(name, rn, tn):
    """The same goldens through the rule-by-rule scan (the default path is the
    match-set scan whenever the ruleset's match sets were built)."""
    _native.set_tuning("algo", 1)
    test_scan_matches_reference_golden(name, rn, tn)


def test_rule_scan_windows_engines_and_samples():
    _native.set_tuning("algo", 1)
    test_scan_windows()
    test_windows_every_alignment_vs_oracle()
    for model in ("data", "function", "hybrid"):
        test_engine_models_match_reference_golden(model)
    test_function_parallel_100k_rules()
    test_adversarial_recipe_sample()
    test_ragged_sizes_and_empty()
    test_unnormalised_and_inverted_rules_never_match()
    test_fused_min_combine_virtual_ranks(1)
    test_fused_min_combine_virtual_ranks(0)


def test_match_sets_built_for_every_config_ruleset():
    for rn in ("r1000_s1", "r4096_s1", "r10000_s1", "r100000_s1"):
        c = compiled(golden_rules(rn))
        assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) > 0


MS_SHAPES = [(8, 4), (8, 2), (16, 4), (16, 2), (32, 2), (32, 1)]


@pytest.mark.parametrize("group,words", MS_SHAPES)
def test_match_set_step_shapes(group, words):
    """Lanes per packet x words per lane (rules per step = 32 x group x words)."""
    _native.set_tuning("algo", 2)
    _native.set_tuning("ms_group", group)
    _native.set_tuning("ms_words", words)
    test_scan_matches_reference_golden("r2048_t1000", "r2048_s21_w15", "t1000_s22")
    test_scan_matches_reference_golden("r1000_t3000icmp", "r1000_s1", "t3000_s11_icmp")
    test_windows_every_alignment_vs_oracle()
    test_engine_models_match_reference_golden("hybrid")
    test_engine_models_match_reference_golden("function")
    test_ragged_sizes_and_empty()
    test_adversarial_recipe_sample()
    test_fused_min_combine_virtual_ranks(0)


@pytest.mark.parametrize("lean", [0, 1, 2, 4, 5, 6])
def test_lean_whole_table_scan(lean):
    """Whole-table scans over plain rows: the general kernel (0) and every
    lean variant (1: 8-lane groups; 2: 4-lane groups with 256-bit loads; 4:
    512-rule steps; 5: 6 blocks per SM; 6: 64-packet batches) are bit-exact
    against the reference goldens, ragged batches and the full-size data
    config's strided oracle sample."""
    _native.set_tuning("algo", 2)
    _native.set_tuning("ms_compress", 0)
    _native.set_tuning("ms_lean", lean)
    for name, rn, tn in (("oracle_r1000_t100000", "r1000_s1", "t100000_s2"), ("r2048_t1000", "r2048_s21_w15", "t1000_s22"),
                         ("r300_t10000", "r300_s40_w30", "t10000_s41"), ("r64_t600", "r64_s30_w40", "t600_s25"),
                         ("r1000_t3000icmp", "r1000_s1", "t3000_s11_icmp")):
        test_scan_matches_reference_golden(name, rn, tn)
    test_ragged_sizes_and_empty()
    test_engine_models_match_reference_golden("data")
    rules = golden_rules("r10000_s1")
    c = compiled(rules)
    n = 1 << 22
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
    verdict = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    first = first_to_host(c.scan_range_device(p, 0, 10_000, comps=comps, verdict=verdict, stats=stats))
    idx = np.arange(0, n, 97)
    sub = {f: v[idx] for f, v in p.columns().items()}
    want = oracle.scan_range(rules, sub, 0, 10_000)
    np.testing.assert_array_equal(first[idx], want)
    cc = comps.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(cc, np.where(first >= 0, first + 1, 10_000))
    assert stats.cpu().tolist() == [int(cc.sum()), int(cc.max())]


@pytest.mark.parametrize("lc", [0, 1, 2, 3])
def test_lean_compressed_rows(lc):
    """Whole-table scans over compressed rows: the general kernel (0) and the
    lean compressed kernel with 8- or 4-lane groups (1, 2) are bit-exact, incl.
    scans that run past the parked blocks (late matches, default deny)."""
    _native.set_tuning("algo", 2)
    _native.set_tuning("ms_compress", 1)
    _native.set_tuning("ms_summary", 0)
    _native.set_tuning("ms_lean_cmp", lc)
    for name, rn, tn in SCANS:
        test_scan_matches_reference_golden(name, rn, tn)
    test_ragged_sizes_and_empty()
    test_adversarial_recipe_sample()        # most packets scan far past the parked blocks
    test_function_parallel_100k_rules()     # nodes = 1 is a whole-table scan
    test_engine_models_match_reference_golden("data")
    rules = golden_rules("r100000_s1")
    c = compiled(rules)
    n = 1 << 20
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    first = first_to_host(c.scan_range_device(p, 0, 100_000))
    idx = np.arange(0, n, 211)
    sub = {f: v[idx] for f, v in p.columns().items()}
    np.testing.assert_array_equal(first[idx], oracle.scan_range(rules, sub, 0, 100_000))


def test_match_set_budget_falls_back_to_rule_scan():
    _native.set_tuning("matchset_budget_mb", 1)        # 10K rules need ~117 MB
    c = compiled(golden_rules("r10000_s1"))
    assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) == 0
    g = golden("scan_r10000_s1_t20000.npz")
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=20_000, seed=2), device=0)
    np.testing.assert_array_equal(c.scan_range(p, 0, c.num_rules), g["first"])   # rule-by-rule scan
    _native.set_tuning("algo", 2)
    with pytest.raises(ValueError, match="no match sets"):
        c.scan_range(p, 0, c.num_rules)
    _native.set_tuning("matchset_budget_mb", 0)
    _native.set_tuning("matchset", 0)
    assert _native.lib().pfw_ruleset_matchset_bytes(compiled(golden_rules("r64_s30_w40")).handle) == 0


def test_match_set_interval_edges():
    """Interval boundaries at the ends of the value domains: /0, /32, host
    255.255.255.255, port 0 / 65535, single-port ranges, adjacent blocks,
    protocols no rule names, packet protocol 0."""
    rng = np.random.default_rng(77)
    R = 700
    rules = oracle.gen_ruleset(R, 78, wp=0.25)
    edge_ips = np.array([0, 1, 0xFFFFFFFF, 0xFFFFFFFE, 0x80000000, 0x7FFFFFFF, 0x0A000000, 0x0A0000FF,
                         0x0A000100, 0xC0A80001], dtype=np.uint32)
    for k in range(0, R, 7):
        plen = int(rng.choice([0, 1, 8, 16, 24, 31, 32]))
        mask = np.uint32(0) if plen == 0 else np.uint32((0xFFFFFFFF << (32 - plen)) & 0xFFFFFFFF)
        ip = np.uint32(rng.choice(edge_ips))
        f = "src" if k % 2 else "dst"
        rules[f + "_base"][k] = ip & mask
        rules[f + "_mask"][k] = mask
        lo = int(rng.choice([0, 1, 80, 1023, 65534, 65535]))
        hi = int(rng.choice([lo, min(lo + 1, 65535), 65535]))
        rules["sport_lo" if k % 3 else "dport_lo"][k] = lo
        rules["sport_hi" if k % 3 else "dport_hi"][k] = hi
    rules["proto"][::31] = 47
    n = 20_000
    pk = oracle.gen_traffic_uniform(n, 79)
    pk["src_ip"][:4000] = rng.choice(edge_ips, 4000)
    pk["dst_ip"][2000:6000] = rng.choice(edge_ips, 4000)
    pk["src_port"][::3] = rng.choice(np.array([0, 1, 80, 1023, 1024, 65534, 65535], np.uint16), len(pk["src_port"][::3]))
    pk["dst_port"][::5] = rng.choice(np.array([0, 1, 80, 1023, 1024, 65534, 65535], np.uint16), len(pk["dst_port"][::5]))
    pk["proto"][::11] = 17
    pk["proto"][::13] = 1
    pk["proto"][::17] = 47
    pk["proto"][::19] = 0
    pk["proto"][::23] = 200
    c = compiled(rules)
    assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) > 0
    _native.set_tuning("algo", 2)
    for group, words in MS_SHAPES:
        _native.set_tuning("ms_group", group)
        _native.set_tuning("ms_words", words)
        for lo, hi in ((0, R), (1, R - 1), (31, 32), (32, 1024 % R), (300, 301), (64, 700)):
            np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))


@pytest.mark.parametrize("summary", [0, 1])
def test_match_set_block_summaries(summary):
    """Block summaries (skip 1024-rule blocks whose AND-summary is zero) forced
    off / on: goldens, windows, engines, the adversarial recipe (where the auto
    mode turns them on) -- identical results."""
    _native.set_tuning("ms_summary", summary)   # applies to rulesets built from here on
    _native.set_tuning("algo", 2)
    test_adversarial_recipe_sample()
    test_scan_matches_reference_golden("r2048_t1000", "r2048_s21_w15", "t1000_s22")
    test_scan_matches_reference_golden("oracle_r1000_t100000", "r1000_s1", "t100000_s2")
    test_windows_every_alignment_vs_oracle()
    for model in ("function", "hybrid"):
        test_engine_models_match_reference_golden(model)
    test_function_parallel_100k_rules()
    test_fused_min_combine_virtual_ranks(1)
    # windows over the adversarial ruleset: blocks skipped inside partial windows
    rules = oracle.adversarial_rules(50_000)
    pk = oracle.adversarial_traffic(6_000)
    c = compiled(rules)
    for lo, hi in ((0, 50_000), (1, 49_999), (1000, 45_001), (44_999, 45_003), (45_001, 50_000), (30_000, 30_001)):
        np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))
    # the block-read counter (bench roofline): only the summary variant counts
    _native.read_counter("blocks_read")
    _native.set_tuning("count_blocks", 1)
    try:
        c.scan_range(dev_pkts(pk), 0, 50_000)
        got = _native.read_counter("blocks_read")
    finally:
        _native.set_tuning("count_blocks", 0)
    assert _native.ruleset_info(c.handle, "summaries") == summary
    if summary:
        assert len(pk["proto"]) <= got < len(pk["proto"]) * 49 // 4   # most decoy blocks skipped
    else:
        assert got == 0


# ------------------------------------------------------------- rule shards

@pytest.mark.parametrize("algo", [0, 1])
def test_rule_shards_function_parallel(algo):
    """Function-parallel with per-rank rule shards (each uploads only its
    partition, engines.py:316-321): local windows, global indices; the
    accumulate and the fused combine over G shard handles equal the
    reference's function-parallel golden results."""
    import ctypes
    _native.set_tuning("algo", algo)
    g = golden("engine_r503_t600.npz")
    full = compiled(golden_rules("r503_s24_w30"))
    p = dev_pkts(golden_traffic("t600_s25"))
    n = len(p)
    for G in (1, 2, 3, 8):
        shards = [full.shard(lo, hi) for lo, hi in pfw.partition_bounds(full.num_rules, G)]
        assert all(s.is_shard for s in shards) == (G > 1)
        first = torch.full((n,), NO_MATCH, dtype=torch.int32, device="cuda:0")
        comps = torch.zeros(n, dtype=torch.int32, device="cuda:0")
        stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
        for s in shards:
            s.scan_partition_accumulate(p, 0, s.num_rules, first, comps, stats)
        np.testing.assert_array_equal(first_to_host(first), g[f"function_{G}_first"])
        np.testing.assert_array_equal(comps.cpu().numpy(), g[f"function_{G}_comps"])
        total, mx, _ = g[f"function_{G}_stats"].tolist()
        assert stats.cpu().tolist() == [total, mx]
        # fused combine from shard handles (virtual ranks, scatter layout)
        ff = torch.full((n,), NO_MATCH, dtype=torch.int32, device="cuda:0")
        fc = torch.zeros(n, dtype=torch.int32, device="cuda:0")
        bounds = pfw.partition_bounds(n, G)
        P = ctypes.c_void_p
        fptr = (P * G)(*[ff.data_ptr() + 4 * a for a, _ in bounds])
        cptr = (P * G)(*[fc.data_ptr() + 4 * a for a, _ in bounds])
        for s in shards:
            _native.check(_native.lib().pfw_scan_fused_min(
                s.handle, 0, s.num_rules, p.data.data_ptr(), n, fptr, cptr,
                (ctypes.c_int64 * G)(*[b - a for a, b in bounds]), G, 1, None,
                torch.cuda.current_stream().cuda_stream), "fused")
        torch.cuda.synchronize()
        np.testing.assert_array_equal(first_to_host(ff), g[f"function_{G}_first"])
        np.testing.assert_array_equal(fc.cpu().numpy(), g[f"function_{G}_comps"])


def test_rule_shard_windows_and_verdicts():
    rules = golden_rules("r2048_s21_w15")
    pk = golden_traffic("t10000_s41")
    full = compiled(rules)
    s = full.shard(300, 1700)
    assert (s.index_base, s.num_rules, s.total_rules) == (300, 1400, 2048)
    d = dev_pkts(pk)
    for lo, hi in ((0, 1400), (17, 1399), (700, 701)):
        np.testing.assert_array_equal(s.scan_range(d, lo, hi), oracle.scan_range(rules, pk, 300 + lo, 300 + hi))
    # verdicts written by the scan use the shard's own actions
    verdict = torch.empty(len(d), dtype=torch.uint8, device="cuda:0")
    f = first_to_host(s.scan_range_device(d, 0, 1400, verdict=verdict))
    want = np.where(f >= 0, rules["action_accept"][np.maximum(f, 0)], False)
    np.testing.assert_array_equal(verdict.cpu().numpy().astype(bool), want)
    # verdicts of combined indices need the whole ruleset's actions
    with pytest.raises(ValueError, match="whole ruleset"):
        s.verdicts_device(torch.zeros(4, dtype=torch.int32, device="cuda:0"))
    with pytest.raises(ValueError):
        full.shard(5, 3000)
    with pytest.raises(ValueError, match="outside"):
        _native.check(_native.lib().pfw_ruleset_set_shard(s.handle, 1000, 2048), "set_shard")


@pytest.mark.parametrize("R", [1, 2, 31, 32, 33, 127, 128, 129, 1023, 1024, 1025, 2047, 4095, 4096, 4097, 5000])
def test_rule_counts_at_word_line_and_step_edges(R):
    """Ruleset sizes at the edges of a 32-rule word, a 1024-rule line and a
    4096-rule step (match-set row padding) and of the rule scan's stages."""
    rules = oracle.gen_ruleset(R, 900 + R, wp=0.3)
    pk = oracle.gen_traffic_uniform(3000, 901)
    c = compiled(rules)
    for algo in (2, 1):
        _native.set_tuning("algo", algo)
        for lo, hi in ((0, R), (R // 2, R), (max(R - 1, 0), R)):
            np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))


# ------------------------------------------------- compressed match-set rows

def test_compressed_rows_forced():
    """Compressed rows (per block the distinct lines + u16 line indices per
    row) forced on: goldens, windows, engines, shards, the adversarial recipe
    (with summaries), every requested shape -- identical results."""
    _native.set_tuning("ms_compress", 1)   # applies to rulesets built from here on
    _native.set_tuning("algo", 2)
    for name, rn, tn in SCANS:
        test_scan_matches_reference_golden(name, rn, tn)
    test_scan_windows()
    test_windows_every_alignment_vs_oracle()
    for model in ("data", "function", "hybrid"):
        test_engine_models_match_reference_golden(model)
    test_function_parallel_100k_rules()
    test_adversarial_recipe_sample()
    test_ragged_sizes_and_empty()
    test_unnormalised_and_inverted_rules_never_match()
    test_fused_min_combine_virtual_ranks(1)
    test_rule_shard_windows_and_verdicts()
    test_rule_shards_function_parallel(2)  # (its algo argument 2 = match sets)
    test_match_set_interval_edges()       # (iterates the shapes: compressed rows ignore them)
    for rn in ("r10000_s1", "r100000_s1"):
        c = compiled(golden_rules(rn))
        g = golden(f"scan_{rn}_t20000.npz")
        p = pfw.generate_traffic_device(pfw.TrafficProfile(count=20_000, seed=2), device=0)
        np.testing.assert_array_equal(c.scan_range(p, 0, c.num_rules), g["first"])
        # a window past the 16 parked blocks (line indices from global memory)
        lo = 20 * 1024 + 7
        rules = golden_rules(rn)
        sub = {k: v for k, v in p.columns().items()}
        if c.num_rules > lo + 100:
            np.testing.assert_array_equal(c.scan_range(p, lo, c.num_rules),
                                          oracle.scan_range(rules, sub, lo, c.num_rules))


def test_compressed_rows_when_plain_exceeds_budget():
    """Auto: plain rows over the memory budget -> compressed rows (not the rule
    scan), also where auto would keep plain rows by size; the reported size is
    the compressed one."""
    _native.set_tuning("ms_compress", 0)
    big = compiled(golden_rules("r10000_s1"))              # plain rows: ~162 MB
    plain = _native.lib().pfw_ruleset_matchset_bytes(big.handle)
    _native.set_tuning("ms_compress", 2)
    _native.set_tuning("matchset_budget_mb", 64)           # too small for the plain rows
    c = compiled(golden_rules("r10000_s1"))
    got = _native.lib().pfw_ruleset_matchset_bytes(c.handle)
    assert 0 < got < plain // 4                            # (10K rules: ~7x; 100K: ~24x)
    assert _native.ruleset_info(c.handle, "compressed") == 1 and _native.ruleset_info(big.handle, "compressed") == 0
    assert _native.ruleset_info(c.handle, "matchset_bytes") == got
    g = golden("scan_r10000_s1_t20000.npz")
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=20_000, seed=2), device=0)
    _native.set_tuning("algo", 2)
    np.testing.assert_array_equal(c.scan_range(p, 0, c.num_rules), g["first"])
    _native.set_tuning("ms_compress", 0)                 # compression off: over budget -> rule scan
    c2 = compiled(golden_rules("r10000_s1"))
    assert _native.lib().pfw_ruleset_matchset_bytes(c2.handle) == 0
    # auto by size: 100K rules build compressed rows
    _native.set_tuning("ms_compress", 2)
    _native.set_tuning("matchset_budget_mb", 0)
    assert _native.ruleset_info(compiled(golden_rules("r100000_s1")).handle, "compressed") == 1


def test_summary_candidates_past_the_parked_ones():
    """Summary scan over compressed rows with more candidate blocks than the
    lookup phase parks (random rules: nearly every block is a candidate), so
    late-matching and default-deny packets continue with the in-loop summary
    search; whole and partial windows, counters."""
    _native.set_tuning("ms_summary", 1)
    _native.set_tuning("ms_compress", 1)
    rules = oracle.gen_ruleset(12_000, 91, wp=0.05)          # few wildcards: late / no matches
    pk = oracle.gen_traffic_uniform(8000, 92)
    c = compiled(rules)
    assert _native.ruleset_info(c.handle, "summaries") == 1 and _native.ruleset_info(c.handle, "compressed") == 1
    _native.set_tuning("algo", 2)
    for lo, hi in ((0, 12_000), (1, 11_999), (700, 9000), (6 * 1024 - 3, 12_000), (11_000, 11_001)):
        np.testing.assert_array_equal(c.scan_range(dev_pkts(pk), lo, hi), oracle.scan_range(rules, pk, lo, hi))
    want = oracle.scan_range(rules, pk, 0, 12_000)
    assert (want < 0).any() and (want > 7 * 1024).any()       # the fallback path is exercised
    res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=3)).run_arrays(c, dev_pkts(pk))
    first, comps, total, mx = oracle.engine_run(rules, pk, "function", 3)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.comparisons, comps)


@pytest.mark.parametrize("n", [917_504, 2_000_001, 3_145_731])
def test_classify_host_ramped_chunk_schedule(n):
    """pfw_classify_host_columns with a chunk small enough that the ramped
    schedule (1/4, 1/2 chunks at both ends, full chunks between) engages:
    identical to the device-resident scan, verdicts and stats included."""
    rules = oracle.gen_ruleset(4096, 1)
    c = compiled(rules)
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=5), device=0)
    dev_first = first_to_host(c.scan_range_device(p, 0, 4096))
    f, v, st = c.classify_host_columns(p.columns(), chunk=1 << 18)
    np.testing.assert_array_equal(f, dev_first)
    np.testing.assert_array_equal(v, np.where(dev_first >= 0, rules["action_accept"][np.maximum(dev_first, 0)], False))
    comps = oracle.sequential_comparisons(dev_first, 4096)
    assert st.tolist() == [int(comps.sum()), int(comps.max())]


@pytest.mark.parametrize("lean_sum", [0, 1, 2])
def test_summary_scan_kernels(lean_sum):
    """Whole-table summary scans over compressed rows on the general kernel (0)
    and the lean candidate walk (1: 5 blocks per SM, 2: 4): the adversarial
    recipe, scans whose candidates outnumber the parked ones (the lane-serial
    continuation after the loop), forced summaries on goldens -- identical."""
    _native.set_tuning("ms_lean_sum", lean_sum)
    test_adversarial_recipe_sample()
    test_summary_candidates_past_the_parked_ones()
    test_compressed_rows_forced()
    test_match_set_block_summaries(1)


def test_many_ip_boundaries_in_one_slash16():
    """More than 255 IP interval boundaries inside one /16 block: the packed
    lookup entry's count saturates and the search runs up to the next block's
    first boundary -- identical to the oracle (src and dst, /32 .. /24 rules)."""
    rng = np.random.default_rng(11)
    R = 1500
    rules = oracle.gen_ruleset(R, 77, wp=0.2)
    plen = rng.integers(24, 33, R)
    mask = np.where(plen == 32, 0xFFFFFFFF, (0xFFFFFFFF << (32 - plen)) & 0xFFFFFFFF).astype(np.uint32)
    base = (np.uint32(0x0A0B0000) | rng.integers(0, 1 << 16, R).astype(np.uint32)) & mask
    rules["src_base"], rules["src_mask"] = base, mask
    rules["dst_base"], rules["dst_mask"] = base[::-1].copy(), mask[::-1].copy()
    pk = oracle.gen_traffic_uniform(50_000, 5)
    pk["src_ip"][:40_000] = 0x0A0B0000 | rng.integers(0, 1 << 16, 40_000).astype(np.uint32)
    pk["dst_ip"][10_000:] = 0x0A0B0000 | rng.integers(0, 1 << 16, 40_000).astype(np.uint32)
    c, p = compiled(rules), dev_pkts(pk)
    assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) > 0
    np.testing.assert_array_equal(c.scan_range(p, 0, R), oracle.scan_range(rules, pk, 0, R))


def test_ip_lookup_entries_sparse_blocks_edges():
    """The 16-byte /16 lookup entries: blocks holding 1..8 and 12 boundaries
    (the first six carried in the entry, more searched), boundaries at low
    half 0x0000 and 0xFFFF (host rules ending a block), adjacent hosts; every
    boundary address and its neighbours probed, src and dst -- identical to
    the oracle."""
    rng = np.random.default_rng(5)
    hosts = []
    for blk, k in ((0x0A01, 1), (0x0A02, 2), (0x0A03, 3), (0x0A04, 5), (0x0A05, 6), (0x0A06, 7),
                   (0x0A07, 8), (0x0A08, 12), (0xFFFF, 6), (0x0000, 6)):
        lows = set(rng.choice(np.arange(1, 0xFFFE), k - 1, replace=False).tolist()) | {0xFFFF}
        if blk in (0x0A05, 0x0000):
            lows |= {0x0000}
        hosts += [(blk << 16) | lo for lo in sorted(lows)[:k]]
    hosts = np.array(hosts, dtype=np.uint32)
    R = 2 * len(hosts) + 40
    rules = oracle.gen_ruleset(R, 91, wp=0.3)
    # /32 hosts (boundaries at a and a + 1) on src for the first half, dst for the second
    # half, /31 pairs among them; then random rules
    for j, a in enumerate(hosts):
        for f, k in (("src", j), ("dst", len(hosts) + j)):
            plen = 31 if j % 5 == 0 else 32
            mask = np.uint32((0xFFFFFFFF << (32 - plen)) & 0xFFFFFFFF)
            rules[f + "_base"][k] = a & mask
            rules[f + "_mask"][k] = mask
            other = "dst" if f == "src" else "src"
            rules[other + "_base"][k] = 0
            rules[other + "_mask"][k] = 0
    probe = np.unique(np.concatenate([hosts, hosts + np.uint32(1), hosts - np.uint32(1),
                                      (hosts & np.uint32(0xFFFF0000)), hosts | np.uint32(0xFFFF)]))
    n = 40_000
    pk = oracle.gen_traffic_uniform(n, 92)
    pk["src_ip"][: n // 2] = rng.choice(probe, n // 2)
    pk["dst_ip"][n // 4:] = rng.choice(probe, n - n // 4)
    c, p = compiled(rules), dev_pkts(pk)
    assert _native.lib().pfw_ruleset_matchset_bytes(c.handle) > 0
    np.testing.assert_array_equal(c.scan_range(p, 0, R), oracle.scan_range(rules, pk, 0, R))
    np.testing.assert_array_equal(c.scan_range(p, 0, len(hosts)), oracle.scan_range(rules, pk, 0, len(hosts)))


@pytest.mark.parametrize("lc", [1, 2, 3])
@pytest.mark.parametrize("R", [6 * 1024 + 1, 12 * 1024, 13 * 1024 - 7, 20_000])
def test_lean_compressed_repark_windows(lc, R):
    """Sparse rulesets over compressed rows: most packets walk past their 6
    parked blocks (the group re-parks the next 6, the last window cut short
    by the table end) or scan everything (default deny) -- bit-exact."""
    _native.set_tuning("algo", 2)
    _native.set_tuning("ms_compress", 1)
    _native.set_tuning("ms_summary", 0)
    _native.set_tuning("ms_lean_cmp", lc)
    rules = oracle.gen_ruleset(R, 300 + R % 97, wp=0.02)
    pk = oracle.gen_traffic_uniform(30_000, 301)
    c, p = compiled(rules), dev_pkts(pk)
    want = oracle.scan_range(rules, pk, 0, R)
    assert (want < 0).mean() > 0.05  # default deny walks every block
    np.testing.assert_array_equal(c.scan_range(p, 0, R), want)


def test_c_abi_argument_errors_new_entry_points():
    """pfw_scan_partitions / pfw_probe_l2_lines reject bad arguments with
    PFW_ERR_INVALID (ValueError) before any launch; a valid probe call runs."""
    c = compiled(oracle.gen_ruleset(100, 3))
    p = dev_pkts(oracle.gen_traffic_uniform(50, 4))
    f = torch.empty(50, dtype=torch.int32, device="cuda:0")
    cm = torch.empty(50, dtype=torch.int32, device="cuda:0")
    with pytest.raises(ValueError):
        c.scan_partitions(p, 0, f, cm)
    lib = _native.lib()
    st = torch.cuda.current_stream().cuda_stream
    with pytest.raises(ValueError):
        _native.check(lib.pfw_scan_partitions(c.handle, 2, p.data.data_ptr(), 50, None, cm.data_ptr(), None, st),
                      "pfw_scan_partitions")
    buf = torch.empty(2 << 20, dtype=torch.uint8, device="cuda:0")
    for k, occ, iters, ok in ((8, 4, 4, True), (3, 4, 4, False), (8, 0, 4, False), (8, 4, 0, False)):
        rc = lib.pfw_probe_l2_lines(buf.data_ptr(), buf.numel(), k, occ, iters, st)
        assert (rc == 0) == ok, (k, occ, iters, rc)
    assert lib.pfw_probe_l2_lines(buf.data_ptr(), 1000, 8, 4, 4, st) != 0   # buffer under 1 MiB
    torch.cuda.synchronize()
