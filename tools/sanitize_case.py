"""Small case exercising every kernel path, checked against the oracle; run
under compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1312_4188_b200 as pfw  # noqa: E402
from paper_1312_4188_b200 import _native  # noqa: E402
from paper_1312_4188_b200.parallel import FusedFunctionParallel  # noqa: E402
from oracle import oracle  # noqa: E402

torch.cuda.set_device(0)
rules = oracle.gen_ruleset(700, 11, wp=0.3)
rules["proto"][::31] = 47
pk = oracle.gen_traffic_uniform(3000, 12)
pk["proto"][::5] = 17
c = pfw.CompiledRuleset.from_columns(rules, device=0)
p = pfw.PacketArrays.from_columns(*[pk[f] for f in oracle.PKT_FIELDS], device=0)
checks = 0
for fp in (64, 1024):           # multi-pass with several passes / a single pass
    _native.set_tuning("first_pass", fp)
    for split in (0, 1):        # single table / protocol-split chains + bucketing
        _native.set_tuning("proto_split", split)
        for lo, hi in ((0, 700), (37, 650)):
            np.testing.assert_array_equal(c.scan_range(p, lo, hi), oracle.scan_range(rules, pk, lo, hi))
            checks += 1
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=3)).run_arrays(c, p)
        first, comps, total, mx = oracle.engine_run(rules, pk, "function", 3)
        np.testing.assert_array_equal(res.first, first)
        np.testing.assert_array_equal(res.comparisons, comps)
        checks += 1
_native.set_tuning("proto_split", 0)
# match-set scan: every step shape, block summaries off / on, windows, partitions
for summary in (0, 1):
    _native.set_tuning("ms_summary", summary)   # applies to rulesets built from here on
    cs = pfw.CompiledRuleset.from_columns(rules, device=0)
    _native.set_tuning("algo", 2)
    for group, words in ((8, 4), (8, 2), (16, 4), (16, 2), (32, 2), (32, 1)):
        _native.set_tuning("ms_group", group)
        _native.set_tuning("ms_words", words)
        for lo, hi in ((0, 700), (37, 650), (699, 700)):
            np.testing.assert_array_equal(cs.scan_range(p, lo, hi), oracle.scan_range(rules, pk, lo, hi))
            checks += 1
        res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=3)).run_arrays(cs, p)
        np.testing.assert_array_equal(res.first, oracle.engine_run(rules, pk, "function", 3)[0])
        checks += 1
    _native.set_tuning("ms_group", 0)
    _native.set_tuning("ms_words", 4)
    _native.set_tuning("algo", 0)
_native.set_tuning("ms_summary", 2)
# compressed rows (forced), with and without summaries, windows and partitions
for summary in (0, 1):
    _native.set_tuning("ms_summary", summary)
    _native.set_tuning("ms_compress", 1)
    cc = pfw.CompiledRuleset.from_columns(rules, device=0)
    _native.set_tuning("algo", 2)
    for lo, hi in ((0, 700), (37, 650), (699, 700)):
        np.testing.assert_array_equal(cc.scan_range(p, lo, hi), oracle.scan_range(rules, pk, lo, hi))
        checks += 1
    res = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.FUNCTION_PARALLEL, nodes=3)).run_arrays(cc, p)
    np.testing.assert_array_equal(res.first, oracle.engine_run(rules, pk, "function", 3)[0])
    checks += 1
    _native.set_tuning("algo", 0)
_native.set_tuning("ms_compress", 2)
_native.set_tuning("ms_summary", 2)
adv_rules = oracle.adversarial_rules(50_000)
adv_pk = oracle.adversarial_traffic(4_000)
ca = pfw.CompiledRuleset.from_columns(adv_rules, device=0)
pa = pfw.PacketArrays.from_columns(*[adv_pk[f] for f in oracle.PKT_FIELDS], device=0)
for lo, hi in ((0, 50_000), (1000, 45_003)):
    np.testing.assert_array_equal(ca.scan_range(pa, lo, hi), oracle.scan_range(adv_rules, adv_pk, lo, hi))
    checks += 1
fused = FusedFunctionParallel(c, len(p))
f, cm = fused.run(p)
np.testing.assert_array_equal(pfw.classifier.first_to_host(f), oracle.engine_run(rules, pk, "function", 1)[0])
fused.close()
g = pfw.generate_traffic_device(pfw.TrafficProfile(5000, seed=3, sport_range=pfw.PortRange(10, 2009)), device=0)
gh = g.columns()
ref = oracle.gen_traffic_uniform(5000, 3, sport_lo=10, sport_hi=2009)
for k in oracle.PKT_FIELDS:
    np.testing.assert_array_equal(gh[k], ref[k])
torch.cuda.synchronize()
print(f"sanitize case ok: {checks + 2} checks")
