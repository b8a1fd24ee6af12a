#!/usr/bin/env python
"""Mpackets/s vs rule count (the BASELINE.json metric's x-axis) on one GPU:
rulesets generate_ruleset(RulesetGenParams(R, seed=1)) (oracle C generator,
bit-identical), packets generate_traffic(TrafficProfile(N, seed=2)) on the
device; for each R the match-set scan (auto representation: plain rows, or
compressed rows when the plain ones exceed the memory budget) and the
rule-by-rule scan, CUDA events, L2 flushed before each timed scan, best of K.
A strided packet subsample is checked against the oracle at every R.

    python tools/rule_sweep.py [--packets N] [--reps K] [--rules 1000,4096,...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rules", default="1000,4096,10000,50000,100000,250000,500000,1000000")
    ap.add_argument("--rule-scan-max", type=int, default=1000000)
    ap.add_argument("--compare-rows", action="store_true",
                    help="also time the match-set scan with plain rows and with compressed rows forced")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE", help="pfw_set_tuning before the sweep")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1312_4188_b200 as pfw
    from paper_1312_4188_b200 import _native
    for kv in args.tune:
        k, _, v = kv.partition("=")
        _native.set_tuning(k, int(v))
    from paper_1312_4188_b200.classifier import NO_MATCH
    from oracle import oracle
    n = args.packets
    p = pfw.generate_traffic_device(pfw.TrafficProfile(count=n, seed=2), device=0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    first = torch.empty(n, dtype=torch.int32, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    idx = torch.arange(0, n, 997, device="cuda:0")
    sub = pfw.PacketArrays(p.data[idx]).columns()
    for R in [int(x) for x in args.rules.split(",")]:
        rules = oracle.gen_ruleset(R, 1)
        t0 = time.perf_counter()
        c = pfw.CompiledRuleset.from_columns(rules, device=0)
        torch.cuda.synchronize()
        create_s = time.perf_counter() - t0
        row = {"rules": R, "packets": n, "create_s": round(create_s, 3),
               "matchset_mib": round(_native.lib().pfw_ruleset_matchset_bytes(c.handle) / 2**20, 1)}
        want = oracle.scan_range(rules, sub, 0, R)
        variants = [(c, 0, "matchset"), (c, 1, "rule_scan")]
        if args.compare_rows:
            for cmpv, key in ((0, "plain"), (1, "compressed")):
                _native.set_tuning("ms_compress", cmpv)
                cv = pfw.CompiledRuleset.from_columns(rules, device=0)
                if _native.lib().pfw_ruleset_matchset_bytes(cv.handle) > 0:
                    variants.append((cv, 0, f"matchset_{key}"))
            _native.set_tuning("ms_compress", 2)
        for cc, algo, key in variants:
            if algo == 1 and R > args.rule_scan_max:
                continue
            _native.set_tuning("algo", algo)
            best = None
            for _ in range(args.reps + 1):
                stats.zero_()
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                cc.scan_range_device(p, 0, R, first=first, stats=stats)
                e1.record()
                e1.synchronize()
                t = e0.elapsed_time(e1)
                best = t if best is None else min(best, t)
            got = first[idx].cpu().numpy().astype(np.int64)
            got[got == NO_MATCH] = -1
            assert np.array_equal(got, want), f"parity failure at R={R} ({key})"
            row[f"{key}_mpps"] = round(n / (best / 1e3) / 1e6, 1)
            row["comparisons_per_packet"] = round(int(stats[0].item()) / n, 1)
        _native.set_tuning("algo", 0)
        print(json.dumps(row), flush=True)
        del c, variants


if __name__ == "__main__":
    main()
