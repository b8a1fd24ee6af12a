#!/usr/bin/env python
"""Per-rank work of the function-parallel model, measured shard by shard on
ONE GPU: for G = 1, 2, 4, 8 the 100K-rule BASELINE ruleset is split into G
rule shards (partition_bounds, engines.py:316-321), each uploaded on its own
(its own match sets), and each shard's accumulate-scan of the replicated
16Mi-packet batch is timed with CUDA events (L2 flushed before each).  The
max over shards is the scan time one rank of a G-GPU job spends per step
(the MIN/SUM combine -- NCCL all-reduce or the fused NVLink epilogue -- is
not included).  This is a per-rank compute measurement, not a multi-GPU run.

    python tools/function_shards.py [--packets N] [--reps K]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1312_4188_b200 as pfw
    from paper_1312_4188_b200 import _native, workloads
    from paper_1312_4188_b200.classifier import NO_MATCH
    w = workloads.WORKLOADS["function"]
    cols = workloads.rule_columns(w)
    R = len(cols["proto"])
    p = workloads.packets(w, 0, args.packets, 0)
    n = len(p)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    first = torch.empty(n, dtype=torch.int32, device="cuda:0")
    comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
    out = []
    for G in (1, 2, 4, 8):
        times, sizes, work = [], [], []
        for lo, hi in pfw.partition_bounds(R, G):
            s = pfw.CompiledRuleset.from_columns({k: v[lo:hi] for k, v in cols.items()}, device=0, shard=(lo, R))
            sizes.append(int(_native.lib().pfw_ruleset_matchset_bytes(s.handle)))
            best = None
            for _ in range(args.reps + 1):
                first.fill_(NO_MATCH)
                comps.zero_()
                stats.zero_()
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                s.scan_partition_accumulate(p, 0, s.num_rules, first, comps, stats)
                e1.record()
                e1.synchronize()
                t = e0.elapsed_time(e1)
                best = t if best is None else min(best, t)
            times.append(best)
            work.append(int(stats[0].item()) / n)
            del s
        row = {"G": G, "max_shard_ms": round(max(times), 3), "shard_ms": [round(t, 3) for t in times],
               "per_rank_mpps": round(n / (max(times) / 1e3) / 1e6, 1),
               "matchset_mib_per_rank": round(max(sizes) / 2**20, 1),
               "comparisons_per_packet_per_rank": round(max(work), 1)}
        out.append(row)
        print(json.dumps(row), flush=True)
    return out


if __name__ == "__main__":
    main()
