"""Multi-rank sharding logic of the two parallel-firewall models, run as
world_size-2 (and 3) gloo process groups on CPU.  The oracle stands in for
the per-GPU scan kernel; what is tested is the rank logic: shard boundaries,
the MIN / SUM / MAX combines and the resulting reference semantics
(engines.py:143-154, 202-212, 302-321, 359-369)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, golden, golden_rules, golden_traffic


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, model, rules_name, traffic_name, golden_name, key, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1312_4188_b200 import parallel
        from paper_1312_4188_b200.parallel import NO_MATCH
        import conftest
        rules = conftest.golden_rules(rules_name)
        pk = conftest.golden_traffic(traffic_name)
        R = len(rules["proto"])
        N = len(pk["proto"])
        info = parallel.rank_info()
        if model == "function":
            def scan(lo, hi):
                f = oracle.scan_range(rules, pk, lo, hi, 1)
                first = torch.tensor(np.where(f >= 0, f, NO_MATCH), dtype=torch.int32)
                comps = torch.tensor(np.where(f >= 0, f - lo + 1, hi - lo), dtype=torch.int32)
                stats = torch.tensor([int(comps.sum()), int(comps.max()) if N else 0], dtype=torch.int64)
                return first, comps, stats
            first, comps, stats = parallel.run_function_parallel(scan, R)
            out = (first.numpy(), comps.numpy(), stats.numpy())
        else:
            def scan(a, b):
                sub = {k: v[a:b] for k, v in pk.items()}
                f = oracle.scan_range(rules, sub, 0, R, 1)
                comps = oracle.sequential_comparisons(f, R)
                stats = torch.tensor([int(comps.sum()), int(comps.max()) if len(f) else 0], dtype=torch.int64)
                return (torch.tensor(np.where(f >= 0, f, NO_MATCH), dtype=torch.int32),
                        torch.tensor(comps, dtype=torch.int32), stats)
            (a, b), first, comps, stats = parallel.run_data_parallel(scan, N, reduce=True)
            gathered = [None] * world
            dist.all_gather_object(gathered, (a, b, first.numpy(), comps.numpy()))
            order = sorted(gathered, key=lambda g: g[0])
            out = (np.concatenate([g[2] for g in order]), np.concatenate([g[3] for g in order]),
                   stats.numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_function_parallel_ranks_match_reference(world):
    # each rank = one rule shard = one function-parallel node, so the combined
    # counters equal the reference model with nodes = world (engines.py:316-369)
    g = golden("engine_r503_t600.npz")
    res = _run(world, "function", "r503_s24_w30", "t600_s25", None, None)
    want_first = g[f"function_{world}_first"]
    for rank, (first, comps, stats) in res.items():
        got = np.where(first == 0x7FFFFFFF, -1, first)
        np.testing.assert_array_equal(got, want_first)
        np.testing.assert_array_equal(comps, g[f"function_{world}_comps"])
        total, mx, _ = g[f"function_{world}_stats"].tolist()
        assert stats.tolist() == [total, mx]


def test_data_parallel_ranks_match_reference():
    g = golden("scan_r300_t10000.npz")
    res = _run(2, "data", "r300_s40_w30", "t10000_s41", None, None)
    first, comps, stats = res[0]
    got = np.where(first == 0x7FFFFFFF, -1, first)
    np.testing.assert_array_equal(got, g["first"])
    assert stats.tolist() == [int(g["total_comparisons"]), int(g["max_worker_comparisons"])]
