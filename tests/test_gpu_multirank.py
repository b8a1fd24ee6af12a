"""Multi-process function-parallel on ONE GPU (2 and 3 ranks, gloo for the host
barriers and gathers): the fused combine through real cross-process CUDA IPC
mappings and the all-reduce combine, each checked against the reference's
golden function-parallel results.  Kernels of different ranks never wait on
each other (completion is a host barrier), so sharing the device is safe."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, golden, gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import conftest
        import paper_1312_4188_b200 as pfw
        from paper_1312_4188_b200 import parallel
        from paper_1312_4188_b200.classifier import first_to_host
        from oracle.oracle import PKT_FIELDS
        c = pfw.CompiledRuleset.from_columns(conftest.golden_rules("r503_s24_w30"), device=0)
        pk = conftest.golden_traffic("t600_s25")
        p = pfw.PacketArrays.from_columns(*[pk[f] for f in PKT_FIELDS], device=0)
        n = len(p)
        out = {}
        # fused, reduce-scatter and all-reduce layouts
        for scatter in (True, False):
            fused = parallel.FusedFunctionParallel(c, n, scatter=scatter)
            for _ in range(3):  # one barrier per call: alternate buffer sets, reset one call ahead
                first, comps = fused.run(p)
                got = (fused.own_range, first_to_host(first), comps.cpu().numpy())
                if ("fused", scatter) in out:
                    assert all(np.array_equal(a, b) for a, b in zip(got[1:], out[("fused", scatter)][1:]))
                out[("fused", scatter)] = got
            fused.close()
        # separate all-reduce combine (gloo here, NCCL on a multi-GPU box)
        import torch
        lo, hi = parallel.rule_shard(c.num_rules, parallel.rank_info())
        first = torch.empty(n, dtype=torch.int32, device="cuda:0")
        comps = torch.empty(n, dtype=torch.int32, device="cuda:0")
        stats = torch.zeros(2, dtype=torch.int64, device="cuda:0")
        pfw._native.check(pfw._native.lib().pfw_accumulator_init(
            n, first.data_ptr(), comps.data_ptr(), torch.cuda.current_stream().cuda_stream), "init")
        c.scan_partition_accumulate(p, lo, hi, first, comps, stats)
        parallel.function_parallel_combine(first, comps, stats)
        out["allreduce"] = ((0, n), first_to_host(first), comps.cpu().numpy(), stats.cpu().numpy())
        # per-rank rule shards (each rank uploads only its partition): fused and all-reduce
        shard = c.shard(lo, hi)
        fused = parallel.FusedFunctionParallel(shard, n, scatter=False)
        f_sh, c_sh = fused.run(p)
        out["shard_fused"] = (first_to_host(f_sh), c_sh.cpu().numpy())
        fused.close()
        first.fill_(2**31 - 1)
        comps.zero_()
        shard.scan_partition_accumulate(p, 0, shard.num_rules, first, comps, None)
        parallel.function_parallel_combine(first, comps, None)
        out["shard_allreduce"] = (first_to_host(first), comps.cpu().numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_function_parallel_multiprocess_one_gpu(world):
    import torch.multiprocessing as mp
    g = golden("engine_r503_t600.npz")
    want_first = g[f"function_{world}_first"]
    want_comps = g[f"function_{world}_comps"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    # reduce-scatter: shards reassemble to the full answer
    firsts, compss = [], []
    for r in range(world):
        (a, b), f, cm = res[r][("fused", True)]
        firsts.append(f[: b - a])
        compss.append(cm[: b - a])
    np.testing.assert_array_equal(np.concatenate(firsts), want_first)
    np.testing.assert_array_equal(np.concatenate(compss), want_comps)
    for r in range(world):
        _, f, cm = res[r][("fused", False)]
        np.testing.assert_array_equal(f, want_first)
        np.testing.assert_array_equal(cm, want_comps)
        _, f, cm, st = res[r]["allreduce"]
        np.testing.assert_array_equal(f, want_first)
        np.testing.assert_array_equal(cm, want_comps)
        total, mx, _ = g[f"function_{world}_stats"].tolist()
        assert st.tolist() == [total, mx]
        for key in ("shard_fused", "shard_allreduce"):
            f, cm = res[r][key]
            np.testing.assert_array_equal(f, want_first)
            np.testing.assert_array_equal(cm, want_comps)


@pytest.mark.parametrize("config", ["data", "function"])
def test_bench_two_ranks_shared_gpu(config):
    """bench.py under torchrun with 2 ranks sharing the one GPU (PFW_SHARE_GPU=1:
    gloo collectives, a functional check of the N>1 path): one JSON line from
    rank 0 with the whole-job packet count and the rank layout."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, PFW_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", config, "--packets", str(1 << 20), "--steps", "3", "--warmup", "3",
           "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    if config == "data":
        # strong by default (BASELINE configs[1]: the packets split over the ranks) + the weak record
        assert d["scaling"] == "strong" and d["config"]["packets"] == 1 << 20 and d["e2e"]["value"] > 0
        assert d["config"]["packets_per_gpu"] == 1 << 19
        assert d["weak"]["packets"] == 2 << 20 and d["weak"]["value"] > 0
    else:
        assert d["config"]["rules_per_gpu"] == [0, 50_000]
