"""Several GPUs for real (skipped unless >= 2 CUDA devices are visible):

* one process per GPU with NCCL: function-parallel rule shards combined by the
  NCCL MIN / SUM all-reduce and by the fused NVLink-atomic epilogue across
  two devices (CUDA IPC peer mappings), and data-parallel packet shards with
  no collective -- each against the reference's golden results
  (engines.py:302-357, :202-212);
* one process driving both GPUs: Engine(devices=[0, 1]) (in-process peer
  access, the fused combine into the owner device's buffers);
* bench.py --gpus 2 spawning its own NCCL ranks.

The one-GPU box of the build loop cannot run these; the same logic is
covered there by virtual devices (tests/test_gpu_engine_api.py), ranks
sharing one GPU (tests/test_gpu_multirank.py) and gloo on CPU
(tests/test_parallel_gloo.py)."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden, golden_rules, golden_traffic

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs at least two CUDA devices", allow_module_level=True)

import paper_1312_4188_b200 as pfw  # noqa: E402
from oracle.oracle import PKT_FIELDS  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    try:
        import conftest
        import paper_1312_4188_b200 as pfw
        from paper_1312_4188_b200 import parallel
        from paper_1312_4188_b200.classifier import first_to_host
        out = {"backend": dist.get_backend()}
        info = parallel.rank_info()
        # function-parallel at 100K rules: this rank uploads only its rule shard
        rules = conftest.golden_rules("r100000_s1")
        c = pfw.CompiledRuleset.from_columns(rules, device=rank)
        p = pfw.generate_traffic_device(pfw.TrafficProfile(count=2000, seed=2), device=rank)
        n = len(p)
        lo, hi = parallel.rule_shard(c.num_rules, info)
        shard = c.shard(lo, hi)
        first = torch.full((n,), 2**31 - 1, dtype=torch.int32, device=f"cuda:{rank}")
        comps = torch.zeros(n, dtype=torch.int32, device=f"cuda:{rank}")
        stats = torch.zeros(2, dtype=torch.int64, device=f"cuda:{rank}")
        shard.scan_partition_accumulate(p, 0, shard.num_rules, first, comps, stats)
        parallel.function_parallel_combine(first, comps, stats)  # NCCL MIN / SUM / MAX
        out["nccl"] = (first_to_host(first), comps.cpu().numpy(), stats.cpu().numpy())
        # the fused combine across the two devices (NVLink atomics through IPC)
        fused = parallel.FusedFunctionParallel(shard, n, scatter=True)
        f_sh, c_sh = fused.run(p)
        out["fused"] = (fused.own_range, first_to_host(f_sh), c_sh.cpu().numpy())
        fused.close()
        # data-parallel: this rank's packet shard of the oracle config, no collective
        c1 = pfw.CompiledRuleset.from_columns(conftest.golden_rules("r1000_s1"), device=rank)
        a, b = parallel.packet_shard(100_000, info)
        pk = pfw.generate_traffic_device(pfw.TrafficProfile(count=100_000, seed=2), device=rank, start=a, count=b - a)
        out["data"] = ((a, b), first_to_host(c1.scan_range_device(pk, 0, 1000)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_nccl_ranks_on_two_devices():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    g = golden("engine_r100000_t2000.npz")
    for r in range(world):
        assert res[r]["backend"] == "nccl"
        f, cm, st = res[r]["nccl"]
        np.testing.assert_array_equal(f, g["function_2_first"])
        np.testing.assert_array_equal(cm, g["function_2_comps"])
        assert st.tolist()[0] == int(g["function_2_stats"][0])
    firsts = np.concatenate([res[r]["fused"][1][: res[r]["fused"][0][1] - res[r]["fused"][0][0]] for r in range(world)])
    comps = np.concatenate([res[r]["fused"][2][: res[r]["fused"][0][1] - res[r]["fused"][0][0]] for r in range(world)])
    np.testing.assert_array_equal(firsts, g["function_2_first"])
    np.testing.assert_array_equal(comps, g["function_2_comps"])
    data = np.concatenate([res[r]["data"][1] for r in range(world)])
    np.testing.assert_array_equal(data, golden("scan_oracle_r1000_t100000.npz")["first"])


@pytest.mark.parametrize("model", ["data", "function", "hybrid"])
def test_engine_drives_two_devices(model):
    g = golden("engine_r503_t600.npz")
    c = pfw.CompiledRuleset.from_columns(golden_rules("r503_s24_w30"), device=0)
    cols = golden_traffic("t600_s25")
    p = pfw.PacketArrays.from_columns(*[cols[f] for f in PKT_FIELDS], device=0)
    for shard in ("rules", "packets"):
        eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.from_key(model), nodes=8, gpus=2, shard=shard))
        assert eng.devices == [0, 1]
        for batch in (p, cols):
            res = eng.run_arrays(c, batch)
            np.testing.assert_array_equal(res.first, g[f"{model}_8_first"])
            np.testing.assert_array_equal(res.comparisons, g[f"{model}_8_comps"])


def test_bench_spawns_nccl_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--packets", str(1 << 22),
                        "--steps", "3", "--warmup", "3", "--no-cpu", "--no-rule-scan"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["config"]["packets_per_gpu"] == 1 << 21 and d["weak"]["value"] > 0
