"""Small-batch latency of the drop-in API (scratch): Engine.run_arrays from
pinned host columns, classify() of one Packet, 1..64K packets, 10K rules."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1312_4188_b200 as pfw
from oracle import oracle
cols = oracle.gen_ruleset(10_000, 1)
c = pfw.CompiledRuleset.from_columns(cols, device=0)
eng = pfw.Engine(pfw.EngineConfig(pfw.ExecutionModel.DATA_PARALLEL))
for n in (1, 64, 1024, 65536):
    pk = oracle.gen_traffic_uniform(n, 3)
    pinned = {}
    for f, a in pk.items():
        t = torch.empty(a.shape, dtype={1: torch.uint8, 2: torch.int16, 4: torch.int32}[a.itemsize], pin_memory=True)
        t.numpy().view(a.dtype)[:] = a
        pinned[f] = t.numpy().view(a.dtype)
    for _ in range(20): eng.run_arrays(c, pinned)
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); eng.run_arrays(c, pinned); ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e6
    f, v, st = c.classify_host(pinned)
    ts2 = []
    for _ in range(200):
        t0 = time.perf_counter(); c.classify_host(pinned); ts2.append(time.perf_counter() - t0)
    ts2 = np.array(ts2) * 1e6
    print(f"n={n}: run_arrays median {np.median(ts):.0f} us p99 {np.percentile(ts, 99):.0f} us; "
          f"classify_host median {np.median(ts2):.0f} us", flush=True)
rs = pfw.generate_ruleset(pfw.RulesetGenParams(10_000, seed=1))
pkt = pfw.generate_traffic(pfw.TrafficProfile(1, seed=2))[0]
for _ in range(10): pfw.classify(rs, pkt)
ts = []
for _ in range(200):
    t0 = time.perf_counter(); pfw.classify(rs, pkt); ts.append(time.perf_counter() - t0)
print(f"classify(ruleset, packet): median {np.median(ts) * 1e6:.0f} us", flush=True)
