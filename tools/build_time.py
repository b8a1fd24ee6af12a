"""Ruleset compile time (pfw_ruleset_create: match-set build on the device) vs rule count (scratch)."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1312_4188_b200 as pfw
from paper_1312_4188_b200 import _native
from oracle import oracle
torch.cuda.init(); torch.zeros(1, device="cuda:0")
for R in (1000, 10_000, 50_000, 100_000, 1_000_000):
    cols = oracle.gen_ruleset(R, 1)
    c = pfw.CompiledRuleset.from_columns(cols, device=0); del c  # warm
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); c = pfw.CompiledRuleset.from_columns(cols, device=0); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        info = (_native.ruleset_info(c.handle, "compressed"), _native.ruleset_info(c.handle, "summaries"), int(_native.lib().pfw_ruleset_matchset_bytes(c.handle)))
        del c
    print(f"R={R}: build {min(ts)*1e3:.1f} ms (compressed, summaries, bytes) = {info}", flush=True)
