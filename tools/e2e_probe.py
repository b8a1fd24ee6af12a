import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1312_4188_b200 import workloads
from paper_1312_4188_b200.classifier import CompiledRuleset
from paper_1312_4188_b200.engines import Engine, EngineConfig, ExecutionModel
w = workloads.WORKLOADS["data"]
c = CompiledRuleset.from_columns(workloads.rule_columns(w), device=0)
pk = workloads.packets(w, 0, w.packets, 0)
hc = pk.columns()
eng = Engine(EngineConfig(ExecutionModel.DATA_PARALLEL), device=0)
for i in range(4):
    t0 = time.perf_counter(); eng.run_arrays(c, hc); t1 = time.perf_counter()
    print(f"pageable run_arrays {(t1-t0)*1e3:.1f} ms", flush=True)
for i in range(2):
    t0 = time.perf_counter(); c.classify_host(hc); t1 = time.perf_counter()
    print(f"pageable classify_host {(t1-t0)*1e3:.1f} ms", flush=True)
