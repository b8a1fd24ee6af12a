"""e2e timing breakdown on the GPU box (scratch): C-side call time (PFW_E2E_TRACE)
vs the Python API call, pinned and pageable host columns."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_1312_4188_b200 import workloads
from paper_1312_4188_b200.classifier import CompiledRuleset
from paper_1312_4188_b200.engines import Engine, EngineConfig, ExecutionModel
w = workloads.WORKLOADS["data"]
c = CompiledRuleset.from_columns(workloads.rule_columns(w), device=0)
pk = workloads.packets(w, 0, w.packets, 0)
hc = pk.columns()
pinned = {}
for f, a in hc.items():
    t = torch.empty(a.shape, dtype={1: torch.uint8, 2: torch.int16, 4: torch.int32}[a.itemsize], pin_memory=True)
    t.numpy().view(a.dtype)[:] = a
    pinned[f] = t.numpy().view(a.dtype)
eng = Engine(EngineConfig(ExecutionModel.DATA_PARALLEL), device=0)
for name, batch in (("pinned", pinned), ("pageable", hc)):
    for i in range(4):
        t0 = time.perf_counter(); eng.run_arrays(c, batch); t1 = time.perf_counter()
        print(f"{name} run_arrays {(t1-t0)*1e3:.2f} ms", flush=True)
