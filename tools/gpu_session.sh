mkdir -p gpurun_out/final
timeout 600 python - <<'PY'
import time, torch
import paper_1312_4188_b200 as pfw
from paper_1312_4188_b200 import _native, workloads
torch.cuda.init()
for name in ["oracle", "grid", "data", "adversarial", "function"]:
    w = workloads.WORKLOADS[name]
    cols = workloads.rule_columns(w)
    for rep in range(2):
        t0 = time.perf_counter()
        c = pfw.CompiledRuleset.from_columns(cols, device=0)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"create {name:12s} R={w.rules:6d}: {dt*1e3:8.1f} ms, match sets {_native.lib().pfw_ruleset_matchset_bytes(c.handle)/2**20:8.1f} MiB", flush=True)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/final/launch_ncu.log 2>&1; echo ncu rc=$?
