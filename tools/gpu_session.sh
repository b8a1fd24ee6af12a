timeout 1500 python tools/rule_sweep.py 2>&1 | grep "^{"
timeout 600 python bench.py --config adversarial --steps 30 --warmup 3 --no-cpu > gpurun_out/final/adversarial.json 2>&1; tail -1 gpurun_out/final/adversarial.json | cut -c1-100
