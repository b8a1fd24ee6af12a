mkdir -p gpurun_out
./tools/l2_probe > gpurun_out/l2_probe.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for cfg in data grid adversarial function oracle; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'])"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ms_default.json 2>&1; tail -1 gpurun_out/ms_default.json | cut -c1-400
