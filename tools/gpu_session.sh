timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "compressed or summaries or edges" 2>&1 | tail -2
for cfg in function adversarial data; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --ms-compress 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg cmp', d['value'], d['ms_per_step'])"
done
timeout 900 python tools/rule_sweep.py --rules 250000,1000000 --reps 3 2>&1 | grep "^{"
