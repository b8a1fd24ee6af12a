mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "not fullsize" 2>&1 | tail -4
for cfg in data grid adversarial function oracle; do
  for v in 1 2 4; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e --algo 2 --ms-words $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg words $v', d['value'], d['ms_per_step'])"
  done
done
