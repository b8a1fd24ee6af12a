mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "not fullsize" 2>&1 | tail -3
for cfg in adversarial data function grid; do
  for sm in 0 1 2; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --ms-summary $sm 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg summary $sm', d['value'], d['ms_per_step'])"
  done
done
