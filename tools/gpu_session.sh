timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for cfg in adversarial data function grid; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['algorithm'])"
done
