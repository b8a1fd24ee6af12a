./tools/l2_probe 2>&1 | grep "64B"
for g in 4 8; do
for cfg in data grid function; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --ms-group $g --ms-words 4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('g$g $cfg', d['value'], d['ms_per_step'])"
done
done
