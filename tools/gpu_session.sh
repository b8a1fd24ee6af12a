for cfg in function data; do
for pf in 0 1; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --ms-prefetch $pf 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg pf $pf', d['value'], d['ms_per_step'])"
done
done
for g in 8 16; do
    timeout 300 python bench.py --config function --steps 10 --warmup 3 --no-cpu --no-e2e --ms-prefetch 1 --ms-group $g 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('function pf 1 g $g', d['value'], d['ms_per_step'])"
done
