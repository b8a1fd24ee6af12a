for cfg in oracle data; do
  for g in "" "--graph"; do
    timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-e2e $g 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $g', d['value'], d['ms_per_step'], d['gpu_launches'])"
  done
done
