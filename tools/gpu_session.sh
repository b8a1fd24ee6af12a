mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "not fullsize" 2>&1 | tail -3
for cfg in adversarial data; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu > gpurun_out/b_$cfg.json 2>&1; tail -1 gpurun_out/b_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', d['value'], r['frac'], r.get('blocks_read_per_packet'), r['algorithmic_bytes_per_packet'], d['e2e']['value'], d['config']['algorithm'])"
done
