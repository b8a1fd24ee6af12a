timeout 1500 python -m pytest tests -x -q -m gpu -k "not fullsize" 2>&1 | tail -3
for cfg in data function; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'])"
done
timeout 300 python bench.py --config function --steps 10 --warmup 3 --no-cpu --no-e2e --fused 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('function fused', d['value'], d['ms_per_step'])"
PFW_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --config function --fused --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('function N=2 shared fused', d['value'], d['config']['rules_per_gpu'], d['config']['algorithm'])"
