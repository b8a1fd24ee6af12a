mkdir -p gpurun_out/final
timeout 600 python bench.py > gpurun_out/final/bench.json 2>gpurun_out/final/bench.err
for cfg in grid adversarial function oracle; do
  timeout 600 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu > gpurun_out/final/$cfg.json 2>&1
done
timeout 600 python bench.py --config function --steps 30 --warmup 3 --no-cpu --fused > gpurun_out/final/function_fused.json 2>&1
echo done
