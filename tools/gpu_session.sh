mkdir -p gpurun_out/final
timeout 600 python bench.py > gpurun_out/final/bench.json 2>gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final/ref.json 2>&1
for cfg in grid adversarial function oracle; do
  timeout 600 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu > gpurun_out/final/$cfg.json 2>&1
done
timeout 600 python bench.py --config function --steps 30 --warmup 3 --no-cpu --fused > gpurun_out/final/function_fused.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ms_scan -s 3 -c 1 -o gpurun_out/final/ms_data -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/final/ncu.log 2>&1
echo ncu rc=$?
