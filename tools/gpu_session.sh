mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --config adversarial --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ms_scan -s 3 -c 1 -o gpurun_out/ms_adv -f \
  python bench.py --config adversarial --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_adv.log 2>&1
echo ncu rc=$?
