mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final/bench.json 2>gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final/ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/final/launch_ncu.log 2>&1; echo ncu rc=$?
