mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r1_bench.json 2>gpurun_out/r1_bench.err; tail -1 gpurun_out/r1_bench.json | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/r1_ref.json 2>&1; tail -1 gpurun_out/r1_ref.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r1_ncu.log 2>&1; echo ncu rc=$?
