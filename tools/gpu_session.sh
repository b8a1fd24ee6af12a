mkdir -p gpurun_out/verify
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --impl reference > gpurun_out/verify/ref.json 2>&1; tail -1 gpurun_out/verify/ref.json | cut -c1-120
