#!/bin/bash
# Round-end evidence run on one B200: GPU suite, smoke, every bench config +
# the reference arm, the default command's launch list, ncu captures of the
# three top kernels.  Outputs under gpurun_out/$1/.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for cfg in oracle grid function adversarial; do
  timeout 600 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 600 python bench.py --config function --fused --no-cpu > $O/bench_function_fused.json 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ms_lean_kernel -c 1 -o $O/ms_lean_data python bench.py --config data --steps 1 --warmup 3 --no-e2e --no-cpu --no-rule-scan > $O/ncu_data.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ms_lean_cmp_kernel -c 1 -o $O/ms_lean_cmp_function python bench.py --config function --steps 1 --warmup 3 --no-e2e --no-cpu --no-rule-scan > $O/ncu_function.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ms_lean_sum_kernel -c 1 -o $O/ms_lean_sum_adversarial python bench.py --config adversarial --steps 1 --warmup 3 --no-e2e --no-cpu --no-rule-scan > $O/ncu_adv.log 2>&1
echo done > $O/DONE
