#!/bin/bash
# The bounds-checked build against the GPU suite, the sanitizer case and one
# bench step of every config; summary into gpurun_out/$1/checked_run.txt.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1
mkdir -p $O
python - <<'PY'
from paper_1312_4188_b200._build import build_native
build_native(force=True, out="build/libpfw_checked.so", defines=["PFW_CHECKS"])
PY
export PFW_LIB=$PWD/build/libpfw_checked.so
R=$O/checked_run.txt
echo "# checked build (-DPFW_CHECKS: device-side traps on every derived index), B200" > $R
echo "## pytest -m gpu (minus full-size) against build/libpfw_checked.so" >> $R
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_gpu_fullsize.py 2>&1 | tail -3 >> $R; echo "rc=${PIPESTATUS[0]}" >> $R
echo "## tools/sanitize_case.py" >> $R
timeout 600 python tools/sanitize_case.py 2>&1 | tail -2 >> $R; echo "rc=${PIPESTATUS[0]}" >> $R
for cfg in data grid function adversarial oracle; do
  echo "## bench.py --config $cfg --steps 2 --warmup 3 (checked build)" >> $R
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --no-e2e > $O/checked_$cfg.json 2>&1; echo "rc=$?" >> $R
  grep -o '"value": [0-9.]*' $O/checked_$cfg.json | head -1 >> $R
done
