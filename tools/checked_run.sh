#!/usr/bin/env bash
# Bounds-checked build (-DPFW_CHECKS: device-side asserts on every derived
# index) and the GPU suite + sanitizer case + one bench step against it.
# compute-sanitizer is closed on the GPU pool; this is the substitute.
set -euo pipefail
cd "$(dirname "$0")/.."
python - <<'PY'
from paper_1312_4188_b200._build import build_native
build_native(force=True, out="build/libpfw_checked.so", defines=["PFW_CHECKS"])
PY
export PFW_LIB=build/libpfw_checked.so
python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_fullsize.py
python tools/sanitize_case.py
python bench.py --steps 2 --warmup 1 --no-cpu
