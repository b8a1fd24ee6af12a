timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "edges" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "2g" 2>&1 | tail -5
