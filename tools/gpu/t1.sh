timeout 300 python -m pytest tests/test_gpu_dense.py -x -q 2>&1 | grep -v "^  " | tail -30
