set -x
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_gpu_dropin.py -x -q -s 2>&1 | tail -30
