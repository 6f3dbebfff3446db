set -x
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_gloo_merge.py tests/test_gpu_sampler.py tests/test_gpu_dense.py tests/test_gpu_fuzz.py tests/test_gpu_stress.py tests/test_gpu_session_reuse.py -x -q 2>&1 | tail -15
