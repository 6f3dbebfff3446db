timeout 300 python tools/quick_sampler_bench.py
MOMC_SAMPLER_WS=0 timeout 300 python tools/quick_sampler_bench.py
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
