for c in 0 1 2; do MOMC_SB_CTA=$c timeout 300 python tools/quick_sampler_bench.py 2>&1 | sed "s/^/cta$c /"; done
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
MOMC_SB_CTA=2 timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
