for c in 1 2; do MOMC_SB_CTA=$c timeout 300 python tools/quick_sampler_bench.py 2>&1 | sed "s/^/cta$c /"; done
MOMC_SB_CTA=1 timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
