set -x
timeout 300 python tools/quick_sampler_bench.py
bash tools/gpu/prof_samp.sh base0
