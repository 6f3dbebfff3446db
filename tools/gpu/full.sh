set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
C4_CPU=0 timeout 300 python tools/c4_bench.py > gpurun_out/c4.json 2>gpurun_out/c4.err; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.json
