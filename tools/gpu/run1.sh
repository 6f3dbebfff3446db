set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dense.py -x -q -s 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_dense_c4.py -x -q -s 2>&1 | tail -15
C4_CPU=0 timeout 300 python tools/c4_bench.py > gpurun_out/c4_r2a.json 2>gpurun_out/c4_r2a.err; tail -3 gpurun_out/c4_r2a.err; cat gpurun_out/c4_r2a.json
