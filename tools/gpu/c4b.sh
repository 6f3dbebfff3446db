C4_CPU=0 timeout 300 python tools/c4_bench.py > gpurun_out/c4_r2.json 2>gpurun_out/c4_r2.err; tail -3 gpurun_out/c4_r2.err; cat gpurun_out/c4_r2.json
