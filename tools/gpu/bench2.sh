set -x
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err
