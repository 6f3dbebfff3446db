timeout 900 python -m pytest tests/test_gpu_pareto.py tests/test_gpu_trace.py tests/test_gpu_multishard.py tests/test_gpu_stress.py tests/test_gpu_session_reuse.py tests/test_gpu_group.py -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-tto --no-cpu-baseline > gpurun_out/pb.json 2> gpurun_out/pb.err; tail -3 gpurun_out/pb.err
python -c "import json; d=json.load(open('gpurun_out/pb.json')); print(d['ms_per_step'], d['stages_s'], d['hv_equals_reference'])"
