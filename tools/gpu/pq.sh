# Pareto stage timings: C2 bench stages + C5 stress (no profiler), and the Pareto tests
timeout 600 python bench.py --steps 5 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/pq.json 2> gpurun_out/pq.err
python -c "
import json;d=json.load(open('gpurun_out/pq.json')); print('c2', d['ms_per_step'], d['stages_s']); c=d['c5']; print('c5', c['ms_per_step'], c['pareto_filtering_s'], c['stages_s'])"
timeout 900 python -m pytest tests/test_gpu_pareto.py tests/test_gpu_stress.py -x -q 2>&1 | tail -2
