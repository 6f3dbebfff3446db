timeout 900 python bench.py --steps 3 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/pb.json 2> gpurun_out/pb.err
python -c "
import json;d=json.load(open('gpurun_out/pb.json')); print(d['ms_per_step'], d['stages_s']['pareto_filtering_s']); c=d['c4']; print('c4', c['ms_per_step'], c['sampling_s'], c['pareto_filtering_s'], c['stages_s']); print('c5', d['c5']['ms_per_step'], d['c5']['pareto_filtering_s'])"
