timeout 900 python bench.py --steps 10 --warmup 3 --no-tto --no-extra --no-cpu-baseline > gpurun_out/pb.json 2> gpurun_out/pb.err; tail -5 gpurun_out/pb.err
python -c "
import json;d=json.load(open('gpurun_out/pb.json')); print(d['value'], d['ms_per_step'], d['step_ms'], d['e2e']['value'], d['e2e']['ms_per_step'], d['hv_equals_reference'], d['gpu_launches'], d['stages_s']['sampling_s'], d['roofline']['kernel_share_of_step'])"
