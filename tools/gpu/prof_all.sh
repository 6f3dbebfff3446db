# launch list of two C2 steps + one --set full capture of the sampler (profiles/ evidence)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$1_launches.csv python tools/profile_step.py > gpurun_out/$1_step.log 2>&1
bash tools/gpu/prof_samp.sh $1_sampler
