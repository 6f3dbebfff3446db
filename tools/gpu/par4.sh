timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/p4_launches.csv python tools/profile_step.py > gpurun_out/p4_step.log 2>&1
