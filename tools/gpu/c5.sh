timeout 600 python tools/c5_stress.py 100 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dedup|k_eval_int|k_collapse" -c 6 --csv python tools/c5_stress.py 100 > gpurun_out/c5_ncu.csv 2>&1; tail -20 gpurun_out/c5_ncu.csv | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_pareto.py -x -q 2>&1 | tail -2
