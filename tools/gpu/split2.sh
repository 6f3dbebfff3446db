timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_dense_c4.py -x -q 2>&1 | tail -3
C4_BATCH=3000 timeout 300 python tools/c4_profile.py
C4_BATCH=3000 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dense -c 6 --csv --log-file gpurun_out/split_launches2.csv python tools/c4_profile.py > /dev/null 2>&1
