timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_dense_c4.py -x -q 2>&1 | tail -3
timeout 300 python tools/c4_profile.py
C4_BATCH=3000 timeout 300 python tools/c4_profile.py
C4_BATCH=3000 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dense -c 12 --csv --log-file gpurun_out/split_launches.csv python tools/c4_profile.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_gemm -s 2 -c 1 -o gpurun_out/c4_gemm python tools/c4_profile.py > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
