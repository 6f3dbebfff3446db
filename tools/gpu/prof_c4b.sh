timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_dense_c4.py -x -q 2>&1 | tail -3
timeout 300 python tools/c4_profile.py && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_fused -s 1 -c 1 -o gpurun_out/c4_fused_g python tools/c4_profile.py > gpurun_out/ncu_c4g.log 2>&1
tail -2 gpurun_out/ncu_c4g.log
