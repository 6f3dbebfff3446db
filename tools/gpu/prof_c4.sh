set -x
timeout 300 python tools/c4_profile.py && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_fused -s 1 -c 1 -o gpurun_out/c4_fused python tools/c4_profile.py > gpurun_out/ncu_c4.log 2>&1
tail -5 gpurun_out/ncu_c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_tc -c 1 -o gpurun_out/c4_eval python tools/c4_profile.py > gpurun_out/ncu_c4e.log 2>&1
tail -3 gpurun_out/ncu_c4e.log
