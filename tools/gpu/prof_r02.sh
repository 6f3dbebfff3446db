# round-2 profile evidence (profiles/): C2 step launch list, C4 GEMM + update full captures,
# C5 launch list + one full capture of its dedup kernel
export C4_BATCH=3000
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2_launches.csv python tools/profile_step.py > gpurun_out/r02_c2_step.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dense_gemm -s 5 -c 1 -o gpurun_out/r02_c4_gemm python tools/c4_profile.py > gpurun_out/r02_c4_gemm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python tools/c4_profile.py > gpurun_out/r02_c4_launches.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches.csv python tools/c5_stress.py 100 > gpurun_out/r02_c5_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dedup -c 1 -o gpurun_out/r02_c5_dedup python tools/c5_stress.py 100 > gpurun_out/r02_c5_dedup.log 2>&1
ls -la gpurun_out/
