# one ncu --set full capture of the C2 sampler launch -> gpurun_out/$1.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sb_(small|batch)_kernel" -c 1 -o gpurun_out/$1 python tools/profile_sampler.py dsb > gpurun_out/$1.log 2>&1
tail -3 gpurun_out/$1.log
