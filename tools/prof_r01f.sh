ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01f_bench.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_tma_kernel<\(int\)3' -s 0 -c 1 -o gpurun_out/prof_r01f_l1dw python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01f_full.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_direct_fwd' -s 0 -c 1 -o gpurun_out/prof_r01f_stem python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_r01f_full.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_strip_kernel' -s 0 -c 1 -o gpurun_out/prof_r01f_l1fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_r01f_full.log 2>&1
ls gpurun_out | grep r01f
