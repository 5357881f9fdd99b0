ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_tma_kernel<3" -s 0 -c 1 -o gpurun_out/prof_r01e_l1dw python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01e.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_tma_kernel<1, 128, 2" -s 0 -c 1 -o gpurun_out/prof_r01e_l2dx python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_r01e.log 2>&1
grep -c "Profiling" gpurun_out/ncu_r01e.log
