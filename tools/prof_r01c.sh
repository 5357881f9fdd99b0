ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 0 -c 1 -o gpurun_out/prof7_l1fwd_3x python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu7.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 0 -c 1 -o gpurun_out/prof7_l1fwd_tf32 python bench.py --math tf32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu7.log 2>&1
tail -2 gpurun_out/ncu7.log
