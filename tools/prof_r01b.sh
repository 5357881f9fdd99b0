# l1.0a fwd (first TMA launch) and l3.1a fwd (a BN=256 layer) in TF32 mode, full sets
ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 0 -c 1 -o gpurun_out/prof6_l1fwd_tf32 python bench.py --math tf32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 12 -c 1 -o gpurun_out/prof6_l3fwd_tf32 python bench.py --math tf32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu6.log 2>&1
tail -2 gpurun_out/ncu6.log
