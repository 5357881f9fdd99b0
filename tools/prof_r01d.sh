# launch list of the default bench (2 timed steps after 3 warm-up) and a full capture of the top kernel
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01d.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01d_bench.log 2>&1
# l1.0a dW is the 3rd conv_tma launch of a step (fwd layers run strip/generic first): capture the first dwT kernel
ncu --set full --clock-control none --import-source on -k regex:"conv_tma_kernel<3" -s 0 -c 1 -o gpurun_out/prof_r01d_l1dw python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01d_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"conv_strip_kernel" -s 0 -c 1 -o gpurun_out/prof_r01d_l1fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_r01d_full.log 2>&1
tail -3 gpurun_out/ncu_r01d_full.log
