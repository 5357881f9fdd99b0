timeout 600 python -m pytest tests/test_parity_gpu.py -q --tb=line -x -k "tma or variants or config1" 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench5.json 2> gpurun_out/bench5.err; cp gpurun_out/bench_layers.json gpurun_out/bench5_layers.json
ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 0 -c 1 -o gpurun_out/prof5_l1fwd_tf32 python bench.py --math tf32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tma_kernel -s 0 -c 1 -o gpurun_out/prof5_l1fwd_3x python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline >> gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu5.log; cut -c1-300 gpurun_out/bench5.json
