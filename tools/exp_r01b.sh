timeout 600 python -m pytest tests/test_parity_gpu.py -q --tb=line -x -k "tma or variants or config1" 2>&1 | tail -2
python tools/layer_bench.py --layer l1.0a,l2.1a,l4.1a --op fwd,dx,dw --reps 10 --math 3xtf32
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8.json 2> gpurun_out/bench8.err; cp gpurun_out/bench_layers.json gpurun_out/bench8_layers.json; cut -c1-200 gpurun_out/bench8.json
