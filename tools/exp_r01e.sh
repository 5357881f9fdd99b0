timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q --tb=short -x 2>&1 | tail -2
python tools/layer_bench.py --layer l2.1a,l3.1a,l4.1a,l3.0a,l4.0a --op dw --reps 10
python bench.py --no-cpu-baseline --no-e2e --layers-out gpurun_out/l3x_r01l.json 2>/dev/null | tail -1
