timeout 500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q --tb=short -x 2>&1 | tail -2
python tools/layer_bench.py --layer l2.0a,l2.1a,l3.0a,l3.1a,l4.0a,l4.1a,l2.0sc,l3.0sc --op fwd,dx --reps 10
python tools/layer_bench.py --layer l2.0a,l3.0a --op dx --reps 10 --math tf32
