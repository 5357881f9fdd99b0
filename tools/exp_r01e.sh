timeout 600 python -m pytest tests/test_parity_gpu.py -q --tb=short -x 2>&1 | tail -2
python tools/layer_bench.py --layer l2.0sc,l3.0sc,l4.0sc --op dx --reps 20
