timeout 900 python -m pytest tests/test_parity_gpu.py -q --tb=short -x 2>&1 | tail -2
