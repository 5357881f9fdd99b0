timeout 600 python -m pytest tests/test_parity_gpu.py -q --tb=line -x -k "tma or variants or config1 or random" 2>&1 | tail -3
python tools/layer_bench.py --layer l2.1a,l3.1a,l4.1a,l2.0a,l4.0sc --op fwd,dx --reps 10 --math 3xtf32
