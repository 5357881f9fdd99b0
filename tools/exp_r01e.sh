timeout 400 python -m pytest tests/test_parity_gpu.py -q --tb=short -x 2>&1 | tail -3
for m in 3xtf32 tf32; do for v in 5 2; do python tools/layer_bench.py --layer l1.1b --op dw --reps 20 --math $m --variant $v; done; done
python bench.py 2>&1 | tail -1
