timeout 400 python -m pytest tests/test_parity_gpu.py -q --tb=short -x -k "dws or direct or dp or random" 2>&1 | tail -2
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
python bench.py --global-batch 512 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null| tail -1
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null| tail -1
