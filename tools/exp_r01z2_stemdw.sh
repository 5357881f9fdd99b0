# r01z2: stem dW heuristic (GENERIC below 32768 rows) — full GPU suite + whole-net A/B (head = SMCONV_DIRECT_DW_MIN_ROWS=0)
D=gpurun_out/r01z2; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --tb=short > $D/tests.log 2>&1; tail -2 $D/tests.log
for rep in 1 2; do for m in 0 32768; do
  echo "min_rows=$m rep $rep"
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' vgg 3x', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3), d['roofline']['kernel'][:24])"
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' vgg tf32', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3), d['roofline']['kernel'][:24])"
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 300 python bench.py --net googlenet --global-batch 256 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' goog 3x', round(d['value']), d['ms_per_step'])"
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 300 python bench.py --global-batch 512 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' r18 b512 3x', round(d['value']), d['ms_per_step'])"
done; done
