# r01z: stem dW heuristic — DIRECT vs GENERIC by (n, oh) row count (SMCONV_DIRECT_DW_MIN_ROWS: 0 = always DIRECT, 1e9 = always GENERIC)
timeout 300 python -m pytest tests -m gpu -q -x --tb=short -k "direct or generic or smoke" 2>&1 | tail -2
for m in 0 1000000000; do
  echo "min_rows=$m"
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 60 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg1 --op dw 2>&1 | tail -1 | cut -c1-90
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 60 python tools/layer_bench.py --net googlenet --batch 256 --layer g.stem --op dw 2>&1 | tail -1 | cut -c1-90
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 60 python tools/layer_bench.py --batch 512 --layer conv1 --op dw 2>&1 | tail -1 | cut -c1-90
  SMCONV_DIRECT_DW_MIN_ROWS=$m timeout 60 python tools/layer_bench.py --batch 1024 --layer conv1 --op dw 2>&1 | tail -1 | cut -c1-90
done
for v in 0 8192 0 8192; do echo "vgg b128 tf32 min_rows=$v: $(SMCONV_DIRECT_DW_MIN_ROWS=$v timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'][:30])")"; done
