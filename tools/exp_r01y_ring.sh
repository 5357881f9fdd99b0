# r01y: DIRECT dW cp.async ring 4 -> 8 rows (head = ab/libsmconv_head.so)
timeout 300 python -m pytest tests -m gpu -q -x --tb=short -k "direct" 2>&1 | tail -2
for v in head new head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  echo "$v $(timeout 60 python tools/layer_bench.py --layer conv1 --op dw 2>&1 | tail -1 | cut -c1-60) | $(timeout 60 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg1 --op dw 2>&1 | tail -1 | cut -c1-60)"
done
unset SMCONV_LIB
timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
