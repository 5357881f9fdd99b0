# r01s: CTA-pair TMA dW (3xTF32, OC % 256: two 128-channel OC blocks per M = 256 tile) — parity + A/B (head = SMCONV_DW_PAIR=0)
D=gpurun_out/r01s_dwpair; mkdir -p $D
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "tma" > $D/tests.log 2>&1; tail -3 $D/tests.log
grep -q "failed" $D/tests.log && exit 1
grep -q " passed" $D/tests.log || exit 1
for v in 0 1; do SMCONV_DW_PAIR=$v timeout 120 python tools/layer_bench.py --layer l3.0a,l3.1a,l4.0a,l4.1a,l3.0sc,l4.0sc --op dw 2>&1 | cut -c1-150; done
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "fullsize" > $D/tests_full.log 2>&1; tail -2 $D/tests_full.log
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_DW_PAIR=0; else export SMCONV_DW_PAIR=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
unset SMCONV_DW_PAIR
