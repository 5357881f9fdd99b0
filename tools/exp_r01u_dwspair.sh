# r01u: retry CTA-pair DWS with the CTA-scope barrier waits (r01q's pair waits each ran CCTL.IVALL)
# parity + same-box A/B (head = SMCONV_DWS_PAIR=0)
D=gpurun_out/r01u_dwspair; mkdir -p $D
timeout 300 python -m pytest tests -m gpu -q -x --tb=short -k "dws" > $D/tests.log 2>&1; tail -3 $D/tests.log
grep -q "failed" $D/tests.log && exit 1
for v in 0 1; do SMCONV_DWS_PAIR=$v timeout 120 python tools/layer_bench.py --layer l1.0a --op dw 2>&1 | cut -c1-120; done
for v in 0 1; do SMCONV_DWS_PAIR=$v timeout 120 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg2 --op dw 2>&1 | cut -c1-120; done
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_DWS_PAIR=0; else export SMCONV_DWS_PAIR=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'],d['roofline']['frac'])")"
done
done
unset SMCONV_DWS_PAIR
