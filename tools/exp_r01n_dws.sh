# r01n: DWS dW with TF32 + bf16 cross terms (HYB) vs the three-TF32-MMA form.  head = SMCONV_DWS_HYB=0.
D=gpurun_out/r01n_dws; mkdir -p $D
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "dws or fullsize or smoke" > $D/tests.log 2>&1; tail -3 $D/tests.log
for v in head new; do
  if [ $v = head ]; then export SMCONV_DWS_HYB=0; else export SMCONV_DWS_HYB=1; fi
  timeout 120 python tools/layer_bench.py --layer l1.0a --op dw --math 3xtf32 2>&1 | cut -c1-160
  timeout 120 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg2 --op dw --math 3xtf32 2>&1 | cut -c1-160
done
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_DWS_HYB=0; else export SMCONV_DWS_HYB=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'],d['roofline']['frac'])")"
done
done
unset SMCONV_DWS_HYB
