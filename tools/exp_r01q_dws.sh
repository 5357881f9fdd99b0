# r01q: CTA-pair DWS (3xTF32: both m-tiles of an item as one M = 256 tile): parity + same-box A/B (head = pairs off)
D=gpurun_out/r01q_dws; mkdir -p $D
timeout 300 python -m pytest tests -m gpu -q -x --tb=short -k "dws" > $D/tests.log 2>&1; tail -3 $D/tests.log
grep -q " passed" $D/tests.log || exit 1
grep -q "failed" $D/tests.log && exit 1
for v in 0 1; do SMCONV_PAIR=$v timeout 120 python tools/layer_bench.py --layer l1.0a --op dw 2>&1 | cut -c1-150; done
for v in 0 1; do SMCONV_PAIR=$v timeout 120 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg2 --op dw 2>&1 | cut -c1-150; done
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "fullsize" > $D/tests_full.log 2>&1; tail -3 $D/tests_full.log
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_PAIR=0; else export SMCONV_PAIR=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'],d['roofline']['frac'])")"
done
done
unset SMCONV_PAIR
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_dws' -o $D/l1dw_pair python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > $D/full.log 2>&1
