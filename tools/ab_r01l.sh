# r01l: TMA kernel 3xTF32 cross terms in bf16 (a_hi*b_hi TF32 + [a_hi|a_lo].[b_lo|b] bf16): parity, same-box A/B
mkdir -p gpurun_out/r01l
timeout 900 python -m pytest tests -m gpu -q -x --tb=short > gpurun_out/r01l/tests.log 2>&1; tail -15 gpurun_out/r01l/tests.log
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out gpurun_out/r01l/layers_${v}_$rep.json 2>/dev/null | tail -1 > gpurun_out/r01l/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('gpurun_out/r01l/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
unset SMCONV_LIB
timeout 300 python tools/layer_bench.py --layer l1.0a,l2.0b,l3.0b --math 3xtf32 | cut -c1-100
