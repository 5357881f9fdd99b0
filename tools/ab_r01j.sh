# r01j: same-box A/B of HEAD lib vs working tree lib (bench step + isolated l1 layers)
mkdir -p gpurun_out/r01j
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out gpurun_out/r01j/layers_${v}_$rep.json 2>/dev/null | tail -1 > gpurun_out/r01j/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('gpurun_out/r01j/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
for v in head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  timeout 300 python tools/layer_bench.py --layer l1.0a --op fwd,dx,dw --math 3xtf32 | cut -c1-80 | sed "s/^/$v /"
done
unset SMCONV_LIB
SMCONV_TMA_CHUNK=18 timeout 300 python tools/layer_bench.py --layer l1.0a --op fwd,dx,dw --math 3xtf32 | cut -c1-80 | sed "s/^/new-chunk18 /"
