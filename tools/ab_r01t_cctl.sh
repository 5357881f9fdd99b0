# r01t: pair-kernel barrier waits without .acquire.cluster (no CCTL.IVALL per wait): parity + same-box A/B
# head = ab/libsmconv_head.so (same code with the cluster-scope acquire), new = in-tree lib
D=gpurun_out/r01t_cctl; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x --tb=short -k "pair or strip or tma or fullsize or smoke" > $D/tests.log 2>&1; tail -3 $D/tests.log
grep -q "failed" $D/tests.log && exit 1
for v in head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  timeout 120 python tools/layer_bench.py --layer l1.0a,l2.0a,l2.1a,l3.1a,l4.1a --op fwd,dx 2>&1 | cut -c1-110
done
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_LIB=$PWD/ab/libsmconv_head.so; else unset SMCONV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
unset SMCONV_LIB
