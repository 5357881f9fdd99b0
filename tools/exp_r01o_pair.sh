# r01o: CTA pairs after the remote-arrival fix (no MEMBAR.ALL.GPU): parity + same-box A/B (head = pairs off)
D=gpurun_out/r01o_pair; mkdir -p $D
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "pair" > $D/tests.log 2>&1; tail -3 $D/tests.log
for v in 0 1 2; do SMCONV_PAIR=$v timeout 120 python tools/layer_bench.py --layer l2.1a,l3.1a,l4.1a --op fwd,dx 2>&1 | cut -c1-150; done
for rep in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMCONV_PAIR=0; else export SMCONV_PAIR=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 > $D/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('$D/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
unset SMCONV_PAIR
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
SMCONV_PAIR=1 $NCU -k 'regex:conv_tma_kernel' -o $D/l31fwd_pair python tools/layer_bench.py --layer l3.1a --op fwd --reps 1 > $D/full.log 2>&1
