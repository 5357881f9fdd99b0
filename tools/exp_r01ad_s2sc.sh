# r01ad: super-pixel dX for the 1x1 stride-2 shortcut (>= 16x16 dY: l2.0sc) — s2dx parity, full suite, A/B (head = SMCONV_S2DX=0)
D=gpurun_out/r01ad; mkdir -p $D
timeout 300 python -m pytest tests -m gpu -q -x --tb=short -k "s2dx" > $D/tests.log 2>&1; tail -2 $D/tests.log
grep -q "failed\|error" $D/tests.log && exit 1
for v in 0 1; do SMCONV_S2DX=$v timeout 120 python tools/layer_bench.py --layer l2.0sc,l2.0a --op dx 2>&1 | cut -c1-120; done
timeout 900 python -m pytest tests -m gpu -q --tb=short > $D/tests_all.log 2>&1; tail -2 $D/tests_all.log
for rep in 1 2; do for v in 0 1; do
  echo "s2dx=$v rep $rep: $(SMCONV_S2DX=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])")"
done; done
