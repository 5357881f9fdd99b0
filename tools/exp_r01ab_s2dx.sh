# r01ab: s2dx restricted to >= 16x16 dY maps (l2.0a only in ResNet-18) — full GPU suite + A/B (head = SMCONV_S2DX=0)
D=gpurun_out/r01ab; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q --tb=short > $D/tests_all.log 2>&1; tail -2 $D/tests_all.log
for rep in 1 2; do for v in 0 1; do
  echo "s2dx=$v rep $rep: $(SMCONV_S2DX=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${v}_$rep.json 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])")"
done; done
for v in 0 1; do echo "tf32 s2dx=$v: $(SMCONV_S2DX=$v timeout 300 python bench.py --math tf32 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'])")"; done
