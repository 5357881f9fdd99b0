# r01ae: promotion chunk 8 vs 16 k-blocks for all 3xTF32 kernels (SMCONV_TMA_CHUNK) — step A/B + full-size parity at 16
D=gpurun_out/r01ae; mkdir -p $D
for rep in 1 2; do for c in 8 16; do
  echo "chunk=$c rep $rep: $(SMCONV_TMA_CHUNK=$c timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out $D/layers_${c}_$rep.json 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])")"
done; done
SMCONV_TMA_CHUNK=16 timeout 900 python -m pytest tests -m gpu -q --tb=short -k "fullsize or random" > $D/tests16.log 2>&1; tail -2 $D/tests16.log
