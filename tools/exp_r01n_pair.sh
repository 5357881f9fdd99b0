# r01n: re-measure CTA pairs (cta_group::2) in the TMA fwd/dX kernel now that the TMEM A-slot ring
# is decoupled from the smem ring and 3xTF32 runs as TF32 + bf16 cross terms.  head = pairs off.
mkdir -p gpurun_out/r01n_pair
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "pair" > gpurun_out/r01n_pair/tests.log 2>&1; tail -3 gpurun_out/r01n_pair/tests.log
for rep in 1 2; do
for v in head new new2; do
  case $v in head) export SMCONV_PAIR=0;; new) export SMCONV_PAIR=1;; new2) export SMCONV_PAIR=2;; esac
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --layers-out gpurun_out/r01n_pair/layers_${v}_$rep.json 2>/dev/null | tail -1 > gpurun_out/r01n_pair/bench_${v}_$rep.json
  echo "$v $rep $(python -c "import json;d=json.load(open('gpurun_out/r01n_pair/bench_${v}_$rep.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])")"
done
done
unset SMCONV_PAIR
