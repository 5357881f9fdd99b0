#!/bin/bash
# r02ae: small-map fwd/dX tile + cluster-split cost model (SMCONV_CSK_MODEL) A/B, parity at bench batch
D=gpurun_out/r02ae; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 900 python -m pytest tests/test_configs_gpu.py -q -x -k "vgg16 or alexnet" > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_epi_gpu.py -q -x -k "tma or csk or epi" > $D/pytest_tma.log 2>&1; tail -2 $D/pytest_tma.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for r in 1 2; do for c in 1 0; do for m in tf32 3xtf32; do
SMCONV_CSK_MODEL=$c timeout 300 python bench.py --net vgg16 --math $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_${m}_c$c.json > $D/b_vgg_${m}_c${c}_r$r.log 2>&1
done; done; done
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
SMCONV_CSK_MODEL=0 timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog0.json > $D/b_goog0.log 2>&1
for f in $D/b_*.log; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"); done
