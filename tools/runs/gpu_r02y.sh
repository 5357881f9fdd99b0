#!/bin/bash
# r02y: STEM variant (tensor-core stems): parity sweep + config parity at bench batch, stem call times, bench lines
D=gpurun_out/r02y; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "stem" > $D/pytest_stem.log 2>&1; tail -3 $D/pytest_stem.log
timeout 900 python -m pytest tests/test_configs_gpu.py -q -x > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for m in 3xtf32 tf32; do
  timeout 120 python tools/layer_bench.py --net resnet18 --layer conv1 --op fwd,dw --batch 4096 --math $m > $D/lb_conv1_$m.log 2>&1
  timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg1 --op fwd,dw --batch 128 --math $m > $D/lb_vgg1_$m.log 2>&1
  SMCONV_STEM=0 timeout 120 python tools/layer_bench.py --net resnet18 --layer conv1 --op fwd,dw --batch 4096 --math $m > $D/lb_conv1_old_$m.log 2>&1
done
timeout 120 python tools/layer_bench.py --net googlenet --layer g.stem --op fwd,dw --batch 256 --math 3xtf32 > $D/lb_goog.log 2>&1
cat $D/lb_*.log | cut -c1-200
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
