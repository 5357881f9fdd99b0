#!/bin/bash
# r02z: STEM fix (OC 192 accumulators / slots), stem dW gather prefetch; config parity; DWS rounds knob; dW stream A/B
D=gpurun_out/r02z; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "stem" > $D/pytest_stem.log 2>&1; tail -2 $D/pytest_stem.log
timeout 900 python -m pytest tests/test_configs_gpu.py -q -x > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for m in 3xtf32 tf32; do
  timeout 120 python tools/layer_bench.py --net resnet18 --layer conv1 --op fwd,dw --batch 4096 --math $m > $D/lb_conv1_$m.log 2>&1
  timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg1 --op fwd,dw --batch 128 --math $m > $D/lb_vgg1_$m.log 2>&1
done
timeout 120 python tools/layer_bench.py --net googlenet --layer g.stem --op fwd,dw --batch 256 --math 3xtf32 > $D/lb_goog.log 2>&1
for r in 4 2 1; do SMCONV_DWS_MIN_ROUNDS=$r timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg2 --op dw --batch 128 --math tf32 > $D/lb_dws_r$r.log 2>&1; done
SMCONV_FORCE_VARIANT=2:2 timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg2 --op dw --batch 128 --math tf32 > $D/lb_dws_tma.log 2>&1
cat $D/lb_*.log | cut -c1-220
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --dw-stream --layers-out $D/l_vgg_tf32_ds.json > $D/b_vgg_tf32_ds.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --dw-stream --layers-out $D/l_vgg_3x_ds.json > $D/b_vgg_3x_ds.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
