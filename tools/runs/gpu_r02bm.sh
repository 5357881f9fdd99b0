#!/bin/bash
# r02bm: hybrid TMA dW on by default: full GPU suite, bench lines (ResNet 3xTF32 x2, VGG 3xTF32, GoogLeNet, b512)
D=gpurun_out/r02bm; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
for r in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet.json > $D/b_resnet_$r.log 2>&1; done
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b_goog.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $D/b_r512.log 2>&1
for f in $D/b_*.log; do echo $f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["clocks"]["sm_mhz"])'); done
bash tools/gpu_tests.sh r02bm/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
