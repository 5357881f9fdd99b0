#!/bin/bash
# r02ab: wide split-K reduce, dW stream default: full GPU suite + bench matrix + VGG launch list
D=gpurun_out/r02ab; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python tools/layer_bench.py --net vgg16 --layer vgg1,vgg2 --op dw --batch 128 --math tf32 > $D/lb_vgg_dw.log 2>&1
timeout 600 python tools/layer_bench.py --net resnet18 --layer conv1,l2.0sc --op dw --batch 4096 --math 3xtf32 > $D/lb_r_dw.log 2>&1
cat $D/lb_*.log | cut -c1-200
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 400 python bench.py --math tf32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet_tf32.json > $D/b_resnet_tf32.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_r512.json > $D/b_r512.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
timeout 300 python bench.py --net alexnet --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_alex.json > $D/b_alex.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
bash tools/gpu_tests.sh r02ab/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
