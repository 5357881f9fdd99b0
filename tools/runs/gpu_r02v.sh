#!/bin/bash
# r02v: HEAD baseline after session restart: trace probe, VGG/ResNet bench lines with layer tables, full GPU tests
D=gpurun_out/r02v; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/trace_probe.py tiny,vgg11,vgg6,vgg9 > $D/trace.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
bash tools/gpu_tests.sh r02v/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
