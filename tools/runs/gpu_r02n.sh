#!/bin/bash
# PDL + fast-division prologue + push csk: correctness (all GPU tests) and VGG / ResNet timing (PDL on / off)
D=gpurun_out/r02n; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python tools/trace_probe.py tiny,vgg11,vgg6,vgg9 > $D/trace.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
SMCONV_PDL=0 timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32_nopdl.json > $D/b_vgg_tf32_nopdl.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph on --layers-out $D/l_vgg_tf32_g.json > $D/b_vgg_tf32_g.log 2>&1
timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
