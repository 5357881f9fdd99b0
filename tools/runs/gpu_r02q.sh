#!/bin/bash
D=gpurun_out/r02q; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_mcast_gpu.py -q -rs > $D/mcast.log 2>&1; tail -5 $D/mcast.log
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --fused-allreduce --layers-out $D/l_resnet_mc.json > $D/b_resnet_mc.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --epi --layers-out $D/l_resnet_epi.json > $D/b_resnet_epi.log 2>&1
bash tools/gpu_sanitize.sh r02q/san > /dev/null 2>&1
cat $D/san/summary.txt
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
