#!/bin/bash
D=gpurun_out/r02u; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
bash tools/prof.sh r02u_s128 resnet18@128 l1.0a fwd 256 3xtf32 regex:conv_strip
bash tools/prof.sh r02u_s32 resnet18 l1.0a fwd 4096 3xtf32 regex:conv_strip
mv gpurun_out/r02u_s128 gpurun_out/r02u_s32 $D/
python tools/trace_probe.py tiny,vgg11,vgg6,vgg9 > $D/trace.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > $D/pytest.log 2>&1; tail -2 $D/pytest.log
