#!/bin/bash
D=gpurun_out/r02r; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_mcast_gpu.py -q -rs > $D/mcast.log 2>&1; tail -5 $D/mcast.log
bash tools/gpu_sanitize.sh r02r/san > /dev/null 2>&1
cat $D/san/summary.txt
timeout 300 python bench.py --net resnet18@128 --steps 5 --warmup 3 --no-cpu-baseline --layers-out $D/l_r128.json > $D/b_r128.log 2>&1
timeout 300 python bench.py --net resnet18@224 --steps 5 --warmup 3 --no-cpu-baseline --layers-out $D/l_r224.json > $D/b_r224.log 2>&1
timeout 300 python bench.py --net resnet18@128 --math tf32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_r128t.json > $D/b_r128_tf32.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
