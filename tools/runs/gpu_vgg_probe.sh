#!/bin/bash
# VGG-16 b128: eager vs CUDA-graph step, and the serialised kernel launch list (ncu) of the same step
D=gpurun_out/${1:-r02c}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for m in tf32 3xtf32; do
  timeout 300 python bench.py --net vgg16 --math $m --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --graph off --layers-out $D/l_vgg_${m}_eager.json > $D/b_vgg_${m}_eager.log 2>&1
  timeout 300 python bench.py --net vgg16 --math $m --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --graph on --layers-out $D/l_vgg_${m}_graph.json > $D/b_vgg_${m}_graph.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/vgg_${m}_launches.csv python bench.py --net vgg16 --math $m --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_vgg_$m.log 2>&1
done
for f in $D/b_vgg_*.log; do echo $f; tail -1 $f | cut -c1-200; done
