#!/bin/bash
# r02ba (session 4 re-entry): baseline of the committed tree: bench matrix + layer tables, launch list, full GPU suite
D=gpurun_out/r02ba; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 400 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 400 python bench.py --math tf32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet_tf32.json > $D/b_resnet_tf32.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-300; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu.log 2>&1; echo ncu rc=$?
bash tools/gpu_tests.sh r02ba/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
