#!/bin/bash
# r02ch: final matrix of the round (after the stem TS form): smoke, full GPU suite, bench lines, layer tables, launch list, ncu of the dominant kernel
D=gpurun_out/r02ch; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 400 python bench.py --math tf32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet_tf32.json > $D/b_resnet_tf32.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_r512.json > $D/b_r512.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
timeout 300 python bench.py --net alexnet --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_alex.json > $D/b_alex.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --epi > $D/b_resnet_epi.log 2>&1
for n in resnet18@64 resnet18@128 resnet18@224; do timeout 400 python bench.py --net $n --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $D/b_$n.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $D/b_reference.log 2>&1
for f in $D/b_*.log; do echo $f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])' 2>&1 | tail -1); done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu.log 2>&1; echo ncu rc=$?
bash tools/prof.sh r02ch_dws resnet18 l1.0a dw 4096 3xtf32 regex:dws
bash tools/gpu_tests.sh r02ch/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
