#!/bin/bash
# r02a: GPU tests (all), then VGG b128 TF32 bench + launch list
set -x
D=gpurun_out/r02a; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest.log 2>&1; echo "pytest rc=$?" >> $D/pytest.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --graph on --layers-out $D/l_vgg_tf32g.json > $D/b_vgg_tf32g.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $D/vgg_tf32_launches.csv python bench.py --net vgg16 --math tf32 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $D/ncu_vgg.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
