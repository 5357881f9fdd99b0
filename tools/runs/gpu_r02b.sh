#!/bin/bash
# r02b: GPU tests (all), then VGG b128 TF32 bench (eager + graph), ResNet headline bench
D=gpurun_out/r02b; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 1800 python -m pytest tests -m gpu -q > $D/pytest.log 2>&1; echo "pytest rc=$?" >> $D/pytest.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
tail -5 $D/pytest.log
