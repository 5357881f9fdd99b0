#!/bin/bash
# r02x: cluster split-K / no-split BN=128 for small-map TMA dW: parity at bench batch + VGG/ResNet lines
D=gpurun_out/r02x; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 900 python -m pytest tests/test_configs_gpu.py -q -x -k "vgg16 or alexnet or resnet18" > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for m in tf32 3xtf32; do
timeout 300 python bench.py --net vgg16 --math $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_$m.json > $D/b_vgg_$m.log 2>&1
done
timeout 300 python bench.py --net resnet18 --global-batch 512 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_r512_tf32.json > $D/b_r512_tf32.log 2>&1
timeout 300 python bench.py --net alexnet --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_alex.json > $D/b_alex.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-220; done
