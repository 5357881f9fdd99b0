#!/bin/bash
# r02ad: 3-MMA form for small 3xTF32 TMA fwd/dX (no wx_prep), PDL waits moved into the TMA kernel's roles
D=gpurun_out/r02ad; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "tma or s2dx or csk or variants or deterministic" > $D/pytest_tma.log 2>&1; tail -2 $D/pytest_tma.log
timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_epi_gpu.py -q -x > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for h in 12 0 30; do
SMCONV_HYB_MIN_GFLOP=$h timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x_h$h.json > $D/b_vgg_3x_h$h.log 2>&1
done
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
SMCONV_PDL=0 timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32_nopdl.json > $D/b_vgg_tf32_nopdl.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_r512.json > $D/b_r512.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
