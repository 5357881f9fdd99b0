#!/bin/bash
# ragged-channel TMA (fwd/dX/dW), bench without per-call events in the timed region, PDL A/B
D=gpurun_out/r02o; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_epi_gpu.py -q -x -k "googlenet or x20x36 or x48x112 or x24x16 or x112x208 or x144x48 or alexnet or epi" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for pdl in 1 0; do
SMCONV_PDL=$pdl timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32_pdl$pdl.json > $D/b_vgg_tf32_pdl$pdl.log 2>&1
SMCONV_PDL=$pdl timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x_pdl$pdl.json > $D/b_vgg_3x_pdl$pdl.log 2>&1
done
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph on --layers-out $D/l_vgg_tf32_g.json > $D/b_vgg_tf32_g.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
timeout 300 python bench.py --net alexnet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_alex.json > $D/b_alex.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
