#!/bin/bash
# pull-batched csk reduce + pipelined TF32 epilogue: full GPU tests, VGG/ResNet/GoogLeNet benches, PDL A/B x2
D=gpurun_out/r02p; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python tools/trace_probe.py tiny,vgg11,vgg6,vgg9 > $D/trace.log 2>&1
for rep in 1 2; do for pdl in 1 0; do
SMCONV_PDL=$pdl timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32_pdl$pdl.json > $D/b_vgg_tf32_pdl${pdl}_$rep.log 2>&1
SMCONV_PDL=$pdl timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x_pdl$pdl.json > $D/b_vgg_3x_pdl${pdl}_$rep.log 2>&1
done; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
SMCONV_PDL=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet0.json > $D/b_resnet_pdl0.log 2>&1
timeout 300 python bench.py --net googlenet --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_goog.json > $D/b_goog.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $D/pytest.log 2>&1; tail -2 $D/pytest.log
cp gpurun_out/parity_errors.json $D/
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
