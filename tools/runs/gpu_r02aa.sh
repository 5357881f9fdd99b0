#!/bin/bash
# r02aa: s2dx zero-block skip (parity + A/B), ResNet b4096 / b512 with and without the dW stream,
# VGG TF32 launch list (kernel durations vs step), ncu full captures of the STEM kernels
D=gpurun_out/r02aa; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "s2dx or stem or epi" > $D/pytest_s2.log 2>&1; tail -2 $D/pytest_s2.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "l2.0a or conv1" > $D/pytest_full.log 2>&1; tail -2 $D/pytest_full.log
timeout 600 python -m pytest tests/test_epi_gpu.py -q -x > $D/pytest_epi.log 2>&1; tail -2 $D/pytest_epi.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
for k in 1 0; do for m in 3xtf32 tf32; do SMCONV_S2DX_SKIP=$k timeout 120 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math $m > $D/lb_s2_${k}_$m.log 2>&1; done; done
cat $D/lb_*.log | cut -c1-200
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dw-stream --layers-out $D/l_resnet_ds.json > $D/b_resnet_ds.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_r512.json > $D/b_r512.log 2>&1
timeout 300 python bench.py --global-batch 512 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dw-stream --layers-out $D/l_r512_ds.json > $D/b_r512_ds.log 2>&1
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-200; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/vgg_launches.csv python bench.py --net vgg16 --math tf32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_ncu.json > $D/vgg_ncu.log 2>&1
bash tools/prof.sh r02aa_stemfwd resnet18 conv1 fwd 4096 3xtf32 regex:stem_fwd
bash tools/prof.sh r02aa_stemdw resnet18 conv1 dw 4096 3xtf32 regex:stem_dw
mv gpurun_out/r02aa_stemfwd gpurun_out/r02aa_stemdw $D/
