#!/bin/bash
# r02bb: ncu full captures of the 1x1 s2 shortcut fwd / dX and the stem dW (HBM-bound calls below 0.5 of HBM)
D=gpurun_out/r02bb; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0sc,l3.0sc,l4.0sc,conv1 --batch 4096 --math 3xtf32 > $D/lb.log 2>&1
cat $D/lb.log | cut -c1-220
bash tools/prof.sh r02bb_scf resnet18 l2.0sc fwd 4096 tf32
bash tools/prof.sh r02bb_scd resnet18 l2.0sc dx 4096 tf32
bash tools/prof.sh r02bb_scd0 resnet18 l2.0sc dx 4096 tf32 regex:zero
bash tools/prof.sh r02bb_c1w resnet18 conv1 dw 4096 3xtf32 regex:stem
ls -la gpurun_out/r02bb*
