#!/bin/bash
# r02bo: ncu of the thin-K calls after the coalesced epilogue: 1x1 s2 shortcut fwd (TF32, 3xTF32), GoogLeNet a3 1x1 dX
D=gpurun_out/r02bo; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
bash tools/prof.sh r02bo_scf resnet18 l2.0sc fwd 4096 tf32 regex:conv_tma
bash tools/prof.sh r02bo_scf3 resnet18 l2.0sc fwd 4096 3xtf32 regex:conv_tma
bash tools/prof.sh r02bo_g1 googlenet g.a3.1x1 dx 256 3xtf32 regex:conv_tma
ls gpurun_out/r02bo_*
