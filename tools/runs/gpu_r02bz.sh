#!/bin/bash
# r02bz: ncu of the DWS pair kernel vs the one-CTA DWS (why the pair's MMA rate is lower)
D=gpurun_out/r02bz; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_DWS_PAIR=1 bash tools/prof.sh r02bz_pair resnet18 l1.0a dw 4096 tf32 regex:dws
bash tools/prof.sh r02bz_one resnet18 l1.0a dw 4096 tf32 regex:dws
ls gpurun_out/r02bz_*
