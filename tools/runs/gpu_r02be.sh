#!/bin/bash
# r02be: small-map call anatomy (per-CTA trace, csk sweep) + ncu of the stage-1 STRIP and l2 TMA pair fwd
D=gpurun_out/r02be; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 300 python tools/trace_probe.py vgg11,vgg9,vgg6 > $D/trace.log 2>&1; cut -c1-400 $D/trace.log
for k in 0 2 4 8 16; do SMCONV_CSK=$k timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg5,vgg8,vgg9,vgg11 --op fwd,dx --batch 128 --math tf32 > $D/lbv_k$k.log 2>&1; done
for f in $D/lbv_k*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:70]}")
P
done
bash tools/prof.sh r02be_l1f resnet18 l1.0a fwd 4096 3xtf32 regex:strip
bash tools/prof.sh r02be_l2f resnet18 l2.1a fwd 4096 3xtf32 regex:conv_tma
bash tools/prof.sh r02be_v11 vgg16 vgg11 fwd 128 tf32 regex:conv_tma
ls gpurun_out/r02be_*
