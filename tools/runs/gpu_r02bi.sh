#!/bin/bash
# r02bi: STRIP converters issue the next window's loads before tcgen05.wait::st; no proxy fence where
# the converters write TMEM only (hybrid fwd / dX)
D=gpurun_out/r02bi; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "strip or tma" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a,l2.1a,l3.1a --op fwd,dx --batch 4096 --math 3xtf32 > $D/lb3.log 2>&1
timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg2,vgg4,vgg6,vgg9 --op fwd,dx --batch 128 --math 3xtf32 > $D/lbv3.log 2>&1
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:60]}")
P
done
for r in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b_resnet_$r.log 2>&1; echo $(tail -1 $D/b_resnet_$r.log | cut -c150-250); done
