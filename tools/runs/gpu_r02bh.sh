#!/bin/bash
# r02bh: every-element-written test (NaN-poisoned outputs), relaxed csk exit barrier, s2dx A/B after 6d
D=gpurun_out/r02bh; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_coverage_gpu.py -q -x > $D/pytest_cov.log 2>&1; tail -3 $D/pytest_cov.log
timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg8,vgg9,vgg11 --op fwd,dx --batch 128 --math tf32 > $D/lbv.log 2>&1
for s in 1 0; do SMCONV_S2DX=$s timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math 3xtf32 > $D/lb_s2dx$s.log 2>&1; SMCONV_S2DX=$s timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math tf32 >> $D/lb_s2dx$s.log 2>&1; done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:60]}")
P
done
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $D/b_vgg_tf32.log 2>&1
for f in $D/b_*.log; do echo $f $(tail -1 $f | cut -c150-250); done
