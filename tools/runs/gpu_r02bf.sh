#!/bin/bash
# r02bf: epi_apply16 out of line (TMA kernels 11.2k -> 7.2k SASS instructions: cold I-cache of short calls)
D=gpurun_out/r02bf; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_epi_gpu.py tests/test_parity_gpu.py -q -x > $D/pytest.log 2>&1; tail -2 $D/pytest.log
timeout 300 python tools/layer_bench.py --net vgg16 --batch 128 --math tf32 > $D/lbv.log 2>&1
python - $D/lbv.log <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:50]}")
P
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --epi > $D/b_resnet_epi.log 2>&1
for f in $D/b_*.log; do echo $f $(tail -1 $f | cut -c150-250); done
bash tools/prof.sh r02bf_v11 vgg16 vgg11 fwd 128 tf32 regex:conv_tma
