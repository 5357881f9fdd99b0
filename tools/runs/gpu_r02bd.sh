#!/bin/bash
# r02bd: coalesced STRIP epilogue + in-epilogue zero fill of the 1x1 s2 dX: parity, A/B, bench
D=gpurun_out/r02bd; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_epi_gpu.py tests/test_configs_gpu.py tests/test_fullsize_gpu.py -q -x > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for c in 0 1; do
SMCONV_COALESCE=$c SMCONV_ZFILL=$c timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a,l2.0sc,l3.0sc,l4.0sc --op fwd,dx --batch 4096 --math 3xtf32 > $D/lb3_c$c.log 2>&1
SMCONV_COALESCE=$c SMCONV_ZFILL=$c timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a,l2.0sc,l3.0sc,l4.0sc --op fwd,dx --batch 4096 --math tf32 > $D/lbt_c$c.log 2>&1
done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['gbs']:7.0f} GB/s {d['tflops']:6.1f} TF  {d['plan'][:40]}")
P
done
for r in 1 2; do for c in 1 0; do SMCONV_COALESCE=$c SMCONV_ZFILL=$c timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b_resnet_c${c}_$r.log 2>&1; echo c$c $(tail -1 $D/b_resnet_c${c}_$r.log | cut -c150-250); done; done
timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --math tf32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet_tf32.json > $D/b_resnet_tf32.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --layers-out $D/l_resnet.json > $D/b_resnet.log 2>&1
for f in $D/b_vgg_tf32.log $D/b_resnet_tf32.log $D/b_resnet.log; do echo $f $(tail -1 $f | cut -c150-250); done
