#!/bin/bash
# r02bc: row-coalesced fwd / dX epilogue (TmaCfg::EPW) + TMEM released before the TF32 stores: parity, A/B
D=gpurun_out/r02bc; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_epi_gpu.py -q -x > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for c in 0 1; do
SMCONV_COALESCE=$c timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0sc,l3.0sc,l4.0sc,l2.0a,l2.1a,l3.1a,l4.1a --op fwd,dx --batch 4096 --math 3xtf32 > $D/lb3_c$c.log 2>&1
SMCONV_COALESCE=$c timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0sc,l3.0sc,l4.0sc,l2.0a,l2.1a,l3.1a,l4.1a --op fwd,dx --batch 4096 --math tf32 > $D/lbt_c$c.log 2>&1
SMCONV_COALESCE=$c timeout 300 python tools/layer_bench.py --net vgg16 --op fwd,dx --batch 128 --math tf32 > $D/lbv_c$c.log 2>&1
done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['gbs']:7.0f} GB/s {d['tflops']:6.1f} TF")
P
done
for c in 1 0; do SMCONV_COALESCE=$c timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b_resnet_c$c.log 2>&1; tail -1 $D/b_resnet_c$c.log | cut -c1-250; done
