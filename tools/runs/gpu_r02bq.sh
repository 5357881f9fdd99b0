#!/bin/bash
# r02bq: TMA-store epilogue in the STRIP kernel: parity, coverage, A/B isolated + in-step
D=gpurun_out/r02bq; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_coverage_gpu.py tests/test_epi_gpu.py -q -x > $D/pytest_cov.log 2>&1; tail -2 $D/pytest_cov.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "strip" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for v in 0 1; do
SMCONV_TSTORE=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a --op fwd,dx --batch 4096 --math 3xtf32 > $D/lb3_$v.log 2>&1
SMCONV_TSTORE=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a,l2.1a --op fwd,dx --batch 4096 --math tf32 > $D/lbt_$v.log 2>&1
SMCONV_TSTORE=$v timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg2,vgg3,vgg4,vgg5 --op fwd,dx --batch 128 --math tf32 > $D/lbv_$v.log 2>&1
done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:9} {d['op']:3} {d['ms']*1000:8.1f} us {d['gbs']:6.0f} GB/s {d['tflops']:6.1f} TF  {d['plan'][:50]}")
P
done
for r in 1 2; do for v in 0 1; do SMCONV_TSTORE=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "TSTORE=$v $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; done; done
for v in 0 1; do SMCONV_TSTORE=$v timeout 300 python bench.py --net vgg16 --math tf32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $D/bv.log 2>&1; echo "VGG TSTORE=$v $(tail -1 $D/bv.log | cut -c150-200)"; done
