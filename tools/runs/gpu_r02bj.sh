#!/bin/bash
# r02bj: 3xTF32 dX with the K-major transposed filter (Wt) + DWS dW with bf16 cross terms (SMCONV_DWS_HYB): parity,
# isolated A/B and IN-STEP A/B (the step runs at the power cap: energy per step, not latency, sets its time)
D=gpurun_out/r02bj; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "tma or dws" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
SMCONV_DWS_HYB=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "dws" > $D/pytest_dwshyb.log 2>&1; tail -2 $D/pytest_dwshyb.log
for v in 0 1; do
SMCONV_DX_BK=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.1a,l3.1a,l4.1a,l3.0a --op dx --batch 4096 --math 3xtf32 > $D/lbdx_$v.log 2>&1
SMCONV_DWS_HYB=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a --op dw --batch 4096 --math 3xtf32 > $D/lbdws_$v.log 2>&1
done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:60]}")
P
done
for r in 1 2; do
for cfg in "SMCONV_DX_BK=0 SMCONV_DWS_HYB=0" "SMCONV_DX_BK=1 SMCONV_DWS_HYB=0" "SMCONV_DX_BK=1 SMCONV_DWS_HYB=1"; do
env $cfg timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "$cfg $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done
SMCONV_DWS_HYB=1 timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "l1" > $D/pytest_full.log 2>&1; tail -2 $D/pytest_full.log
