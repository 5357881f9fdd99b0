#!/bin/bash
# r02bl: 3xTF32 TMA dW with bf16 cross terms (SMCONV_DW_HYB=1): parity, isolated and in-step A/B
D=gpurun_out/r02bl; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_DW_HYB=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "tma or pair" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
SMCONV_DW_HYB=1 timeout 900 python -m pytest tests/test_configs_gpu.py -q -x -k "resnet18 and l3" > $D/pytest_cfg.log 2>&1; tail -2 $D/pytest_cfg.log
for v in 0 1; do SMCONV_DW_HYB=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.1a,l3.1a,l4.1a,l2.0a,l2.0sc --op dw --batch 4096 --math 3xtf32 > $D/lb_$v.log 2>&1; done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f} us {d['tflops']:6.1f} TF  {d['plan'][:60]}")
P
done
for r in 1 2 3; do for v in 0 1; do SMCONV_DW_HYB=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "DW_HYB=$v $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; done; done
grep -h "3xtf32" gpurun_out/parity_errors.json > /dev/null 2>&1; cp gpurun_out/parity_errors.json $D/ 2>/dev/null
