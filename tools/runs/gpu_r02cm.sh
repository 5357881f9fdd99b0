#!/bin/bash
# r02cm: super-pixel dX with one phase per n-tile (SMCONV_S2DX_BN=64): parity, isolated + in-step A/B
D=gpurun_out/r02cm; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_S2DX_BN=64 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_coverage_gpu.py tests/test_epi_gpu.py tests/test_fullsize_gpu.py tests/test_configs_gpu.py -q -x -k "s2dx or coverage or epi or l2.0a" > $D/pytest.log 2>&1; echo "tests rc=$?"; tail -2 $D/pytest.log
grep -q " passed" $D/pytest.log && ! grep -q "failed" $D/pytest.log || exit 0
for v in 0 64; do SMCONV_S2DX_BN=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math 3xtf32 > $D/lb_$v.log 2>&1; SMCONV_S2DX_BN=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math tf32 >> $D/lb_$v.log 2>&1; done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:9} {d['op']:3} {d['ms']*1000:8.1f} us  {d['plan'][:60]}")
P
done
for v in 0 64; do SMCONV_S2DX_BN=$v timeout 300 python tools/power_probe.py --layer l2.0a --op dx --math 3xtf32 > $D/p_$v.log 2>&1; tail -1 $D/p_$v.log | cut -c1-160; done
for r in 1 2 3; do for v in 0 64; do SMCONV_S2DX_BN=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "S2DX_BN=$v $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; done; done
