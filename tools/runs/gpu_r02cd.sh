#!/bin/bash
# r02cd: STRIP converters in two groups on alternate stages (SMCONV_STRIP_ALT=1): parity, isolated + in-step A/B
D=gpurun_out/r02cd; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_STRIP_ALT=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_coverage_gpu.py tests/test_epi_gpu.py -q -x -k "strip or coverage or epi" > $D/pytest.log 2>&1; echo "tests rc=$?"; tail -2 $D/pytest.log
grep -q " passed" $D/pytest.log && ! grep -q "failed" $D/pytest.log || exit 0
SMCONV_STRIP_ALT=1 timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_fullsize_gpu.py -q -x -k "resnet18 or vgg2 or l1" > $D/pytest2.log 2>&1; echo "tests2 rc=$?"; tail -2 $D/pytest2.log
for v in 0 1; do SMCONV_STRIP_ALT=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a --op fwd,dx --batch 4096 --math 3xtf32 > $D/lb_$v.log 2>&1; SMCONV_STRIP_ALT=$v timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg2 --op fwd,dx --batch 128 --math 3xtf32 >> $D/lb_$v.log 2>&1; done
paste <(python - $D/lb_0.log <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"{d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f}")
P
) <(python - $D/lb_1.log <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"{d['ms']*1000:8.1f}")
P
)
for r in 1 2 3; do for v in 0 1; do SMCONV_STRIP_ALT=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "STRIP_ALT=$v $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; done; done
