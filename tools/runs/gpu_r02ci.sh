#!/bin/bash
# r02ci: halved-BN cluster-split tiles for the smallest maps (SMCONV_CSK_BN64=1): parity, isolated + VGG step A/B
D=gpurun_out/r02ci; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_CSK_BN64=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_coverage_gpu.py tests/test_configs_gpu.py tests/test_epi_gpu.py -q -x -k "csk or vgg or coverage or epi" > $D/pytest.log 2>&1; echo "tests rc=$?"; tail -2 $D/pytest.log
grep -q " passed" $D/pytest.log && ! grep -q "failed" $D/pytest.log || exit 0
for v in 0 1; do for m in tf32 3xtf32; do SMCONV_CSK_BN64=$v timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg5,vgg8,vgg9,vgg11,vgg12 --op fwd,dx --batch 128 --math $m > $D/lb_${m}_$v.log 2>&1; done; done
for m in tf32 3xtf32; do paste <(python - $D/lb_${m}_0.log <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"{d['layer']:7} {d['op']:3} {d['ms']*1000:8.1f}")
P
) <(python - $D/lb_${m}_1.log <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"{d['ms']*1000:8.1f}  {d['plan'][:40]}")
P
); done
for r in 1 2; do for v in 0 1; do for m in tf32 3xtf32; do SMCONV_CSK_BN64=$v timeout 300 python bench.py --net vgg16 --math $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "CSK_BN64=$v $m $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; done; done; done
