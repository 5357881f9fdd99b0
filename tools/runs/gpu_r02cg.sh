#!/bin/bash
# r02cg: stem dW 3xTF32 in TS form (dY^T in TMEM; SMCONV_STEM_TS=0: SS form): parity, isolated + in-step A/B
D=gpurun_out/r02cg; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_coverage_gpu.py tests/test_configs_gpu.py tests/test_fullsize_gpu.py -q -x -k "stem or conv1 or vgg1 or g.stem or alex1 or coverage" > $D/pytest.log 2>&1; echo "tests rc=$?"; tail -2 $D/pytest.log
grep -q " passed" $D/pytest.log && ! grep -q "failed" $D/pytest.log || exit 0
for v in 0 1; do SMCONV_STEM_TS=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer conv1 --op dw --batch 4096 --math 3xtf32 > $D/lb_$v.log 2>&1; SMCONV_STEM_TS=$v timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg1 --op dw --batch 128 --math 3xtf32 >> $D/lb_$v.log 2>&1; SMCONV_STEM_TS=$v timeout 300 python tools/layer_bench.py --net googlenet --layer g.stem --op dw --batch 256 --math 3xtf32 >> $D/lb_$v.log 2>&1; done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:9} {d['op']:3} {d['ms']*1000:8.1f} us {d['gbs']:6.0f} GB/s  {d['plan'][:60]}")
P
done
for r in 1 2; do for v in 0 1; do SMCONV_STEM_TS=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "STEM_TS=$v $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; done; done
