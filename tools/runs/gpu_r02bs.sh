#!/bin/bash
# r02bs: TMA store for the super-pixel dX; CUDA graph by default below 1024 images/GPU
D=gpurun_out/r02bs; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python -m pytest tests/test_coverage_gpu.py tests/test_epi_gpu.py tests/test_s2dx_identity.py -q -x > $D/pytest_cov.log 2>&1; tail -2 $D/pytest_cov.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x -k "s2dx or l2.0a" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for v in 0 1; do SMCONV_TSTORE_S2DX=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math 3xtf32 > $D/lb_$v.log 2>&1; SMCONV_TSTORE_S2DX=$v timeout 300 python tools/layer_bench.py --net resnet18 --layer l2.0a --op dx --batch 4096 --math tf32 >> $D/lb_$v.log 2>&1; done
for f in $D/lb*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:9} {d['op']:3} {d['ms']*1000:8.1f} us {d['gbs']:6.0f} GB/s {d['tflops']:6.1f} TF  {d['plan'][:50]}")
P
done
for n in "vgg16 --math tf32" "vgg16" "resnet18 --global-batch 512" "googlenet" "alexnet"; do timeout 300 python bench.py --net $n --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "$n $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["config"]["cuda_graph"], d["roofline"]["frac"])')"; done
