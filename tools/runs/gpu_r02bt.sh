#!/bin/bash
# r02bt: same-box A/B of the CUDA-graph default for the 3xTF32 small-batch lines
D=gpurun_out/r02bt; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
for r in 1 2; do for gr in off on; do for n in "vgg16" "vgg16 --math tf32" "alexnet" "resnet18 --global-batch 512"; do timeout 300 python bench.py --net $n --graph $gr --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "$gr | $n | $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["config"]["dw_stream"])')"; done; done; done
for gr in off on; do SMCONV_PDL=2 timeout 300 python bench.py --net vgg16 --graph $gr --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "PDL2 $gr | vgg16 | $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; done
