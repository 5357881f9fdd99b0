#!/bin/bash
# r02br: in-step knob sweep on the current tree (ResNet-18 b4096 3xTF32; VGG-16 b128): PDL, dW stream, graph, promotion chunk
D=gpurun_out/r02br; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
run() { local tag="$1"; shift; env "$@" timeout 400 python bench.py $BARGS --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "$tag $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; }
for r in 1 2; do
BARGS="--steps 10 --warmup 3"
run "base" X=1
run "PDL=2" SMCONV_PDL=2
run "CHUNK=16" SMCONV_TMA_CHUNK=16
BARGS="--steps 10 --warmup 3 --dw-stream on"; run "dwstream" X=1
BARGS="--steps 10 --warmup 3 --graph on"; run "graph" X=1
done
for r in 1 2; do
BARGS="--net vgg16 --math tf32 --steps 30 --warmup 5"; run "vgg-tf32 base" X=1; run "vgg-tf32 PDL=0" SMCONV_PDL=0; BARGS="--net vgg16 --math tf32 --steps 30 --warmup 5 --graph on"; run "vgg-tf32 graph" X=1
BARGS="--net vgg16 --steps 30 --warmup 5"; run "vgg-3x base" X=1; run "vgg-3x PDL=2" SMCONV_PDL=2
done
