#!/bin/bash
# r02ck: in-step knob sweep on the final tree (ResNet-18 b4096 3xTF32): promotion chunk, PDL, dW stream
D=gpurun_out/r02ck; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
run() { local tag="$1"; shift; env "$@" timeout 400 python bench.py $BARGS --no-cpu-baseline --no-e2e > $D/b.log 2>&1; echo "$tag $(tail -1 $D/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')"; }
for r in 1 2 3; do
BARGS="--steps 10 --warmup 3"
run "base" X=1
run "CHUNK=16" SMCONV_TMA_CHUNK=16
run "PDL=2" SMCONV_PDL=2
BARGS="--steps 10 --warmup 3 --dw-stream on"; run "dwstream" X=1
done
