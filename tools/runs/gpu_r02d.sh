#!/bin/bash
# small-map VGG b128 layers: isolated timing (csk on/off) and ncu full captures of vgg11 / vgg6 fwd TF32
D=gpurun_out/r02d; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for csk in 8 0; do
  SMCONV_CSK=$csk timeout 300 python tools/layer_bench.py --net vgg16 --layer vgg5,vgg6,vgg8,vgg9,vgg11 --op fwd,dx,dw --batch 128 --math tf32 --reps 50 > $D/lb_tf32_csk$csk.log 2>&1
done
bash tools/prof.sh r02d_v11 vgg16 vgg11 fwd 128 tf32
bash tools/prof.sh r02d_v6 vgg16 vgg6 fwd 128 tf32
mv gpurun_out/r02d_v11 gpurun_out/r02d_v6 $D/
