#!/bin/bash
# r02w: ncu full captures (warm: 3rd launch) of the VGG b128 small-map TF32 calls: where the fixed cost goes
D=gpurun_out/r02w; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
cap() {  # TAG LAYER OP
  timeout 600 ncu --set full --clock-control none --import-source on -s 2 -c 1 -k regex:conv_tma \
    -o $D/$1 python tools/layer_bench.py --net vgg16 --layer $2 --op $3 --batch 128 --math tf32 --reps 1 > $D/$1.log 2>&1
  ncu -i $D/$1.ncu-rep --page raw --csv > $D/$1.raw.csv 2>/dev/null
  ncu -i $D/$1.ncu-rep --page source --csv --print-source sass > $D/$1.sass.csv 2>/dev/null
  ncu -i $D/$1.ncu-rep --page details --csv > $D/$1.details.csv 2>/dev/null
  rm -f $D/$1.ncu-rep
}
cap v9fwd vgg9 fwd
cap v11fwd vgg11 fwd
cap v6fwd vgg6 fwd
