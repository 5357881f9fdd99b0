#!/bin/bash
# r02ac: stem dW ring depth (parity + times), VGG 3xTF32 launch list, ncu full of vgg6 fwd vs dX (3xTF32)
D=gpurun_out/r02ac; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "stem" > $D/pytest_stem.log 2>&1; tail -2 $D/pytest_stem.log
for m in 3xtf32 tf32; do
  timeout 120 python tools/layer_bench.py --net resnet18 --layer conv1 --op dw --batch 4096 --math $m > $D/lb_conv1_$m.log 2>&1
  timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg1 --op dw --batch 128 --math $m > $D/lb_vgg1_$m.log 2>&1
done
timeout 120 python tools/layer_bench.py --net vgg16 --layer vgg6,vgg9 --op fwd,dx,dw --batch 128 --math 3xtf32 > $D/lb_vgg69_3x.log 2>&1
cat $D/lb_*.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/vgg3x_launches.csv python bench.py --net vgg16 --steps 2 --warmup 3 --dw-stream off --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_ncu.json > $D/vgg_ncu.log 2>&1
cap() {  # TAG LAYER OP
  timeout 600 ncu --set full --clock-control none --import-source on -s 2 -c 1 -k regex:conv_tma \
    -o $D/$1 python tools/layer_bench.py --net vgg16 --layer $2 --op $3 --batch 128 --math 3xtf32 --reps 1 > $D/$1.log 2>&1
  ncu -i $D/$1.ncu-rep --page raw --csv > $D/$1.raw.csv 2>/dev/null
  ncu -i $D/$1.ncu-rep --page source --csv --print-source sass > $D/$1.sass.csv 2>/dev/null
  rm -f $D/$1.ncu-rep
}
cap v6fwd3 vgg6 fwd
cap v6dx3 vgg6 dx
timeout 300 python bench.py --net vgg16 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
tail -1 $D/b_vgg_3x.log | cut -c1-250
