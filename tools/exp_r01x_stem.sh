# r01x: stem dW (DIRECT) block-count sweep and the GENERIC tensor-core variant, ResNet b4096 and VGG b128
for cfg in "32 444" "16 444" "8 444" "32 888" "16 888" "8 1184" "4 1184"; do
  set -- $cfg
  echo "rows>=$1 blocks<=$2: $(SMCONV_DIRECT_DW_ROWS=$1 SMCONV_DIRECT_DW_BLOCKS=$2 timeout 60 python tools/layer_bench.py --layer conv1 --op dw 2>&1 | tail -1 | cut -c1-110) | $(SMCONV_DIRECT_DW_ROWS=$1 SMCONV_DIRECT_DW_BLOCKS=$2 timeout 60 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg1 --op dw 2>&1 | tail -1 | cut -c1-110)"
done
timeout 60 python tools/layer_bench.py --layer conv1 --op dw,fwd --variant 1 2>&1 | cut -c1-130
timeout 60 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg1 --op dw,fwd --variant 1 2>&1 | cut -c1-130
