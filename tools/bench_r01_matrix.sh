# r01 bench matrix (1 GPU): default line (+ layers) + TF32 + VGG-16 b128 + ResNet-18 b512 + GoogLeNet b256, and the reference arm
D=gpurun_out/r01_matrix2; mkdir -p $D
python bench.py --layers-out $D/l_3x.json > $D/resnet18_b4096_3x.json 2> $D/err.log
python bench.py --math tf32 --no-cpu-baseline --layers-out $D/l_tf32.json > $D/resnet18_b4096_tf32.json 2>> $D/err.log
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg.json > $D/vgg16_b128_3x.json 2>> $D/err.log
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/vgg16_b128_tf32.json 2>> $D/err.log
python bench.py --global-batch 512 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_r512.json > $D/resnet18_b512_3x.json 2>> $D/err.log
python bench.py --net googlenet --global-batch 256 --steps 20 --warmup 3 --no-cpu-baseline --layers-out $D/l_goog.json > $D/googlenet_b256_3x.json 2>> $D/err.log
python bench.py --impl reference --steps 2 --warmup 1 > $D/reference.json 2>> $D/err.log
ls -la $D
