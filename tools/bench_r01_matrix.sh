# r01 bench matrix (1 GPU): default line + TF32 + VGG-16 b128 + ResNet-18 b512 + GoogLeNet b256, and the reference arm
mkdir -p gpurun_out/r01_matrix
python bench.py > gpurun_out/r01_matrix/resnet18_b4096_3x.json 2> gpurun_out/r01_matrix/err1.log
python bench.py --math tf32 --no-cpu-baseline --layers-out gpurun_out/r01_matrix/l_tf32.json > gpurun_out/r01_matrix/resnet18_b4096_tf32.json 2>> gpurun_out/r01_matrix/err1.log
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --no-cpu-baseline --layers-out gpurun_out/r01_matrix/l_vgg.json > gpurun_out/r01_matrix/vgg16_b128_3x.json 2>> gpurun_out/r01_matrix/err1.log
python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline --layers-out gpurun_out/r01_matrix/l_vgg_tf32.json > gpurun_out/r01_matrix/vgg16_b128_tf32.json 2>> gpurun_out/r01_matrix/err1.log
python bench.py --global-batch 512 --steps 30 --warmup 5 --no-cpu-baseline --layers-out gpurun_out/r01_matrix/l_r512.json > gpurun_out/r01_matrix/resnet18_b512_3x.json 2>> gpurun_out/r01_matrix/err1.log
python bench.py --net googlenet --global-batch 256 --steps 20 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/r01_matrix/l_goog.json > gpurun_out/r01_matrix/googlenet_b256_3x.json 2>> gpurun_out/r01_matrix/err1.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01_matrix/reference.json 2>> gpurun_out/r01_matrix/err1.log
tail -c 300 gpurun_out/r01_matrix/*.json
