# r01fin: final round-1 measurement (pairs for TMA fwd/dX/dW + STRIP, s2dx, stem dW heuristic)
# full GPU suite, smoke, bench matrix (+ per-call layers), reference arm, launch list, ncu full captures
D=gpurun_out/r01fin; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --tb=short > $D/tests.log 2>&1; tail -3 $D/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 600 python bench.py --layers-out $D/l_3x.json > $D/resnet18_b4096_3x.json 2> $D/err.log; tail -1 $D/resnet18_b4096_3x.json | cut -c1-200
timeout 300 python bench.py --math tf32 --no-cpu-baseline --layers-out $D/l_tf32.json > $D/resnet18_b4096_tf32.json 2>> $D/err.log
timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg.json > $D/vgg16_b128_3x.json 2>> $D/err.log
timeout 300 python bench.py --net vgg16 --global-batch 128 --steps 50 --warmup 5 --math tf32 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/vgg16_b128_tf32.json 2>> $D/err.log
timeout 300 python bench.py --global-batch 512 --steps 30 --warmup 5 --no-cpu-baseline --layers-out $D/l_r512.json > $D/resnet18_b512_3x.json 2>> $D/err.log
timeout 300 python bench.py --net googlenet --global-batch 256 --steps 20 --warmup 3 --no-cpu-baseline --layers-out $D/l_goog.json > $D/googlenet_b256_3x.json 2>> $D/err.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $D/reference.json 2>> $D/err.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $D/ncu_bench.log 2>&1
NCU="timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_dws' -o $D/l1dw python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > $D/full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)0' -o $D/l1fwd python tools/layer_bench.py --layer l1.1b --op fwd --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)2' -o $D/l31dw python tools/layer_bench.py --layer l3.1a --op dw --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)2' -o $D/l21dw python tools/layer_bench.py --layer l2.1a --op dw --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)0' -o $D/l20dx_s2dx python tools/layer_bench.py --layer l2.0a --op dx --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)0' -o $D/l21fwd python tools/layer_bench.py --layer l2.1a --op fwd --reps 1 >> $D/full.log 2>&1
for f in $D/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null; rm -f $f; done
du -sh $D; ls $D
