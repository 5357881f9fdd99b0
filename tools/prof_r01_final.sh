# r01 final profile pass: launch list of the default bench + full captures of the top kernels
# (full captures through tools/layer_bench.py, which launches the plan bench.py times)
mkdir -p gpurun_out/r01f
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r01f/ncu_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_dws' -o gpurun_out/r01f/l1dw python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > gpurun_out/r01f/full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)0' -o gpurun_out/r01f/l1fwd python tools/layer_bench.py --layer l1.1b --op fwd --reps 1 >> gpurun_out/r01f/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/r01f/l21dx python tools/layer_bench.py --layer l2.1a --op dx --reps 1 >> gpurun_out/r01f/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)2' -o gpurun_out/r01f/l41dw python tools/layer_bench.py --layer l4.1a --op dw --reps 1 >> gpurun_out/r01f/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/r01f/l20dx python tools/layer_bench.py --layer l2.0a --op dx --reps 1 >> gpurun_out/r01f/full.log 2>&1
$NCU -k 'regex:conv_direct_fwd' -o gpurun_out/r01f/stem python tools/layer_bench.py --layer conv1 --op fwd --reps 1 >> gpurun_out/r01f/full.log 2>&1
ls -la gpurun_out/r01f
