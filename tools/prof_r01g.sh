# r01 final profile pass: launch list of the default bench + full captures of the top kernels
# (captured through tools/layer_bench.py, which launches the same plan bench.py times)
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r01g_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_tma_kernel<\(int\)3' -o gpurun_out/prof_r01g_l1dw python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > gpurun_out/ncu_r01g_full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)0' -o gpurun_out/prof_r01g_l1fwd python tools/layer_bench.py --layer l1.1b --op fwd --reps 1 >> gpurun_out/ncu_r01g_full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)1' -o gpurun_out/prof_r01g_l1dx python tools/layer_bench.py --layer l1.1b --op dx --reps 1 >> gpurun_out/ncu_r01g_full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/prof_r01g_l20dx python tools/layer_bench.py --layer l2.0a --op dx --reps 1 >> gpurun_out/ncu_r01g_full.log 2>&1
$NCU -k 'regex:conv_direct' -o gpurun_out/prof_r01g_stem python tools/layer_bench.py --layer conv1 --op fwd --reps 1 >> gpurun_out/ncu_r01g_full.log 2>&1
ls -la gpurun_out | grep r01g
