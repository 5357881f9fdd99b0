# r01m profile pass on the committed code: launch list of the default bench, full captures of the
# top kernels (through tools/layer_bench.py, the plan bench.py times), default bench line, smoke
mkdir -p gpurun_out/r01m_prof
timeout 600 python bench.py > gpurun_out/r01m_prof/bench.json 2>gpurun_out/r01m_prof/bench.err; tail -1 gpurun_out/r01m_prof/bench.json | cut -c1-300
cp gpurun_out/bench_layers.json gpurun_out/r01m_prof/bench_layers.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01m_prof/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r01m_prof/ncu_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_dws' -o gpurun_out/r01m_prof/l1dw python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > gpurun_out/r01m_prof/full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)0' -o gpurun_out/r01m_prof/l1fwd python tools/layer_bench.py --layer l1.1b --op fwd --reps 1 >> gpurun_out/r01m_prof/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/r01m_prof/l21dx python tools/layer_bench.py --layer l2.1a --op dx --reps 1 >> gpurun_out/r01m_prof/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)0' -o gpurun_out/r01m_prof/l31fwd python tools/layer_bench.py --layer l3.1a --op fwd --reps 1 >> gpurun_out/r01m_prof/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)2' -o gpurun_out/r01m_prof/l21dw python tools/layer_bench.py --layer l2.1a --op dw --reps 1 >> gpurun_out/r01m_prof/full.log 2>&1
ls gpurun_out/r01m_prof
