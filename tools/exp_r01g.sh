# r01g: dX stride-phase walk (image-block-major across phases) + look at the HBM-bound small kernels
mkdir -p gpurun_out/r01g
timeout 900 python -m pytest tests -m gpu -q -x --tb=short -k "tma or fullsize or variants or integer" > gpurun_out/r01g/tests.log 2>&1; tail -3 gpurun_out/r01g/tests.log
for m in 3xtf32 tf32; do
timeout 300 python tools/layer_bench.py --layer l2.0a,l2.0sc,l3.0a,l3.0sc,l4.0a,l4.0sc,conv1 --math $m > gpurun_out/r01g/layers_$m.jsonl 2>&1
done
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/r01g/l20dx python tools/layer_bench.py --layer l2.0a --op dx --reps 1 > gpurun_out/r01g/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)0' -o gpurun_out/r01g/l2scfwd python tools/layer_bench.py --layer l2.0sc --op fwd --reps 1 >> gpurun_out/r01g/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o gpurun_out/r01g/l2scdx python tools/layer_bench.py --layer l2.0sc --op dx --reps 1 >> gpurun_out/r01g/full.log 2>&1
$NCU -k 'regex:zero' -o gpurun_out/r01g/l2sczero python tools/layer_bench.py --layer l2.0sc --op dx --reps 1 >> gpurun_out/r01g/full.log 2>&1
$NCU -k 'regex:direct_dw' -o gpurun_out/r01g/stemdw python tools/layer_bench.py --layer conv1 --op dw --reps 1 >> gpurun_out/r01g/full.log 2>&1
ls gpurun_out/r01g
