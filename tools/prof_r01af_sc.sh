# r01af: ncu source-level capture of the l2.0sc fwd (1x1 s2, K = 64) to test the epilogue-store hypothesis
D=gpurun_out/r01af; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1 -k 'regex:conv_tma_kernel' -o $D/l2scfwd python tools/layer_bench.py --layer l2.0sc --op fwd --reps 1 > $D/full.log 2>&1
ncu -i $D/l2scfwd.ncu-rep --page raw --csv > $D/l2scfwd.raw.csv 2>/dev/null
ncu -i $D/l2scfwd.ncu-rep --page source --csv --print-source sass > $D/l2scfwd.sass.csv 2>/dev/null
rm -f $D/l2scfwd.ncu-rep; ls -la $D
