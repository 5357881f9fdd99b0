# r01r (part 2): ncu --set full captures of the top kernels; raw counters exported to CSV on the box
D=gpurun_out/r01r_ncu; mkdir -p $D
NCU="timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
$NCU -k 'regex:conv_dws' -o $D/l1dw python tools/layer_bench.py --layer l1.1b --op dw --reps 1 > $D/full.log 2>&1
$NCU -k 'regex:conv_strip_kernel<\(int\)0' -o $D/l1fwd python tools/layer_bench.py --layer l1.1b --op fwd --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o $D/l21dx python tools/layer_bench.py --layer l2.1a --op dx --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)0' -o $D/l31fwd python tools/layer_bench.py --layer l3.1a --op fwd --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)2' -o $D/l21dw python tools/layer_bench.py --layer l2.1a --op dw --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o $D/l20dx python tools/layer_bench.py --layer l2.0a --op dx --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_tma_kernel<\(int\)1' -o $D/l2scdx python tools/layer_bench.py --layer l2.0sc --op dx --reps 1 >> $D/full.log 2>&1
$NCU -k 'regex:conv_direct_fwd' -o $D/stem python tools/layer_bench.py --layer conv1 --op fwd --reps 1 >> $D/full.log 2>&1
for f in $D/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null; done
for f in $D/*.ncu-rep; do case $f in *l1dw*|*l20dx*) ;; *) rm -f $f;; esac; done
du -sh $D; ls $D
