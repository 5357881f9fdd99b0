# r01n: why are CTA-pair tiles slower?  ncu --set full of l3.1a fwd with and without pairs
D=gpurun_out/r01n_pairprof; mkdir -p $D
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -s 0 -c 1"
SMCONV_PAIR=0 $NCU -k 'regex:conv_tma_kernel' -o $D/l31fwd_single python tools/layer_bench.py --layer l3.1a --op fwd --reps 1 > $D/full.log 2>&1
SMCONV_PAIR=1 $NCU -k 'regex:conv_tma_kernel' -o $D/l31fwd_pair python tools/layer_bench.py --layer l3.1a --op fwd --reps 1 >> $D/full.log 2>&1
for v in 0 1; do SMCONV_PAIR=$v timeout 120 python tools/layer_bench.py --layer l3.1a,l2.1a --op fwd,dx 2>&1 | cut -c1-170; done
ls $D
