#!/bin/bash
# ncu capture of ONE conv call (one layer, one op) for the profiles/ evidence.
#   tools/prof.sh TAG NET LAYER OP BATCH MATH [KERNEL_REGEX]
# writes gpurun_out/TAG/{TAG.raw.csv, TAG.sass.csv, full.log}; read here with tools/ncu_summary.py.
set -u
TAG=$1; NET=$2; LAYER=$3; OP=$4; BATCH=$5; MATH=$6; KRE=${7:-regex:conv_}
D=gpurun_out/$TAG; mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 \
  -k "$KRE" -o $D/$TAG python tools/layer_bench.py --net $NET --layer $LAYER --op $OP --batch $BATCH \
  --math $MATH --reps 1 > $D/full.log 2>&1
ncu -i $D/$TAG.ncu-rep --page raw --csv > $D/$TAG.raw.csv 2>/dev/null
ncu -i $D/$TAG.ncu-rep --page source --csv --print-source sass > $D/$TAG.sass.csv 2>/dev/null
rm -f $D/$TAG.ncu-rep
