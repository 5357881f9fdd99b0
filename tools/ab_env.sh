#!/bin/bash
# A/B a library knob on the same box: tools/ab_env.sh TAG "ENV=val ..." BENCH_ARGS...
# runs bench.py with and without the env assignment (3 alternations), layer tables in gpurun_out/TAG/
TAG=$1; ENVS=$2; shift 2
D=gpurun_out/$TAG; mkdir -p $D
for i in 1 2 3; do
  timeout 300 python bench.py "$@" --no-cpu-baseline --layers-out $D/l_base_$i.json > $D/b_base_$i.log 2>&1
  timeout 300 env $ENVS python bench.py "$@" --no-cpu-baseline --layers-out $D/l_exp_$i.json > $D/b_exp_$i.log 2>&1
done
for f in $D/b_*.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -1) $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
