# sustained MMA rate and power with random operands: 1-CTA vs CTA pair (N = 64, 128), ~3 s each
run() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 200 > gpurun_out/pw_$1.csv & P=$!; sleep 0.5; shift; "$@"; kill $P; }
run r64 ./tools/ring_bench.bin 600000 0
run r128 ./tools/ring_bench.bin 500000 1
run p64 ./tools/pair_bench.bin 1300000 0
run p128 ./tools/pair_bench.bin 650000 1
