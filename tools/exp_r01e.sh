python tools/layer_bench.py --layer conv1 --op fwd --reps 20
