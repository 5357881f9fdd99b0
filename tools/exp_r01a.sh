timeout 600 python -m pytest tests/test_parity_gpu.py -q --tb=line -x 2>&1 | tail -2
L="--layer l1.0a,l4.1a --op fwd --reps 10"
python tools/layer_bench.py $L --math tf32
SMCONV_TMA_G=32 python tools/layer_bench.py $L --math tf32
SMCONV_TMA_L2PROMO=0 python tools/layer_bench.py $L --math tf32
SMCONV_TMA_L2PROMO=2 python tools/layer_bench.py $L --math tf32
python tools/layer_bench.py $L --math 3xtf32
SMCONV_TMA_G=32 python tools/layer_bench.py $L --math 3xtf32
python tools/layer_bench.py --layer l1.0a --op fwd --batch 512 --math tf32 --reps 10
python tools/layer_bench.py --layer l1.0a --op fwd --batch 128 --math tf32 --reps 10
