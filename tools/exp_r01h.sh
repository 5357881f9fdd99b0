# r01h: STRIP 3xTF32 with 2 MMAs per k-step (a_hi x [b_hi;b_lo] at N=2BN, a_lo x b_hi at N=BN)
mkdir -p gpurun_out/r01h
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "strip or config1 or fullsize" > gpurun_out/r01h/tests.log 2>&1; tail -3 gpurun_out/r01h/tests.log
timeout 300 python tools/layer_bench.py --layer l1.0a,l2.0b --op fwd,dx --math 3xtf32 > gpurun_out/r01h/layers.jsonl 2>&1
timeout 300 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg2,vgg4 --op fwd,dx --math 3xtf32 >> gpurun_out/r01h/layers.jsonl 2>&1
cat gpurun_out/r01h/layers.jsonl | cut -c1-150
