# r01i: DWS 3xTF32 with 2 MMAs per k-step; full bench with STRIP + DWS changes
mkdir -p gpurun_out/r01i
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -k "dws or strip or fullsize" > gpurun_out/r01i/tests.log 2>&1; tail -3 gpurun_out/r01i/tests.log
timeout 300 python tools/layer_bench.py --layer l1.0a --op dw,fwd --math 3xtf32 > gpurun_out/r01i/layers.jsonl 2>&1
timeout 300 python tools/layer_bench.py --net vgg16 --batch 128 --layer vgg2 --op dw --math 3xtf32 >> gpurun_out/r01i/layers.jsonl 2>&1
cut -c1-150 gpurun_out/r01i/layers.jsonl
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01i/bench.json; cut -c1-400 gpurun_out/r01i/bench.json
cp gpurun_out/bench_layers.json gpurun_out/r01i/ 2>/dev/null
