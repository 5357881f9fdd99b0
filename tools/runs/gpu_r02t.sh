#!/bin/bash
D=gpurun_out/r02t; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python tools/mc_probe.py > $D/mc_probe.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "x64x64x64 or x16x96 or dws" > $D/pytest_dws.log 2>&1; tail -2 $D/pytest_dws.log
timeout 300 python bench.py --net resnet18@128 --steps 5 --warmup 3 --no-cpu-baseline --layers-out $D/l_r128.json > $D/b_r128.log 2>&1
timeout 300 python bench.py --net resnet18@224 --steps 5 --warmup 3 --no-cpu-baseline --layers-out $D/l_r224.json > $D/b_r224.log 2>&1
timeout 300 python bench.py --net resnet18@64 --steps 5 --warmup 3 --no-cpu-baseline --layers-out $D/l_r64.json > $D/b_r64.log 2>&1
bash tools/gpu_sanitize.sh r02t/san > /dev/null 2>&1; cat $D/san/summary.txt
timeout 2400 python -m pytest tests -m gpu -q > $D/pytest.log 2>&1; tail -2 $D/pytest.log
cp gpurun_out/parity_errors.json $D/
for f in $D/b_*.log; do echo $f; tail -1 $f | cut -c1-150; done
