#!/bin/bash
D=gpurun_out/r02m; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
python tools/trace_probe.py tiny,vgg11,vgg6,vgg9 > $D/trace.log 2>&1
python tools/lat_probe.py --shape=tiny,vgg11,vgg6 > $D/lat.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_epi_gpu.py tests/test_configs_gpu.py -q -x -k "csk or tma or vgg or epi" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
timeout 300 python bench.py --net vgg16 --math tf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_tf32.json > $D/b_vgg_tf32.log 2>&1
timeout 300 python bench.py --net vgg16 --math 3xtf32 --steps 20 --warmup 5 --no-cpu-baseline --layers-out $D/l_vgg_3x.json > $D/b_vgg_3x.log 2>&1
