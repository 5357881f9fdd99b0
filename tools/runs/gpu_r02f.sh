#!/bin/bash
# fused-epilogue GPU tests + ncu launch stats of the tiny / vgg11 calls (fixed per-kernel cost)
D=gpurun_out/r02f; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_epi_gpu.py -q > $D/epi.log 2>&1; tail -3 $D/epi.log
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_elapsed.max,launch__cluster_max_active,launch__grid_size,smsp__cycles_active.avg --clock-control none --csv --log-file $D/lat_ncu.csv python tools/lat_probe.py --quick > $D/lat_ncu.log 2>&1
