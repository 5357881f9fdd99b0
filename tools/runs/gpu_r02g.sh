#!/bin/bash
D=gpurun_out/r02g; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_epi_gpu.py -q > $D/epi.log 2>&1; tail -3 $D/epi.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:conv_tma -c 1 -o $D/tiny python tools/lat_probe.py --quick --shape=tiny > $D/tiny.log 2>&1
ncu -i $D/tiny.ncu-rep --page raw --csv > $D/tiny.raw.csv 2>/dev/null
ncu -i $D/tiny.ncu-rep --page source --csv --print-source sass > $D/tiny.sass.csv 2>/dev/null
rm -f $D/tiny.ncu-rep
