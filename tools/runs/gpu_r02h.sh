#!/bin/bash
D=gpurun_out/r02h; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for c in 8 4 2 0; do SMCONV_CSK=$c timeout 200 python tools/lat_probe.py --shape=tiny,vgg11,vgg6 > $D/lat_csk$c.log 2>&1; done
SMCONV_TMA_L2PROMO=0 timeout 200 python tools/lat_probe.py --shape=tiny,vgg11 > $D/lat_promo0.log 2>&1
