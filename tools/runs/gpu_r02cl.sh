#!/bin/bash
# r02cl: energy per call on the final tree (ResNet-18 b4096 3xTF32 and TF32)
D=gpurun_out/r02cl; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
timeout 900 python tools/power_probe.py --layer conv1,l1.0a,l2.0a,l2.1a,l3.1a,l4.1a,l2.0sc --math 3xtf32 > $D/p3.log 2>&1
timeout 600 python tools/power_probe.py --layer l1.0a,l2.1a,l3.1a --math tf32 > $D/pt.log 2>&1
for f in $D/p*.log; do echo $f; python - $f <<'P'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(f"  {d['layer']:7} {d['op']:3} {d['ms']*1000:7.0f}us {d['watts']:6.0f}W {d['sm_mhz']:6.0f}MHz {d['mj_per_call']:7.1f}mJ {d['pj_per_flop']:6.2f}pJ/flop {d['plan'][:45]}")
P
done
