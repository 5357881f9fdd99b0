#!/bin/bash
# r02cn: final HEAD check of the round (knob-off code since r02cj): smoke, full GPU suite, default bench line
D=gpurun_out/r02cn; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > $D/b_default.log 2>&1; tail -1 $D/b_default.log | cut -c1-300
bash tools/gpu_tests.sh r02cn/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
