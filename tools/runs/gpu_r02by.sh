#!/bin/bash
# r02by: validation of the tree after the DWS-pair experiment (kept behind SMCONV_DWS_PAIR=1, off): full GPU suite
# on the default path + the pair kernel's parity / coverage / full-size tests, its isolated time and the default bench line
D=gpurun_out/r02by; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_DWS_PAIR=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_coverage_gpu.py tests/test_configs_gpu.py tests/test_fullsize_gpu.py -q -x -k "dws or resnet18 or vgg2" > $D/pytest_pair.log 2>&1; echo "pair tests rc=$?"; tail -2 $D/pytest_pair.log
SMCONV_DWS_PAIR=1 timeout 300 python tools/layer_bench.py --net resnet18 --layer l1.0a --op dw --batch 4096 --math 3xtf32 > $D/lb_pair.log 2>&1; cut -c1-160 $D/lb_pair.log
timeout 400 python bench.py --steps 10 --warmup 3 > $D/b_resnet.log 2>&1; tail -1 $D/b_resnet.log | cut -c1-400
bash tools/gpu_tests.sh r02by/t > /dev/null 2>&1; tail -3 $D/t/pytest.log
