#!/bin/bash
# r02cf: the full GPU suite with programmatic dependent launch on EVERY kernel (SMCONV_PDL=2, what bench.py
# uses below 1024 images/GPU), and the coverage test repeated 3x (intermittent races)
D=gpurun_out/r02cf; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1 || { tail -20 $D/build.log; exit 1; }
SMCONV_PDL=2 timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_pdl2.log 2>&1; echo "pdl2 rc=$?"; tail -2 $D/pytest_pdl2.log
for r in 1 2 3; do SMCONV_PDL=2 timeout 300 python -m pytest tests/test_coverage_gpu.py -q > $D/cov_$r.log 2>&1; echo "cov $r rc=$?"; tail -1 $D/cov_$r.log; done
