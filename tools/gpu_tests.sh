#!/bin/bash
# GPU test pass: build, the listed test files (default: all -m gpu), parity log -> gpurun_out/$TAG/
TAG=${1:-r02}; shift; FILES=${@:-tests}
D=gpurun_out/$TAG; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
rm -f gpurun_out/parity_errors.json
timeout 2400 python -m pytest $FILES -m gpu -q > $D/pytest.log 2>&1; echo "pytest rc=$?" >> $D/pytest.log
cp gpurun_out/parity_errors.json $D/ 2>/dev/null
tail -30 $D/pytest.log
