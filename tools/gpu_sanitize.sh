#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over one small call per kernel family (tools/sanitize_probe.py)
D=gpurun_out/${1:-san}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --kernel-name kns=smconv python tools/sanitize_probe.py > $D/$tool.log 2>&1
  echo "$tool rc=$?" >> $D/summary.txt; tail -3 $D/$tool.log >> $D/summary.txt
done
cat $D/summary.txt
