# r01n: re-verify HEAD on a fresh box: GPU suite, smoke, default bench line (+ layers)
mkdir -p gpurun_out/r01n
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r01n/tests.log 2>&1; tail -5 gpurun_out/r01n/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01n/smoke.log 2>&1; tail -2 gpurun_out/r01n/smoke.log
timeout 600 python bench.py --layers-out gpurun_out/r01n/layers.json 2>gpurun_out/r01n/bench.err | tail -1 > gpurun_out/r01n/bench.json; cat gpurun_out/r01n/bench.json
