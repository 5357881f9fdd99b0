# end-of-round check: full GPU suite, smoke(), default bench line
timeout 1200 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py 2>/dev/null | tail -1
