python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; PYTHONPATH=. timeout 900 python scripts/layout_bench.py 2>&1 | tail -2
