python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python scripts/dbg_pairs.py 2>&1 | tail -60
