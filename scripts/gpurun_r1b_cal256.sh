python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
PYTHONPATH=. timeout 1500 python scripts/calibrate_shape.py 32 8 128 262144 128 0.8386 0.4 1.2 2>&1 | tail -2
