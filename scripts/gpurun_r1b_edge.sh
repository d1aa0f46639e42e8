python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_shapes.py -q -k "tiny or stride8" 2>&1 | tail -15
