python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; timeout 600 python -m pytest tests/test_gpu_shapes.py -q -x -k varlen 2>&1 | tail -3
