python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; timeout 900 python -m pytest tests/test_gpu_shapes.py -q -x -k "forward_host" 2>&1 | tail -3
