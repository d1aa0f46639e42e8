python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_shapes.py -q -x -k "varlen" 2>&1 | tail -2
PYTHONPATH=. timeout 600 python scripts/varlen_bench.py 2>&1 | tail -1
PYTHONPATH=. timeout 600 python scripts/varlen_bench.py 32768,16384,8192,8192,4096,2048,2048,1000 2>&1 | tail -1
