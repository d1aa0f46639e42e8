python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=5 2>&1 | tail -12
