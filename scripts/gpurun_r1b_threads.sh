python -c "import __graft_entry__ as g; g.build()" > gpurun_out/th_build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_threads.py tests/test_gpu_graphs.py -q -p no:cacheprovider > gpurun_out/th_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/th_pytest.log
