python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mx_build.log 2>&1; echo build=$?
free -g | head -2; nproc
timeout 1500 python -m pytest tests/test_gpu_maxsize.py -x -q -p no:cacheprovider --durations=5 > gpurun_out/mx_pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/mx_pytest.log
