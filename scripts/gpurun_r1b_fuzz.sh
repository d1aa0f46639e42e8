python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fz_build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider --durations=3 > gpurun_out/fz_pytest.log 2>&1; echo pytest=$?
grep -E "FAILED|passed|failed|assert|Error" gpurun_out/fz_pytest.log | head -30; tail -5 gpurun_out/fz_pytest.log
