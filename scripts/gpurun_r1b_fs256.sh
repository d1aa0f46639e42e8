python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fs_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k "256k or 70b or g95" -q -s -p no:cacheprovider --durations=5 > gpurun_out/fs_pytest.log 2>&1; echo pytest=$?
grep -E "recall|passed|failed|Error|assert" gpurun_out/fs_pytest.log | head; tail -8 gpurun_out/fs_pytest.log
