set -x
timeout 2400 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_avgpool.py tests/test_gpu_graphs.py tests/test_gpu_parity.py tests/test_gpu_threads.py tests/test_gpu_shapes.py -q -s -p no:cacheprovider > gpurun_out/g2_tests.log 2>&1
echo tests_rc=$?
tail -5 gpurun_out/g2_tests.log
