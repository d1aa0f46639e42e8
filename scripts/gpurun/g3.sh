set -x
./scripts/probe_f16p > gpurun_out/g3_probe.log 2>&1; echo probe_rc=$?
cat gpurun_out/g3_probe.log
timeout 1200 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_fuzz.py tests/test_gpu_layouts.py -q -s -p no:cacheprovider > gpurun_out/g3_tests.log 2>&1
echo tests_rc=$?
tail -3 gpurun_out/g3_tests.log
