set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_avgpool.py tests/test_gpu_graphs.py tests/test_gpu_parity.py -x -q -s -p no:cacheprovider > gpurun_out/g1_tests.log 2>&1
echo tests_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
echo bench_rc=$?
tail -3 gpurun_out/g1_tests.log
