# Round 2: full GPU suite, smoke, bench on the current tree
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1
echo tests_rc=$?
tail -30 gpurun_out/r2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/r2_smoke.log
#timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo bench_rc=$?
#cat gpurun_out/r2_bench.json; tail -20 gpurun_out/r2_bench.err
