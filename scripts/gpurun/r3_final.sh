# Round 2, session 3 final tree: full GPU suite, smoke, default bench line
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3_final_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3_final_tests.log 2>&1
echo tests_rc=$?
tail -5 gpurun_out/r3_final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_final_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/r3_final_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3_final_bench.json 2> gpurun_out/r3_final_bench.err
echo bench_rc=$?
cut -c1-400 gpurun_out/r3_final_bench.json
