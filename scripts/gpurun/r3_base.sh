# Session 3 of round 2: state of the restored tree (full GPU suite, smoke, bench) and an ncu
# --set full of cuDNN's dense kernel on the same 128K inputs (comparison for A7)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3_build.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
echo bench_rc=$?
cut -c1-600 gpurun_out/r3_bench.json
timeout 600 ncu --set full --clock-control none --profile-from-start off -o gpurun_out/r3_cudnn \
  python scripts/cudnn_ncu.py > gpurun_out/r3_cudnn_ncu.log 2>&1; echo ncu_cudnn_rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3_tests.log 2>&1
echo tests_rc=$?
tail -3 gpurun_out/r3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1; echo smoke_rc=$?
