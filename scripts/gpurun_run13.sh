mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -4
nproc
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 4000 gpurun_out/bench_full.json; tail -5 gpurun_out/bench_full.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 2> gpurun_out/bench_ref.err | tail -1 > gpurun_out/bench_ref.json; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
