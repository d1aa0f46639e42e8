python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_shapes.py -q > gpurun_out/pytest_shapes.log 2>&1; echo shapes=$?
tail -3 gpurun_out/pytest_shapes.log
for wl in llama3.1-8b-attn-128k-b64; do
timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_$wl.log 2>&1; echo $wl rc=$?
tail -1 gpurun_out/bench_$wl.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["dense_ms"], j["sparsity"], j["roofline"]["frac"], j["clocks"]["sm_mhz"])'
done
PYTHONPATH=. timeout 900 python scripts/calibrate_shape.py 32 8 64 131072 128 0.8386 0.5 4.0 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["dense_ms"], j["roofline"]["frac"], j["clocks"]["sm_mhz"])'
