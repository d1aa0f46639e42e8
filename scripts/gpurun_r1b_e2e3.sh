python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-lib-dense > gpurun_out/bench_e2e.log 2>&1; tail -1 gpurun_out/bench_e2e.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["e2e"])'
