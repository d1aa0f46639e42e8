python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
bash scripts/gpurun_r1b_mp2.sh
for n in 16384 32768 131072; do timeout 600 python bench.py --seq-len $n --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["config"]["seq_len"], j["value"], j["estimate_ms"], j["prefill_ms"], j["sparsity"])'; done
timeout 600 python bench.py --workload qwen2.5-7b-attn-64k --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("qwen", j["value"], j["estimate_ms"], j["prefill_ms"], j["sparsity"])'
