python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python bench.py --workload llama3.1-8b-attn-128k-g95 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g95.json 2>/dev/null; echo rc=$?
tail -1 gpurun_out/g95.json | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["dense_ms"], j["dense_library"]["ms"], j["sparsity"], j["roofline"]["frac"], j["speedup_vs_dense"])'
