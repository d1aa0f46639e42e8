python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f3_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/f3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/f3_head.json 2>gpurun_out/f3_head.err; echo head=$?
tail -1 gpurun_out/f3_head.json | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["dense_ms"], j["dense_library"]["ms"], j["roofline"]["frac"], j["clocks"], j["e2e"]["value"], j["gpu_launches"])'
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f3_ref.json 2>/dev/null; echo ref=$?
