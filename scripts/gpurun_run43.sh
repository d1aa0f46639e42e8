timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b43.json 2>/dev/null; tail -1 gpurun_out/b43.json
PROXYATTN_ATTN=7 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("dense v7", j["dense_ms"])'
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc7 -c 1 -o gpurun_out/attn7_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
