timeout 900 python -m pytest tests/test_gpu_layouts.py -m gpu -x -q --timeout=600 -p no:faulthandler 2>&1 | tail -25
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), round(j["estimate_ms"],3), round(j["prefill_ms"],3), round(j["roofline"]["frac"],4), j["clocks"].get("sm_mhz"), j["dense_ms"])'
PROXYATTN_ATTN=8 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("dense v8", j["dense_ms"])'
