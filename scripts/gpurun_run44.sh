export PROXYATTN_ATTN=8
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout=200 -p no:faulthandler -k "structured or spikes or single_block or row_range or determinism" 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), round(j["prefill_ms"],3), round(j["roofline"]["frac"],4), j["clocks"], j["dense_ms"])'
