PROXYATTN_ATTN=8 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench3.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench3.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["dense_ms"], j["dense_library"], j["prefill_ms"])'
