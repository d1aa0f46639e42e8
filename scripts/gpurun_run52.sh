timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:faulthandler -k "forward_host" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), j["e2e"])'
