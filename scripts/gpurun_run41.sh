export PROXYATTN_ATTN=7
PYTHONPATH=. timeout 300 python scripts/dbg_spike.py
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout=600 -p no:faulthandler 2>&1 | tail -3
for e in 2 3 4; do echo "emu $e $(PROXYATTN_EXP_EMU=$e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), round(j["prefill_ms"],3), round(j["roofline"]["frac"],4))')"; done
