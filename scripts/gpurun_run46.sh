for v in 7 8; do
for n in 16384 32768 65536 262144; do echo "v$v $n $(PROXYATTN_ATTN=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --seq-len $n 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), round(j["prefill_ms"],3), round(j["roofline"]["frac"],4), j["clocks"]["sm_mhz"])')"; done
for w in qwen2.5-7b-attn-64k llama3.1-70b-attn-128k; do echo "v$v $w $(PROXYATTN_ATTN=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload $w 2>/dev/null | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["value"],3), round(j["prefill_ms"],3), round(j["roofline"]["frac"],4), j["clocks"]["sm_mhz"])')"; done
done
