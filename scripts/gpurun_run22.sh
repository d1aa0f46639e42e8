timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print({k:round(d[k],3) for k in ['value','speedup_vs_dense','dense_ms','estimate_ms','prefill_ms','tflops_exec']}, round(d['roofline']['frac'],3), d['clocks'])"
PYTHONPATH=. timeout 300 python scripts/trace_attn.py 2>&1 | tail -4
