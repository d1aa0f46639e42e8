mkdir -p gpurun_out
for e in 0 1 2; do PROXYATTN_EXP_EMU=$e timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "structured_staged or single_block or determinism" 2>&1 | tail -1; done
for e in 0 1 2 3; do PROXYATTN_EXP_EMU=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('emu',$e,{k:round(d[k],3) for k in ['value','speedup_vs_dense','dense_ms','estimate_ms','prefill_ms','tflops_exec']}, round(d['roofline']['frac'],3), d['clocks'])"; done
