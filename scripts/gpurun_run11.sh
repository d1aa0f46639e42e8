mkdir -p gpurun_out
for e in 1 2; do PROXYATTN_SCORE_EMU=$e timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=300 2>&1 | tail -1; done
for e in 0 1 2 3; do PROXYATTN_SCORE_EMU=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('semu',$e,{k:round(d[k],3) for k in ['value','speedup_vs_dense','estimate_ms','prefill_ms','tflops_exec']}, round(d['roofline']['frac'],3))"; done
PROXYATTN_SCORE_EMU=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN2pa --csv --log-file gpurun_out/launches_r1d.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
