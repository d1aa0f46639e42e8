mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=300 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print({k:round(d[k],3) for k in ['value','speedup_vs_dense','dense_ms','estimate_ms','prefill_ms','tflops_exec']}, round(d['roofline']['frac'],3), d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN2pa --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
