timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=300 -k "structured_staged" 2>&1 | tail -3
PYTHONPATH=. timeout 900 python scripts/estimation_sweep.py 2>&1 | tail -18 > gpurun_out/estimation_sweep.jsonl; cat gpurun_out/estimation_sweep.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload llama3.1-70b-attn-128k 2>/dev/null | tail -1 > gpurun_out/bench_70b.json; cat gpurun_out/bench_70b.json | head -c 1200
