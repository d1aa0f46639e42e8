rm -f gpurun_out/sweep3.jsonl
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full4.json 2> gpurun_out/bench_full4.err; tail -c 3000 gpurun_out/bench_full4.json
for n in 16384 32768 65536 262144; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --seq-len $n 2>/dev/null | tail -1 >> gpurun_out/sweep3.jsonl; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload qwen2.5-7b-attn-64k 2>/dev/null | tail -1 >> gpurun_out/sweep3.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload llama3.1-70b-attn-128k 2>/dev/null | tail -1 >> gpurun_out/sweep3.jsonl
PYTHONPATH=. timeout 900 python scripts/estimation_sweep.py > gpurun_out/est_sweep3.jsonl 2>/dev/null; tail -3 gpurun_out/est_sweep3.jsonl
