timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full2.json 2> gpurun_out/bench_full2.err; tail -c 2500 gpurun_out/bench_full2.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:attn_tc6 -c 1 -o gpurun_out/attn6_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN2pa --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for n in 16384 32768 65536 262144; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --seq-len $n 2>/dev/null | tail -1 >> gpurun_out/sweep2.jsonl; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload qwen2.5-7b-attn-64k 2>/dev/null | tail -1 >> gpurun_out/sweep2.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload llama3.1-70b-attn-128k 2>/dev/null | tail -1 >> gpurun_out/sweep2.jsonl
