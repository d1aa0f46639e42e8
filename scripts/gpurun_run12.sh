mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
nproc; lscpu | grep "Model name"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 3000 gpurun_out/bench_full.json
for n in 16384 32768 65536 262144; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --seq-len $n 2>/dev/null | tail -1 >> gpurun_out/sweep.jsonl; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload qwen2.5-7b-attn-64k 2>/dev/null | tail -1 >> gpurun_out/sweep.jsonl
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/bench_ref.json; cat gpurun_out/bench_ref.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:score_tc -c 3 -o gpurun_out/score_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"pool_bf16|select_kernel|budget_combine|budget_finalize" -c 4 -o gpurun_out/small_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:attn_tc -c 1 -o gpurun_out/attn_full3 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN2pa --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
