python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python bench.py > gpurun_out/bench_head.json 2>gpurun_out/bench_head.err; echo head=$?
tail -1 gpurun_out/bench_head.json | cut -c1-400
for wl in llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k llama3.1-70b-attn-128k qwen2.5-7b-attn-64k; do
timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/bench_wl.jsonl 2>/dev/null; echo $wl rc=$?
done
for n in 16384 32768 65536 262144; do
timeout 900 python bench.py --seq-len $n --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/bench_seq.jsonl 2>/dev/null; echo $n rc=$?
done
for wl in llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_l $wl=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -c 1 -o gpurun_out/attn_full_$wl python bench.py --workload $wl --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_f $wl=$?
done
