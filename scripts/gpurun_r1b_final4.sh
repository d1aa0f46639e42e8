python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python bench.py > gpurun_out/final4_head.json 2>gpurun_out/final4_head.err; echo head=$?
for wl in llama3.1-70b-attn-128k qwen2.5-7b-attn-64k llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k llama3.1-8b-attn-128k-g95; do
timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/final4_wl.jsonl 2>/dev/null; echo $wl rc=$?
done
for n in 16384 32768 65536 262144; do
timeout 900 python bench.py --seq-len $n --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/final4_seq.jsonl 2>/dev/null; echo $n rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_l=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -c 1 -o gpurun_out/final4_attn_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_f=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/final4_est.csv -k regex:"pool|score_tc|lse_combine|maxpool|budget|select" python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_e=$?
for p in 2 4 8; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 131072 --graph 2>&1 | tail -1 >> gpurun_out/final4_ranks.jsonl; done; echo ranks=$?
