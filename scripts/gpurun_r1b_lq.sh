python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lq.csv python bench.py --workload qwen2.5-7b-attn-64k --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu=$?
