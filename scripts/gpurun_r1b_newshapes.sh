python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for wl in llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k; do
timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$wl.log 2>&1; echo $wl rc=$?
tail -1 gpurun_out/bench_$wl.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["dense_ms"], j.get("dense_library"), j["sparsity"], j["roofline"]["frac"], j["clocks"]["sm_mhz"])'
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b64.csv python bench.py --workload llama3.1-8b-attn-128k-b64 --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu=$?
