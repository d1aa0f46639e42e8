python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for gm in 0.7 0.8 0.85 0.9 0.95 0.98; do
timeout 900 python bench.py --gamma $gm --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/gsweep.jsonl 2>/dev/null
tail -1 gpurun_out/gsweep.jsonl | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["config"]["gamma"], round(j["sparsity"],4), round(j["value"],3), round(j["estimate_ms"],3), round(j["prefill_ms"],3), round(j["dense_ms"],2), round(j["dense_library"]["ms"],2), round(j["speedup_vs_dense"],2), round(j["dense_library"]["speedup_vs_library"],2), round(j["roofline"]["frac"],3))'
done
