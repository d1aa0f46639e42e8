python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for e in 2 3 2 3; do
PROXYATTN_EXP_EMU64=$e timeout 600 python bench.py --workload llama3.2-1b-attn-128k --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("emu64",'$e', j["value"], j["estimate_ms"], j["prefill_ms"], j["roofline"]["frac"], j["clocks"]["sm_mhz"])'
done
