python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for rep in 1 2; do for e in 0 1 2; do
PROXYATTN_EXP_EMU64=$e timeout 600 python bench.py --workload llama3.2-1b-attn-128k --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("d64 emu",'$e', round(j["prefill_ms"],3), round(j["roofline"]["frac"],3))'
done; done
