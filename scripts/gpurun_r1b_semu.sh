python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for e in 0 1 2 3; do
PROXYATTN_SCORE_EMU=$e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("emu",'$e', j["value"], j["estimate_ms"], j["prefill_ms"], j["clocks"]["sm_mhz"])'
done
for c in 32 64; do
PROXYATTN_SCORE_CHUNK=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print("chunk",'$c', j["value"], j["estimate_ms"], j["prefill_ms"], j["clocks"]["sm_mhz"])'
done
