python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for c in 4 8 16 32; do
PROXYATTN_HOST_CHUNKS=$c timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-lib-dense > gpurun_out/bench_e2e.log 2>&1; tail -1 gpurun_out/bench_e2e.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print('$c', j["value"], j["e2e"]["value"])'
done
