python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for p in 8; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 131072 2>&1 | tail -1 > gpurun_out/ranks_$p.json; python -c "import json; j=json.load(open('gpurun_out/ranks_$p.json')); print(j['P'], j['single_gpu_step_ms'], j['max_rank_step_ms'], j['projected_speedup'], [(o['estimate_ms'], o['attention_ms']) for o in j['ranks']])"; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/bench_s.log 2>&1; tail -1 gpurun_out/bench_s.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["roofline"]["frac"], j["clocks"]["sm_mhz"])'
