python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for p in 2 4 8; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 131072 --graph 2>&1 | tail -1 > gpurun_out/ranks_$p.json; python -c "import json; j=json.load(open('gpurun_out/ranks_$p.json')); print(j['P'], j['single_gpu_step_ms'], j['max_rank_step_ms'], j['projected_speedup'])"; done
cat gpurun_out/ranks_2.json gpurun_out/ranks_4.json gpurun_out/ranks_8.json > gpurun_out/ranks_all.jsonl
