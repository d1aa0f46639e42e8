python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
rm -f gpurun_out/ranks_final.jsonl
for p in 2 4 8; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 131072 --graph 2>&1 | tail -1 >> gpurun_out/ranks_final.jsonl; done
for p in 2 4; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 65536 --graph --qwen 2>&1 | tail -1 >> gpurun_out/ranks_final_qwen.jsonl; done
python -c "
import json
for f in ['gpurun_out/ranks_final.jsonl','gpurun_out/ranks_final_qwen.jsonl']:
    for l in open(f):
        j=json.loads(l); print(j['workload'], j['P'], j['single_gpu_step_ms'], j['max_rank_step_ms'], j['projected_speedup'], max(o['estimate_ms'] for o in j['ranks']))"
