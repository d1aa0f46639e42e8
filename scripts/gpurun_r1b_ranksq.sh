python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for p in 2 4; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 65536 --graph --qwen 2>&1 | tail -1 >> gpurun_out/ranks_qwen.jsonl; done
cat gpurun_out/ranks_qwen.jsonl | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); print(j['P'], j['single_gpu_step_ms'], j['max_rank_step_ms'], j['projected_speedup'], [(o['estimate_ms'],o['attention_ms']) for o in j['ranks']])"
