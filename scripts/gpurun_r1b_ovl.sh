python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_shapes.py -q -x -k "scores_only or concurrent" 2>&1 | tail -1
for p in 4 8; do PYTHONPATH=. timeout 900 python scripts/rank_emulation.py $p 131072 --graph 2>&1 | tail -1 > gpurun_out/ranks_$p.json; python -c "import json; j=json.load(open('gpurun_out/ranks_$p.json')); print(j['P'], j['single_gpu_step_ms'], j['max_rank_step_ms'], j['projected_speedup'], [(o['estimate_ms'], o['attention_ms']) for o in j['ranks']])"; done
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-lib-dense --no-e2e > gpurun_out/bench_2r.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/bench_2r.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["gpu_launches"], j["config"]["launch"])'
grep -iE "Traceback|Error" gpurun_out/bench_2r.log | head -3
