python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_shapes.py -q -x -k "head_sharded" 2>&1 | tail -2
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-lib-dense > gpurun_out/bench_2r.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/bench_2r.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["work_share"], j["config"]["parallelism"], j["gpu_launches"])'
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 3 --warmup 3 --no-lib-dense --alg1 replicated > gpurun_out/bench_2r_rep.log 2>&1; echo bench2rep=$?
grep '^{' gpurun_out/bench_2r_rep.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["estimate_ms"], j["prefill_ms"], j["work_share"], j["config"]["parallelism"])'
tail -5 gpurun_out/bench_2r.log
