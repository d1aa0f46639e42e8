python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-lib-dense > gpurun_out/bench_2r.log 2>&1; echo bench2=$?
grep '^{' gpurun_out/bench_2r.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["e2e"], j["gpu_launches"], j["config"]["parallelism"])'
grep -iE "error|Traceback" gpurun_out/bench_2r.log | head -5
