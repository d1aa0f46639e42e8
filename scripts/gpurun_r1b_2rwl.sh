python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for wl in llama3.1-8b-attn-128k-b64 qwen2.5-7b-attn-64k; do
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --workload $wl --steps 3 --warmup 3 --no-lib-dense > gpurun_out/bench_2r_$wl.log 2>&1; echo $wl rc=$?
grep '^{' gpurun_out/bench_2r_$wl.log | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["value"], j["work_share"], j["e2e"] and j["e2e"]["value"], j["config"]["parallelism"])'
grep -E "Traceback|Error" gpurun_out/bench_2r_$wl.log | head -3
done
