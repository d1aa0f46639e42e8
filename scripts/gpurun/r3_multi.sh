# Round 2 session 3 (row-pair A7): multi-rank bench paths on one GPU (BENCH_SAME_DEVICE=1: gloo only, timings meaningless),
# the full 32K oracle layer vs the GPU on every element, and the 32K full-size test
mkdir -p gpurun_out
for sh in rows heads; do
  BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 3 --warmup 3 --shard $sh --no-cpu > gpurun_out/r3_multi_$sh.json 2> gpurun_out/r3_multi_$sh.err
  echo "multi $sh rc=$?"; tail -c 1500 gpurun_out/r3_multi_$sh.json; tail -3 gpurun_out/r3_multi_$sh.err
done
timeout 1500 python scripts/oracle_full_32k.py --out gpurun_out/r3_oracle_full_32k.json > gpurun_out/r3_oracle_full_32k.log 2>&1
echo "oracle32k rc=$?"; tail -c 2000 gpurun_out/r3_oracle_full_32k.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider -k "32k" > gpurun_out/r3_fullsize32k.log 2>&1
echo "fullsize32k rc=$?"; tail -15 gpurun_out/r3_fullsize32k.log
