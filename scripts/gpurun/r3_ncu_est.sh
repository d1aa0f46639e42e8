# ncu --set full (with source) of the estimation kernels at 128K: per-line stalls of the score passes
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"score_tc" -c 2 \
  -o gpurun_out/r3_est python scripts/attn_time.py --estimate --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_est.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/r3_ncu_est.log
