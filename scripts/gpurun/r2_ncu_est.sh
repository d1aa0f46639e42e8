# Round 2: MUFU probe + ncu --set full of the estimation kernels at 128K (one eager step)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/probe_mufu.cu -o /tmp/probe_mufu && /tmp/probe_mufu > gpurun_out/r2_probe_mufu.log 2>&1
cat gpurun_out/r2_probe_mufu.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"score_tc|select_kernel|pool_bf16|maxpool_from|budget_" -c 8 \
  -o gpurun_out/r2_est python bench.py --steps 1 --warmup 0 --no-graph --no-cpu --no-e2e --no-lib-dense --no-comparator > gpurun_out/r2_ncu_est.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/r2_ncu_est.log
ls -la gpurun_out/
