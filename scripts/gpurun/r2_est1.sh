# Round 2: estimation changes (FMNMX3 window maxima, 64-bit sort words) — parity + timing, exp split sweep
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_maxsize.py tests/test_gpu_avgpool.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/r2_est1_tests.log 2>&1
echo tests_rc=$?; tail -3 gpurun_out/r2_est1_tests.log
for e in 1 2 0; do
  PROXYATTN_NVCC_DEFINES="-DPA_SCORE_EMU=$e" python -m paper_2509_24745_b200.build --force > /dev/null
  for w in llama3.1-8b-attn-128k; do
    PROXYATTN_NVCC_DEFINES="-DPA_SCORE_EMU=$e" timeout 300 python scripts/attn_time.py --estimate --tag "est_emu$e" --workload $w --steps 30 >> gpurun_out/r2_est1.jsonl 2>>gpurun_out/r2_est1.err
  done
done
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_est1_launches.csv python bench.py --steps 2 --warmup 1 --no-graph --no-cpu --no-e2e --no-lib-dense --no-comparator > /dev/null 2>&1
echo ncu_rc=$?
cat gpurun_out/r2_est1.jsonl; tail -3 gpurun_out/r2_est1.err
