# Round 2: ncu --set full (with source) of the d = 64 attention launch; fullsize parity incl. M-C-fixed
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -s 0 -c 1 -o gpurun_out/r2_attn8_d64 \
  python scripts/attn_time.py --workload llama3.2-1b-attn-128k --steps 1 --warmup 0 --tag ncu > gpurun_out/r2_ncu_d64.log 2>&1; echo ncu_rc=$?
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "fixed" > gpurun_out/r2_fixed_tests.log 2>&1; echo fixed_tests_rc=$?; tail -2 gpurun_out/r2_fixed_tests.log
