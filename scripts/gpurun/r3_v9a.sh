# v9 (row-pair attention) first test: timing + output diff vs v8 at 128K, then the parity suite
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 300 python scripts/attn_time.py --tag v8 --steps 10 --save-out /tmp/O8.pt >> gpurun_out/r3_v9a.jsonl 2>> gpurun_out/r3_v9a.err
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9=1" python -m paper_2509_24745_b200.build --force > gpurun_out/r3_v9a_build.log 2>&1 || echo build_failed
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9=1" timeout 300 python scripts/attn_time.py --tag v9 --steps 10 --check-out /tmp/O8.pt >> gpurun_out/r3_v9a.jsonl 2>> gpurun_out/r3_v9a.err
echo v9_rc=$?
cat gpurun_out/r3_v9a.jsonl
tail -5 gpurun_out/r3_v9a.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -p no:cacheprovider > gpurun_out/r3_v9a_tests.log 2>&1
echo tests_rc=$?
tail -30 gpurun_out/r3_v9a_tests.log
