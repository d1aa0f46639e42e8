mkdir -p gpurun_out
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9=1 -DPA_WAIT_LOG" python -m paper_2509_24745_b200.build --force > gpurun_out/r3_v9dbg_build.log 2>&1 || echo build_failed
timeout 300 python scripts/v9_debug.py > gpurun_out/r3_v9dbg.log 2>&1; echo rc=$?
tail -40 gpurun_out/r3_v9dbg.log
