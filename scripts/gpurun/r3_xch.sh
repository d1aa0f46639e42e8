# v9 with a 3-stage K ring (exchange / row-sum scratch shared): correctness, then A/B at 128K
# on the headline and the M-C-fixed inputs (x2)
mkdir -p gpurun_out
PROXYATTN_NVCC_DEFINES="-DPA_V9_XCH=1" python -m paper_2509_24745_b200.build --force > gpurun_out/r3_xch_build.log 2>&1 || echo build_failed
timeout 300 python scripts/v9_debug.py > gpurun_out/r3_xch_dbg.log 2>&1; echo dbg_rc=$?; tail -6 gpurun_out/r3_xch_dbg.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/r3_xch_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r3_xch_tests.log
for rep in 1 2; do
for d in "" "-DPA_V9_XCH=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  for w in llama3.1-8b-attn-128k llama3.1-8b-attn-128k-fixed; do
    PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload $w --tag "$w$d" --steps 20 >> gpurun_out/r3_xch.jsonl 2>> gpurun_out/r3_xch.err
  done
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_xch.jsonl'):
    d=json.loads(l); print(f"{d['tag']:50s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
