# v9 at d = 64 (a S buffer per softmax group): oracle check of small cases (wait-log build),
# A7 timing v8 / v9 at d = 64 (x2), then the d = 64 GPU tests on the v9-d64 build
mkdir -p gpurun_out
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9_D64=1 -DPA_WAIT_LOG" python -m paper_2509_24745_b200.build --force > /dev/null 2>&1 || echo build_failed
timeout 300 python scripts/v9_debug.py 64 > gpurun_out/r3_d64_dbg.log 2>&1; echo dbg_rc=$?
grep -v "line 4\|progress" gpurun_out/r3_d64_dbg.log | head -20
for rep in 1 2; do
for d in "" "-DPA_ATTN_V9_D64=1" "-DPA_ATTN_V9_D64=1 -DPA_EMU_V9_D64=3" "-DPA_ATTN_V9_D64=1 -DPA_EMU_V9_D64=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload llama3.2-1b-attn-128k --tag "d64$d" --steps 20 >> gpurun_out/r3_d64.jsonl 2>> gpurun_out/r3_d64.err
done
done
python - <<'PY'
import json
for l in open('gpurun_out/r3_d64.jsonl'):
    d=json.loads(l); print(f"{d['tag']:50s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9_D64=1" python -m paper_2509_24745_b200.build --force > /dev/null
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_layouts.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/r3_d64_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/r3_d64_tests.log
python -m paper_2509_24745_b200.build --force > /dev/null
