# attn_tc9 with an S buffer per group and P written over it (PA_V9_PINS): oracle cases (wait-log
# build), tests, then A/B at 128K (headline, M-C-fixed, dense) x2
mkdir -p gpurun_out
PROXYATTN_NVCC_DEFINES="-DPA_V9_PINS=1 -DPA_WAIT_LOG" python -m paper_2509_24745_b200.build --force > gpurun_out/r3_pins_build.log 2>&1 || echo build_failed
timeout 300 python scripts/v9_debug.py > gpurun_out/r3_pins_dbg.log 2>&1; echo dbg_rc=$?; grep -v "line \|progress" gpurun_out/r3_pins_dbg.log | tail -8; grep -c "line " gpurun_out/r3_pins_dbg.log
PROXYATTN_NVCC_DEFINES="-DPA_V9_PINS=1" python -m paper_2509_24745_b200.build --force > /dev/null
PROXYATTN_NVCC_DEFINES="-DPA_V9_PINS=1" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -x -p no:cacheprovider > gpurun_out/r3_pins_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r3_pins_tests.log
for rep in 1 2; do
for d in "" "-DPA_V9_PINS=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  for w in llama3.1-8b-attn-128k llama3.1-8b-attn-128k-fixed; do
    PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload $w --tag "$w$d" --steps 20 >> gpurun_out/r3_pins.jsonl 2>> gpurun_out/r3_pins.err
  done
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --dense --tag "dense$d" --steps 5 >> gpurun_out/r3_pins.jsonl 2>> gpurun_out/r3_pins.err
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_pins.jsonl'):
    d=json.loads(l); print(f"{d['tag']:50s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
