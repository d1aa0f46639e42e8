# v9 as the default A7 kernel: full GPU suite, then A/B timing v8 / v9 / v9 + 1/4 poly exp2 (x2)
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3_v9b_tests.log 2>&1
echo tests_rc=$?
tail -15 gpurun_out/r3_v9b_tests.log
for rep in 1 2; do
for d in "-DPA_ATTN_V9=0" "" "-DPA_EMU_V9=2" "-DPA_EMU_V9=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --tag "x$d" --steps 20 >> gpurun_out/r3_v9b.jsonl 2>> gpurun_out/r3_v9b.err
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_v9b.jsonl'):
    d=json.loads(l); print(f"{d['tag']:30s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
