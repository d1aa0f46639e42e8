# attn_tc9: dense as a template parameter (sparse instantiation back to its pre-dense code) and the
# split S load (PA_V9_SPLIT) A/B at 128K, headline and M-C-fixed (x2); correctness of both builds
mkdir -p gpurun_out
for d in "" "-DPA_V9_SPLIT=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -x -p no:cacheprovider > gpurun_out/r3_split_tests$d.log 2>&1; echo "tests$d rc=$?"; tail -1 gpurun_out/r3_split_tests$d.log
done
for rep in 1 2; do
for d in "" "-DPA_V9_SPLIT=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  for w in llama3.1-8b-attn-128k llama3.1-8b-attn-128k-fixed; do
    PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload $w --tag "$w$d" --steps 20 >> gpurun_out/r3_split.jsonl 2>> gpurun_out/r3_split.err
  done
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --dense --tag "dense$d" --steps 5 >> gpurun_out/r3_split.jsonl 2>> gpurun_out/r3_split.err
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_split.jsonl'):
    d=json.loads(l); print(f"{d['tag']:50s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
