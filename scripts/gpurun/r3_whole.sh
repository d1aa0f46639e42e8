# v8 whole-S (S tile loaded at once, buffer released before the exp2s) A/B: d = 64 sparse, d = 128 dense
mkdir -p gpurun_out
for rep in 1 2; do
for d in "" "-DPA_WHOLE_S=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload llama3.2-1b-attn-128k --tag "d64$d" --steps 20 >> gpurun_out/r3_whole.jsonl 2>> gpurun_out/r3_whole.err
done
for d in "" "-DPA_WHOLE_S=2"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --dense --tag "dense$d" --steps 5 >> gpurun_out/r3_whole.jsonl 2>> gpurun_out/r3_whole.err
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_whole.jsonl'):
    d=json.loads(l); print(f"{d['tag']:30s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
PY
