# A/B of the P pack in attn_tc8 (F2FP vs integer-pipe packs) and the 1/4 poly exp2 split, at 128K
mkdir -p gpurun_out
python scripts/attn_time.py --tag ref --steps 3 --warmup 1 --save-out /tmp/O_ref.pt > /dev/null 2>&1
for rep in 1 2; do
for d in "" "-DPA_PACK=1" "-DPA_PACK=2" "-DPA_PACK=3" "-DPA_EMU_D128=2" "-DPA_EMU_D128=2 -DPA_PACK=3"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --tag "x$d" --steps 20 --check-out /tmp/O_ref.pt >> gpurun_out/r3_pack.jsonl 2>> gpurun_out/r3_pack.err
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json
for l in open('gpurun_out/r3_pack.jsonl'):
    d=json.loads(l); print(f"{d['tag']:40s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz  maxdiff {d.get('max_diff_vs_ref')}  meandiff {d.get('mean_diff_vs_ref')}")
PY
