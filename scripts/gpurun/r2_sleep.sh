# Round 2: suspend-hint barrier waits by role (PA_SLEEP 0-3), A7 alone at 128K (d = 128 / 64, b = 64)
mkdir -p gpurun_out
for lv in 0 1 2 3; do
  PROXYATTN_NVCC_DEFINES="-DPA_SLEEP=$lv" python -m paper_2509_24745_b200.build --force > /dev/null || { echo build_fail $lv; continue; }
  for w in llama3.1-8b-attn-128k llama3.2-1b-attn-128k llama3.1-8b-attn-128k-b64; do
    if [ $lv = 0 ]; then extra="--save-out /tmp/O_$w.pt"; else extra="--check-out /tmp/O_$w.pt"; fi
    PROXYATTN_NVCC_DEFINES="-DPA_SLEEP=$lv" timeout 240 python scripts/attn_time.py --workload $w --tag "sleep$lv" --steps 20 $extra >> gpurun_out/r2_sleep.jsonl 2>> gpurun_out/r2_sleep.err
    echo "lv=$lv $w rc=$?"
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r2_sleep.jsonl"):
    d = json.loads(l); print(d["tag"], d["workload"], round(d["ms"], 3), d["clocks"]["sm_mhz"], d.get("max_diff_vs_ref"))
PY
