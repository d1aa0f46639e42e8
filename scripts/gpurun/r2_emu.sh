# Round 2: exp2 split of the attention kernel re-measured per shape (A7 alone, L2 flushed, medians)
mkdir -p gpurun_out
for e in 0 1 2; do
  d="-DPA_EMU_D128=$e -DPA_EMU_B64=$e -DPA_EMU_D64=$((e+1))"
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null
  for w in llama3.1-8b-attn-128k llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k; do
    PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload $w --tag "emu$d" --steps 20 >> gpurun_out/r2_emu.jsonl 2>> gpurun_out/r2_emu.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r2_emu.jsonl"):
    d = json.loads(l); print(d["workload"], d["defines"], round(d["ms"], 3), d["clocks"]["sm_mhz"])
PY
python -m paper_2509_24745_b200.build --force > /dev/null
for P in 2 4 8; do timeout 900 python scripts/rank_emulation.py $P 131072 --graph >> gpurun_out/r2_rank_emulation.jsonl 2>> gpurun_out/r2_rank_emulation.err; echo "P=$P rc=$?"; done
cat gpurun_out/r2_rank_emulation.jsonl; tail -3 gpurun_out/r2_rank_emulation.err
