# Round 2: interleaved A/B of the d = 128 exp split (0 vs 1 of 8 on the FMA pipe), and varlen batches
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
PROXYATTN_NVCC_DEFINES="-DPA_EMU_D128=1" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/emu1.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/emu0.so
for rep in 1 2 3 4; do
  for e in 0 1; do
    cp /tmp/emu$e.so $SO
    timeout 300 python scripts/attn_time.py --tag "ab_emu$e" --steps 20 >> gpurun_out/r2_ab.jsonl 2>> gpurun_out/r2_ab.err
  done
done
cp /tmp/emu0.so $SO
python - <<'PY'
import json
for l in open("gpurun_out/r2_ab.jsonl"):
    d = json.loads(l); print(d["tag"], round(d["ms"], 3), d["clocks"]["sm_mhz"])
PY
for lens in 2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048,2048 8192,8192,8192,8192,8192,8192,8192,8192 16384,16384,16384,16384,16384,16384,16384,16384; do
  timeout 600 python scripts/varlen_bench.py $lens >> gpurun_out/r2_varlen.jsonl 2>> gpurun_out/r2_varlen.err
done
cat gpurun_out/r2_varlen.jsonl | cut -c1-400
