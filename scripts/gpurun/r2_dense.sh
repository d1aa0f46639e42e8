# Round 2: the dense baseline (A8) at 128K — v3 (attn_tc) vs the v8 kernel's dense mode; launch split
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/v3.so
PROXYATTN_NVCC_DEFINES="-DPA_DENSE_TC8" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/v8.so
for v in v3 v8 v3 v8; do
  cp /tmp/$v.so $SO
  timeout 300 python scripts/attn_time.py --dense --tag "dense_$v" --steps 6 --warmup 2 >> gpurun_out/r2_dense.jsonl 2>> gpurun_out/r2_dense.err
done
cp /tmp/v8.so $SO
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_dense_v8_launches.csv -k regex:attn_tc8 \
  python scripts/attn_time.py --dense --tag ncu --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu_rc=$?
grep -o '"attn_tc8[^"]*","[^"]*","[^"]*",[^,]*,"gpu__time_duration.sum","[^"]*","[0-9.,]*"' gpurun_out/r2_dense_v8_launches.csv | head; tail -4 gpurun_out/r2_dense_v8_launches.csv | cut -c1-300
cp /tmp/v3.so $SO
python - <<'PY'
import json
for l in open("gpurun_out/r2_dense.jsonl"):
    d = json.loads(l); print(d["tag"], round(d["ms"], 2), round(d["tflops"]), d["clocks"]["sm_mhz"])
PY
