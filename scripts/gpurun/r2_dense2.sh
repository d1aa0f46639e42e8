# Round 2: dense mode of the v8 kernel with blocks in descending order vs v3, + launch split + dense parity
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/v3.so
PROXYATTN_NVCC_DEFINES="-DPA_DENSE_TC8" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/v8.so
for v in v3 v8 v3 v8; do
  cp /tmp/$v.so $SO
  timeout 300 python scripts/attn_time.py --dense --tag "dense_$v" --steps 6 --warmup 2 >> gpurun_out/r2_dense2.jsonl 2>> gpurun_out/r2_dense2.err
done
cp /tmp/v8.so $SO
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_dense2_v8_launches.csv -k regex:attn_tc8 \
  python scripts/attn_time.py --dense --tag ncu --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu_rc=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2_dense2_v8_launches.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr=rows[h]; vi=hdr.index('Metric Value'); mi=hdr.index('Metric Name')
print("v8 dense launches (ns):", [r[vi] for r in rows[h+1:] if r[mi]=='gpu__time_duration.sum'])
PY
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_fullsize.py -k "dense or gamma or fixed_launch or 128k and not b64 and not 70b and not g95 and not fixed" -q -p no:cacheprovider > gpurun_out/r2_dense2_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2_dense2_tests.log
cp /tmp/v3.so $SO
python - <<'PY'
import json
for l in open("gpurun_out/r2_dense2.jsonl"):
    d = json.loads(l); print(d["tag"], round(d["ms"], 2), round(d["tflops"]), d["clocks"]["sm_mhz"])
PY
