# Round 2: b = 64 dense walked diagonal-first — parity + timing vs the ascending build
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/new.so
timeout 1200 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "dense or b64 or 64-64 or 128-64 or gamma" -q -p no:cacheprovider > gpurun_out/r2_dense3_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2_dense3_tests.log
for v in new new; do
  timeout 300 python scripts/attn_time.py --dense --workload llama3.1-8b-attn-128k-b64 --tag "dense_b64_desc" --steps 4 --warmup 2 >> gpurun_out/r2_dense3.jsonl 2>> gpurun_out/r2_dense3.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_dense3_launches.csv -k regex:attn_tc8 \
  python scripts/attn_time.py --dense --workload llama3.1-8b-attn-128k-b64 --tag ncu --steps 1 --warmup 0 > /dev/null 2>&1
python - <<'PY'
import csv, json
rows=list(csv.reader(open('gpurun_out/r2_dense3_launches.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr=rows[h]; vi=hdr.index('Metric Value'); mi=hdr.index('Metric Name')
print("launches (ns):", [r[vi] for r in rows[h+1:] if r[mi]=='gpu__time_duration.sum'])
for l in open("gpurun_out/r2_dense3.jsonl"):
    d = json.loads(l); print(d["tag"], round(d["ms"], 2), d["clocks"]["sm_mhz"])
PY
