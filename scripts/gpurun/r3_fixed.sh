# M-C-fixed with the row-pair kernel: launch list (exact re-run share?) and v8 for comparison
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_fixed_v9_launches.csv \
  python scripts/attn_time.py --workload llama3.1-8b-attn-128k-fixed --steps 2 --warmup 0 --tag ncu > /dev/null 2>&1; echo rc=$?
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9=0" python -m paper_2509_24745_b200.build --force > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_fixed_v8_launches.csv \
  python scripts/attn_time.py --workload llama3.1-8b-attn-128k-fixed --steps 2 --warmup 0 --tag ncu > /dev/null 2>&1; echo rc=$?
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import csv
for f in ['gpurun_out/r3_fixed_v9_launches.csv','gpurun_out/r3_fixed_v8_launches.csv']:
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
    print(f, [(r[ki][:20], r[vi]) for r in rows[1:] if 'attn_tc' in r[ki]])
PY
