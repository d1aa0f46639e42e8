# Round 2: how long the exact (re-run) launch takes in the sparse paths of every shape
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
for w in llama3.1-8b-attn-128k llama3.2-1b-attn-128k llama3.1-8b-attn-128k-b64 llama3.1-8b-attn-128k-g95 qwen2.5-7b-attn-64k; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_exact_$w.csv -k regex:attn_tc8 \
    python scripts/attn_time.py --workload $w --tag ncu --steps 1 --warmup 0 > /dev/null 2>&1
  python - $w <<'PY'
import csv, sys
w = sys.argv[1]
rows=list(csv.reader(open(f'gpurun_out/r2_exact_{w}.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr=rows[h]; vi=hdr.index('Metric Value'); mi=hdr.index('Metric Name')
print(w, "launches (us):", [round(float(r[vi].replace(',',''))/1000, 1) for r in rows[h+1:] if r[mi]=='gpu__time_duration.sum'])
PY
done
