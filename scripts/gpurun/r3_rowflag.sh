# v9 with per-row exact re-runs: correctness (oracle cases, parity / shapes / fuzz / graphs),
# A/B v8 / v9 at 128K on the headline and M-C-fixed inputs (x2), M-C-fixed launch list
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > gpurun_out/r3_rowflag_build.log 2>&1 || echo build_failed
timeout 300 python scripts/v9_debug.py > gpurun_out/r3_rowflag_dbg.log 2>&1; echo dbg_rc=$?; tail -4 gpurun_out/r3_rowflag_dbg.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py -q -x -p no:cacheprovider > gpurun_out/r3_rowflag_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r3_rowflag_tests.log
for rep in 1 2; do
for d in "-DPA_ATTN_V9=0" ""; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  for w in llama3.1-8b-attn-128k llama3.1-8b-attn-128k-fixed; do
    PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --workload $w --tag "$w$d" --steps 20 >> gpurun_out/r3_rowflag.jsonl 2>> gpurun_out/r3_rowflag.err
  done
done
done
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_fixed_v9c_launches.csv \
  python scripts/attn_time.py --workload llama3.1-8b-attn-128k-fixed --steps 2 --warmup 0 --tag ncu > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import json, csv
for l in open('gpurun_out/r3_rowflag.jsonl'):
    d=json.loads(l); print(f"{d['tag']:50s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
rows=[r for r in csv.reader(open('gpurun_out/r3_fixed_v9c_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
print([r[vi] for r in rows[1:] if 'attn_tc' in r[ki]])
PY
