# A8 (dense) on the row-pair kernel (diagonal-first walk): correctness on the dense tests, then
# A/B vs attn_tc8's dense mode at 128K (x2) and the launch list (exact re-run share)
mkdir -p gpurun_out
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9_DENSE=1" python -m paper_2509_24745_b200.build --force > gpurun_out/r3_dense9_build.log 2>&1 || echo build_failed
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_layouts.py -q -x -k "dense or config_a or structured or token_major" -p no:cacheprovider > gpurun_out/r3_dense9_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r3_dense9_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "dense and (128k and not b64 and not 1b and not 70b and not g95 and not fixed)" -p no:cacheprovider > gpurun_out/r3_dense9_full.log 2>&1; echo full_rc=$?; tail -3 gpurun_out/r3_dense9_full.log
for rep in 1 2; do
for d in "" "-DPA_ATTN_V9_DENSE=1"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --dense --tag "dense$d" --steps 5 >> gpurun_out/r3_dense9.jsonl 2>> gpurun_out/r3_dense9.err
done
done
PROXYATTN_NVCC_DEFINES="-DPA_ATTN_V9_DENSE=1" python -m paper_2509_24745_b200.build --force > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_dense9_launches.csv \
  python scripts/attn_time.py --dense --steps 1 --warmup 0 --tag ncu > /dev/null 2>&1; echo rc=$?
python -m paper_2509_24745_b200.build --force > /dev/null
python - <<'PY'
import json, csv
for l in open('gpurun_out/r3_dense9.jsonl'):
    d=json.loads(l); print(f"{d['tag']:40s} {d['ms']:.3f} ms  min {d['min_ms']:.3f}  {d['tflops']:.0f} TF/s  {d['clocks']['sm_mhz']} MHz")
rows=[r for r in csv.reader(open('gpurun_out/r3_dense9_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
print([r[vi] for r in rows[1:] if 'attn_tc' in r[ki]])
PY
