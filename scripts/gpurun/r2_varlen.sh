# Round 2: varlen estimates over up to 8 lanes — tests + timing
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 1200 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_graphs.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -k "varlen" > gpurun_out/r2_varlen_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2_varlen_tests.log
L32=$(python -c "print(','.join(['2048']*32))"); L64=$(python -c "print(','.join(['1024']*64))"); LMIX=$(python -c "print(','.join(str(x) for x in [32768,1024,4096,512,8192,2048,16384,1000,3000,700]*2))")
for lens in $L32 $L64 8192,8192,8192,8192,8192,8192,8192,8192 16384,16384,16384,16384,16384,16384,16384,16384 $LMIX; do
  timeout 600 python scripts/varlen_bench.py $lens >> gpurun_out/r2_varlen_lanes.jsonl 2>> gpurun_out/r2_varlen_lanes.err
done
python - <<'PY'
import json
for l in open("gpurun_out/r2_varlen_lanes.jsonl"):
    d = json.loads(l); print(len(d["lens"]), sum(d["lens"]), {k: round(v, 3) for k, v in d.items() if k != "lens"})
PY
