# Round 2: persistent score kernels — parity, then interleaved A/B of the estimate at 128K / 32K
# (the persistent score kernel was measured and reverted: profiles/r02_score_persistent_ab.jsonl)
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
cp paper_2509_24745_b200/csrc/score_tc.cu /tmp/new_score.cu
cp scripts/_base_score_tc.cu paper_2509_24745_b200/csrc/score_tc.cu
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/base.so
cp /tmp/new_score.cu paper_2509_24745_b200/csrc/score_tc.cu
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/pers.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_fuzz.py tests/test_gpu_maxsize.py tests/test_gpu_layouts.py tests/test_gpu_avgpool.py tests/test_gpu_graphs.py tests/test_gpu_threads.py "tests/test_gpu_fullsize.py" -k "not 256k and not 70b and not g95" -q -p no:cacheprovider > gpurun_out/r2_pers_tests.log 2>&1
echo tests_rc=$?; tail -3 gpurun_out/r2_pers_tests.log
for rep in 1 2 3; do
  for v in base pers; do
    cp /tmp/$v.so $SO
    timeout 200 python scripts/attn_time.py --estimate --tag "est_$v" --steps 30 >> gpurun_out/r2_pers.jsonl 2>> gpurun_out/r2_pers.err
    timeout 200 python scripts/attn_time.py --estimate --workload llama3.1-8b-attn-128k-b64 --tag "estb64_$v" --steps 30 >> gpurun_out/r2_pers.jsonl 2>> gpurun_out/r2_pers.err
  done
done
cp /tmp/pers.so $SO
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_pers_launches.csv python bench.py --steps 2 --warmup 1 --no-graph --no-cpu --no-e2e --no-lib-dense --no-comparator > /dev/null 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/r2_pers.jsonl"):
    d = json.loads(l); print(d["tag"], d["workload"], round(d["ms"], 4))
PY
