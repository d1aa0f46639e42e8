# Round 2: row-pair multicast attention (PA_MC) — correctness first, then interleaved A/B timing
# (targets the round-2 row-pair multicast build, measured and reverted: see DESIGN.md §6 and
# profiles/r02_attn_rowpair_multicast_ab.jsonl; PA_MC no longer exists in the tree)
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/base.so
PROXYATTN_NVCC_DEFINES="-DPA_MC=1" python -m paper_2509_24745_b200.build --force > gpurun_out/r2_mc_build.log 2>&1 && cp $SO /tmp/mc.so || { echo build_fail; cat gpurun_out/r2_mc_build.log | tail; exit 1; }
cp /tmp/base.so $SO
timeout 120 python scripts/attn_time.py --tag base_ref --steps 3 --save-out /tmp/O_ref.pt >> gpurun_out/r2_mc.jsonl 2>> gpurun_out/r2_mc.err
cp /tmp/mc.so $SO
timeout 120 python scripts/attn_time.py --tag mc_check --steps 3 --check-out /tmp/O_ref.pt >> gpurun_out/r2_mc.jsonl 2>> gpurun_out/r2_mc.err; echo "mc first run rc=$?"
tail -3 gpurun_out/r2_mc.err; tail -1 gpurun_out/r2_mc.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_graphs.py tests/test_gpu_threads.py tests/test_gpu_fullsize.py -k "not 256k and not 16k and not 64k and not g95" -x -q -p no:cacheprovider > gpurun_out/r2_mc_tests.log 2>&1; echo mc_tests_rc=$?; tail -3 gpurun_out/r2_mc_tests.log
for rep in 1 2 3; do
  for v in base mc; do
    cp /tmp/$v.so $SO
    timeout 200 python scripts/attn_time.py --tag "ab_$v" --steps 20 >> gpurun_out/r2_mc.jsonl 2>> gpurun_out/r2_mc.err
  done
done
cp /tmp/base.so $SO
python - <<'PY'
import json
for l in open("gpurun_out/r2_mc.jsonl"):
    d = json.loads(l); print(d["tag"], round(d["ms"], 3), d["clocks"]["sm_mhz"], d.get("max_diff_vs_ref"), d.get("mean_diff_vs_ref"))
PY
