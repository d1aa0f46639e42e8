# Round 2: lazy softmax reference in the score passes (A2 always in this build; A4 with PA_LAZY_BUDGET)
# (the lazy-reference build was measured and dropped: profiles/r02_score_lazy_reference.jsonl; it
# needs scripts/_base_score_tc.cu and the lazy score_tc.cu from round-2 history to rerun)
mkdir -p gpurun_out
cp paper_2509_24745_b200/csrc/score_tc.cu /tmp/new_score_tc.cu
cp scripts/_base_score_tc.cu paper_2509_24745_b200/csrc/score_tc.cu
python -m paper_2509_24745_b200.build --force > /dev/null
for w in llama3.1-8b-attn-128k; do timeout 300 python scripts/attn_time.py --estimate --tag base --steps 30 >> gpurun_out/r2_lazy.jsonl 2>>gpurun_out/r2_lazy.err; done
cp /tmp/new_score_tc.cu paper_2509_24745_b200/csrc/score_tc.cu
for d in "" "-DPA_LAZY_BUDGET"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --estimate --tag "lazy$d" --steps 30 >> gpurun_out/r2_lazy.jsonl 2>>gpurun_out/r2_lazy.err
  PROXYATTN_NVCC_DEFINES="$d" timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_fuzz.py tests/test_gpu_maxsize.py tests/test_gpu_layouts.py "tests/test_gpu_fullsize.py" -k "not 256k and not 70b and not g95 and not 16k" -q -p no:cacheprovider > "gpurun_out/r2_lazy_tests$d.log" 2>&1
  echo "tests$d rc=$?"; tail -2 "gpurun_out/r2_lazy_tests$d.log"
done
cat gpurun_out/r2_lazy.jsonl
