# Round 2: K/V load attribution of attn_tc8 at 128K (wrong outputs; timing only)
mkdir -p gpurun_out
for d in "" "-DPA_X_HALFLOAD" "-DPA_X_NOKLOAD" "-DPA_X_NOVLOAD" "-DPA_X_NOLOAD" ""; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --tag "x$d" --steps 20 >> gpurun_out/r2_energy2.jsonl 2>> gpurun_out/r2_energy2.err
done
cat gpurun_out/r2_energy2.jsonl
tail -5 gpurun_out/r2_energy2.err
