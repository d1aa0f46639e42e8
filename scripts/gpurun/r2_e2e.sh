# Round 2: host pipeline order (last rows first + V whole, vs first rows first + V progressive) x chunk count
# (PA_HOST_FWD / PA_HOST_CHUNKS existed only in the measured build, commit history of round 2; the
# forward order measured slower and was not kept: profiles/r02_e2e_order_sweep.jsonl)
mkdir -p gpurun_out
for d in "" "-DPA_HOST_FWD" "-DPA_HOST_FWD -DPA_HOST_CHUNKS=32" "-DPA_HOST_FWD -DPA_HOST_CHUNKS=8" "-DPA_HOST_CHUNKS=32"; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/e2e_time.py --tag "e2e$d" >> gpurun_out/r2_e2e.jsonl 2>> gpurun_out/r2_e2e.err
done
cat gpurun_out/r2_e2e.jsonl; tail -3 gpurun_out/r2_e2e.err
