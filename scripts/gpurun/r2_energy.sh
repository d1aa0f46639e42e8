# Round 2: energy attribution of attn_tc8 at 128K (each variant removes one component; wrong outputs)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_24745_b200/csrc scripts/probe_f16p.cu -o /tmp/probe_f16p && /tmp/probe_f16p > gpurun_out/r2_probe.log 2>&1
cat gpurun_out/r2_probe.log
for d in "" "-DPA_X_NOMUFU" "-DPA_X_NOLOAD" "-DPA_X_NOQK" "-DPA_X_NOPV" "-DPA_X_EXBF16" "-DPA_X_NOQK -DPA_X_NOPV" ""; do
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --tag "x$d" --steps 10 >> gpurun_out/r2_energy.jsonl 2>> gpurun_out/r2_energy.err
done
cat gpurun_out/r2_energy.jsonl
tail -5 gpurun_out/r2_energy.err
