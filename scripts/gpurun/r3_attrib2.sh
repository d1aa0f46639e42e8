# Round 2 (session 3): softmax-loop microbenchmark (no barriers / MMAs) and ncu --set full of
# the A7 fast launch at 128K: shipped build and the softmax-path-only build (no MMAs, no K/V loads)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2509_24745_b200/csrc -o /tmp/mbt scripts/microbench_tmem.cu && /tmp/mbt > gpurun_out/r3_mb_tmem.txt 2>&1
cat gpurun_out/r3_mb_tmem.txt
for d in "" "-DPA_X_NOQK -DPA_X_NOPV -DPA_X_NOLOAD"; do
  tag=$(echo "f$d" | tr -d ' ' | tr '=' '_')
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -s 0 -c 1 -o gpurun_out/r3_$tag \
    python scripts/attn_time.py --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_$tag.log 2>&1; echo "$tag ncu_rc=$?"
done
python -m paper_2509_24745_b200.build --force > /dev/null
