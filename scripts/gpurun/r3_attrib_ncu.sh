# Round 2 (session 3): ncu --set full of the A7 launch at 128K under the energy-attribution
# builds (wrong outputs; timing only) -- per-launch SM and L2 clocks, pipe use and L2 load
# throughput, to find what bounds the softmax / load path
mkdir -p gpurun_out
for d in "" "-DPA_X_NOLOAD" "-DPA_X_NOQK -DPA_X_NOPV" "-DPA_X_NOQK -DPA_X_NOPV -DPA_X_NOLOAD" "-DPA_X_NOMUFU"; do
  tag=$(echo "x$d" | tr -d ' ' | tr '=' '_')
  PROXYATTN_NVCC_DEFINES="$d" python -m paper_2509_24745_b200.build --force > /dev/null || { echo "build failed $d"; continue; }
  PROXYATTN_NVCC_DEFINES="$d" timeout 300 python scripts/attn_time.py --tag "$tag" --steps 10 >> gpurun_out/r3_attrib.jsonl 2>> gpurun_out/r3_attrib.err
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -s 0 -c 1 -o gpurun_out/r3_$tag \
    python scripts/attn_time.py --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_$tag.log 2>&1; echo "$tag ncu_rc=$?"
done
python -m paper_2509_24745_b200.build --force > /dev/null
cat gpurun_out/r3_attrib.jsonl
