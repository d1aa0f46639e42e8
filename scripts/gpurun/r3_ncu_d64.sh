# ncu --set full (source) of the d = 64 A7 launch (attn_tc8<2,64,128>) at 128K: where its softmax stalls
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -s 0 -c 1 -o gpurun_out/r3_d64 \
  python scripts/attn_time.py --workload llama3.2-1b-attn-128k --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_d64.log 2>&1; echo rc=$?
