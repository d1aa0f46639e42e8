# final attn_tc9 (per-row exact re-runs): ncu --set full of the headline launch + the step's launch list
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc9 -s 0 -c 1 -o gpurun_out/r3_attn9_final \
  python scripts/attn_time.py --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_attn9_final.log 2>&1; echo ncu_attn_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph --no-comparator > /dev/null 2>&1; echo ncu_list_rc=$?
