# Session-3 evidence on the v9 tree: bench line, launch list, ncu --set full of attn_tc9,
# compute-sanitizer over every kernel family
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3_bench_v9.json 2> gpurun_out/r3_bench_v9.err; echo bench_rc=$?
cut -c1-300 gpurun_out/r3_bench_v9.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph --no-comparator > /dev/null 2>&1; echo ncu_list_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc9 -s 0 -c 1 -o gpurun_out/r3_attn9 \
  python scripts/attn_time.py --steps 1 --warmup 0 --tag ncu > gpurun_out/r3_ncu_attn9.log 2>&1; echo ncu_attn_rc=$?
( for tool in memcheck synccheck initcheck racecheck; do
    echo "## $tool"
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py 2>&1 | grep -v "^=========     \|Saved host backtrace" | tail -20
    echo "rc=$?"
  done ) > gpurun_out/r3_sanitizer.txt 2>&1
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ok|rc=" gpurun_out/r3_sanitizer.txt
