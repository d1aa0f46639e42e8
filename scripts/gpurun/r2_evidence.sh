# Round 2 evidence: sanitizer over every kernel family, ncu --set full of A7, launch list, bench line
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
( for tool in memcheck synccheck initcheck racecheck; do
    echo "## $tool"
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py 2>&1 | grep -v "^=========     \|Saved host backtrace" | tail -40
    echo "rc=$?"
  done ) > gpurun_out/r2_sanitizer.txt 2>&1
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ok|rc=" gpurun_out/r2_sanitizer.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -s 0 -c 1 -o gpurun_out/r2_attn8 \
  python scripts/attn_time.py --steps 1 --warmup 0 --tag ncu > gpurun_out/r2_ncu_attn.log 2>&1; echo ncu_attn_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph --no-comparator > /dev/null 2>&1; echo ncu_list_rc=$?
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
cat gpurun_out/r2_bench.json
