# compute-sanitizer over every kernel family (scripts/sanitize_cases.py); small ragged cases
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1; echo build=$?
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo $tool=$?; tail -3 gpurun_out/san_$tool.log
done
