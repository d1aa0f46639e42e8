# Round 2 checkpoint: full GPU suite + smoke + sanitizer (memcheck / racecheck) on the current tree
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_check_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2_check_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
( for tool in memcheck racecheck synccheck initcheck; do echo "## $tool"; timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_cases.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ok|Error" | head -5; done ) > gpurun_out/r2_check_sanitizer.txt 2>&1
cat gpurun_out/r2_check_sanitizer.txt
