python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_tc --launch-skip 1 -c 1 -o gpurun_out/a2b_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu=$?
