python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l16.csv python bench.py --seq-len 16384 --steps 2 --warmup 3 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu=$?
