timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full3.json 2> gpurun_out/bench_full3.err; tail -c 3000 gpurun_out/bench_full3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -c 1 -o gpurun_out/attn8_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:_ZN2pa --csv --log-file gpurun_out/launches_r1g.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref3.json 2>/dev/null; tail -c 1500 gpurun_out/bench_ref3.json
