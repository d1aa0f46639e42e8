python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc8 -c 1 -o gpurun_out/attn_full_64k_b python bench.py --seq-len 65536 --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu=$?
