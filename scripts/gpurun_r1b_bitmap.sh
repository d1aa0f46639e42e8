python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_shapes.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k b64 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"pair_union" python bench.py --workload llama3.1-8b-attn-128k-b64 --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph 2>/dev/null | grep pair_union | awk -F'","' '{print $(NF-2)" "$(NF-1)" "$NF}' | head -3
