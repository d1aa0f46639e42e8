python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for wl in llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k; do
timeout 900 ncu --set full --clock-control none -k regex:attn_tc8 -c 1 -o gpurun_out/shapes2_$wl python bench.py --workload $wl --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph > /dev/null 2>&1; echo ncu_f $wl=$?
done
