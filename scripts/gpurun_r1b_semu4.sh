python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2 3; do for e in 0 1; do
PROXYATTN_BUDGET_EMU=$e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"score_tc" python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph 2>/dev/null | grep -E "score_tc" | python -c "
import sys,csv
print('bemu $e', [r[-1] for r in csv.reader(sys.stdin)])"
done; done
