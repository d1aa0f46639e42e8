timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"maxpool|score_tc" python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-lib-dense --no-graph 2>/dev/null | grep -E "maxpool|score_tc" | python -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print(r[4][:40], r[-1])"
