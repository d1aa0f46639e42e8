# run-to-run spread of the headline (5 back-to-back default-workload runs, 10 timed steps each)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sp_build.log 2>&1; echo build=$?
for i in 1 2 3 4 5; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/spread.jsonl 2>/dev/null; echo run$i=$?
done
python - <<'PY'
import json
for l in open('gpurun_out/spread.jsonl'):
    d=json.loads(l); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
