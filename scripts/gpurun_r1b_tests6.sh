python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t6_build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/t6_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/t6_pytest.log 2>&1; echo pytest=$?
tail -14 gpurun_out/t6_pytest.log
timeout 600 python bench.py > gpurun_out/t6_bench.json 2> gpurun_out/t6_bench.err; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/t6_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
