python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e64_build.log 2>&1; echo build=$?
for e in 1 2 3 4 2; do
PROXYATTN_EXP_EMU64=$e timeout 600 python bench.py --workload llama3.2-1b-attn-128k --steps 10 --warmup 3 --no-cpu --no-e2e --no-lib-dense > gpurun_out/e64_$e.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/e64_$e.json').read().strip().splitlines()[-1]);print('emu64=$e', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
