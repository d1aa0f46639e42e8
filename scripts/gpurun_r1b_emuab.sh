python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for rep in 1 2 3; do for e in 1 2 0; do
echo "emu=$e $(PROXYATTN_EXP_EMU=$e PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py 131072 2>&1 | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["bench_lists"]["ms"],3), round(j["bench_lists"]["ns_per_block"],3))')"
done; done
