for rep in 1 2; do for v in "-DPA_KSTAGES=3 -DPA_VSTAGES=2" "-DPA_KSTAGES=2 -DPA_VSTAGES=3" "-DPA_KSTAGES=2 -DPA_VSTAGES=2"; do
PROXYATTN_NVCC_DEFINES="$v" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || echo buildfail
echo "[$v] $(PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py 131072 2>&1 | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["bench_lists"]["ms"],3), round(j["bench_lists"]["ns_per_block"],3))') $(PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py 32768 2>&1 | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(round(j["bench_lists"]["ms"],3), round(j["bench_lists"]["ns_per_block"],3))')"
done; done
