for v in "" "-DPA_S_EARLY" "" "-DPA_S_EARLY"; do
PROXYATTN_NVCC_DEFINES="$v" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build [$v]=$?"
for n in 65536 131072; do PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py $n 2>&1 | tail -1 | python -c 'import sys,json; j=json.loads(sys.stdin.read()); print(j["N"], round(j["bench_lists"]["ms"],3), round(j["bench_lists"]["ns_per_block"],3))'; done
done
