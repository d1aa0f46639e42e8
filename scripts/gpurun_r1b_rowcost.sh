python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for n in 32768 65536 131072; do PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py $n 2>&1 | tail -1; done
PYTHONPATH=. PROXYATTN_ATTN=8 timeout 600 python scripts/attn_rowcost.py 65536 2>&1 | tail -1
