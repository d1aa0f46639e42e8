python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for n in 65536 131072; do PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py $n 2>&1 | tail -1; PROXYATTN_DIAG_NOLOAD=1 PYTHONPATH=. timeout 600 python scripts/attn_rowcost.py $n 2>&1 | tail -1; done
