python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for rep in 1 2; do for c in 1 4 8 12 16 24; do PROXYATTN_HOST_CHUNKS=$c PYTHONPATH=. timeout 600 python scripts/e2e_chunks.py 10 2>&1 | tail -1; done; done
