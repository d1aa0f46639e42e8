python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
PROXYATTN_HOST_ORDER=fwd timeout 900 python -m pytest tests -m gpu -q -x -k "forward_host" 2>&1 | tail -1
for rep in 1 2; do for o in rev fwd; do for c in 8 16 32; do PROXYATTN_HOST_ORDER=$o PROXYATTN_HOST_CHUNKS=$c PYTHONPATH=. timeout 600 python scripts/e2e_chunks.py 8 2>&1 | tail -1 | sed "s/^/$o /"; done; done; done
