export PROXYATTN_ATTN=7
PYTHONPATH=. timeout 300 python scripts/cta_times.py
