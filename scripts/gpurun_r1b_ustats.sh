PYTHONPATH=. timeout 600 python scripts/pair_union_stats.py 131072 2>&1 | tail -2
