PYTHONPATH=. timeout 600 python scripts/pair_union_stats.py 131072 128 2>&1 | tail -1; PYTHONPATH=. timeout 600 python scripts/pair_union_stats.py 65536 128 2>&1 | tail -1
