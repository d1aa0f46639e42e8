PYTHONPATH=. timeout 600 python scripts/pcie_bw.py 2>&1 | tail -1
