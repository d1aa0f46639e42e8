timeout 900 python -m pytest tests/test_gpu_layouts.py -m gpu -q --timeout=600 -p no:faulthandler 2>&1 | tail -5
