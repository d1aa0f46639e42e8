set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "umma" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=300 2>&1 | tail -60
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
