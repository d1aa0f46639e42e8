set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1
PROXYATTN_PAIR_MODE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:attn_tc -c 1 -o gpurun_out/attn_full2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_full2.log 2>&1; tail -1 gpurun_out/ncu_full2.log
