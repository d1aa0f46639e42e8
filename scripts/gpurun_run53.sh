timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:faulthandler -k "row_range" 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:faulthandler 2>&1 | tail -3
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | cut -c1-1500
