timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench2.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench2.log
