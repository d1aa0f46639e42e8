# softmax inner-loop microbenchmark (bf16 pack variants) + the pipe microbenchmark
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2509_24745_b200/csrc -o /tmp/mbt scripts/microbench_tmem.cu && /tmp/mbt > gpurun_out/r3_mb_tmem2.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_pipes.cu && /tmp/mb > gpurun_out/r3_mb_pipes.txt 2>&1
cat gpurun_out/r3_mb_tmem2.txt gpurun_out/r3_mb_pipes.txt
