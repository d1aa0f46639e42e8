# Round 2: M-C-fixed workload (static K* = 164) and the per-rank emulation on the round-2 build
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
timeout 900 python bench.py --workload llama3.1-8b-attn-128k-fixed --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/r2_fixed.json 2> gpurun_out/r2_fixed.err; echo fixed_rc=$?
tail -c 600 gpurun_out/r2_fixed.json
for P in 2 4 8; do timeout 900 python scripts/rank_emulation.py $P 131072 --graph >> gpurun_out/r2_rank_emulation.jsonl 2>> gpurun_out/r2_rank_emulation.err; echo "P=$P rc=$?"; done
cat gpurun_out/r2_rank_emulation.jsonl; tail -3 gpurun_out/r2_rank_emulation.err
