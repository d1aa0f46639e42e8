# per-rank emulation of the 2/4/8-GPU zig-zag step with the row-pair attention (one GPU)
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
for P in 2 4 8; do timeout 900 python scripts/rank_emulation.py $P 131072 --graph >> gpurun_out/r3_rank_emulation.jsonl 2>> gpurun_out/r3_rank_emulation.err; echo "P=$P rc=$?"; done
cat gpurun_out/r3_rank_emulation.jsonl; tail -3 gpurun_out/r3_rank_emulation.err
