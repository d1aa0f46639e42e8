# multicast debugging: which launch fails at 64K
# (targets the round-2 row-pair multicast build, measured and reverted: see DESIGN.md §6 and
# profiles/r02_attn_rowpair_multicast_ab.jsonl; PA_MC no longer exists in the tree)
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
PROXYATTN_NVCC_DEFINES="-DPA_MC=1" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/mc.so
PROXYATTN_NVCC_DEFINES="-DPA_MC=1 -DPA_MC_NOEXACT" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/mcne.so
cp /tmp/mc.so $SO
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/mc_check.py 65536 32 8 --preset llama-64k 2>&1 | grep -E "Error|error|bitwise|File.*_lib|line" | head -12
echo "== noexact"
cp /tmp/mcne.so $SO
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/mc_check.py 65536 32 8 --preset llama-64k 2>&1 | grep -E "Error|error|bitwise" | head -5
echo "== noexact 8/2 128K"
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/mc_check.py 131072 8 2 --preset llama-128k 2>&1 | grep -E "Error|error|bitwise" | head -5
echo "== 48K"
cp /tmp/mc.so $SO
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/mc_check.py 49152 32 8 2>&1 | grep -E "Error|error|bitwise" | head -5
