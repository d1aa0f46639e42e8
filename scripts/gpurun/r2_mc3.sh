# multicast debugging: bisect the 128K failure
# (targets the round-2 row-pair multicast build, measured and reverted: see DESIGN.md §6 and
# profiles/r02_attn_rowpair_multicast_ab.jsonl; PA_MC no longer exists in the tree)
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/base.so
PROXYATTN_NVCC_DEFINES="-DPA_MC=1" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/mc.so
for shape in "65536 32 8 llama-64k" "131072 8 2 llama-128k" "131072 32 8" "131072 32 8 llama-128k"; do
  set -- $shape
  pr=""; [ -n "$4" ] && pr="--preset $4"
  cp /tmp/base.so $SO; timeout 120 python scripts/mc_check.py $1 $2 $3 $pr --save /tmp/O.pt > /dev/null 2>&1
  cp /tmp/mc.so $SO; timeout 120 python scripts/mc_check.py $1 $2 $3 $pr --check /tmp/O.pt 2>&1 | tail -2
  echo "== $shape rc=$?"
done
