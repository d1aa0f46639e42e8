# multicast debugging: multi-item clusters at growing sizes, then sanitizer on a small multi-item case
# (targets the round-2 row-pair multicast build, measured and reverted: see DESIGN.md §6 and
# profiles/r02_attn_rowpair_multicast_ab.jsonl; PA_MC no longer exists in the tree)
mkdir -p gpurun_out
SO=paper_2509_24745_b200/libproxyattn.so
python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/base.so
PROXYATTN_NVCC_DEFINES="-DPA_MC=1" python -m paper_2509_24745_b200.build --force > /dev/null && cp $SO /tmp/mc.so
for shape in "4096 8 2" "8192 8 2" "16384 16 4" "32768 32 8"; do
  set -- $shape
  cp /tmp/base.so $SO; timeout 120 python scripts/mc_check.py $1 $2 $3 --save /tmp/O_$1.pt > /dev/null 2>&1
  cp /tmp/mc.so $SO; timeout 120 python scripts/mc_check.py $1 $2 $3 --check /tmp/O_$1.pt 2>&1 | tail -1
done
cp /tmp/mc.so $SO
timeout 600 compute-sanitizer --tool memcheck python scripts/mc_check.py 8192 8 2 --check /tmp/O_8192.pt 2>&1 | grep -v "^=========     " | tail -15
timeout 600 compute-sanitizer --tool synccheck python scripts/mc_check.py 8192 8 2 --check /tmp/O_8192.pt 2>&1 | grep -v "^=========     " | tail -15
