python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
nproc
s=$(date +%s); timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$? secs=$(( $(date +%s) - s ))
grep -E "Elapsed|Maximum resident" gpurun_out/ref.err
cut -c1-300 gpurun_out/ref.json
