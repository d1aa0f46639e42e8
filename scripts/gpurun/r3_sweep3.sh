# Round 2, session 3 final kernels incl. A8 on the row-pair kernel: full GPU suite + every workload + reference line + default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3_sweep3_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r3_sweep3_tests.log
run() { timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" >> gpurun_out/r3_sweep3.jsonl 2>> gpurun_out/r3_sweep3.err; echo "$* rc=$?"; }
run --workload llama3.1-8b-attn-128k
for n in 16384 32768 65536 262144; do run --workload llama3.1-8b-attn-128k --seq-len $n --no-comparator; done
for w in llama3.1-70b-attn-128k qwen2.5-7b-attn-64k llama3.1-8b-attn-128k-g95 llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k llama3.1-8b-attn-128k-fixed; do run --workload $w --no-comparator; done
python - <<'PY'
import json
for l in open("gpurun_out/r3_sweep3.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["config"]["seq_len"], round(d["value"], 2), round(d["estimate_ms"], 3), round(d["prefill_ms"], 2),
          round(d["dense_ms"], 1), round((d.get("dense_library") or {}).get("ms") or 0, 1), round(d["speedup_vs_dense"], 2), round(d["speedup_vs_own_dense"], 2),
          round(d["tflops_exec"]), round(d["roofline"]["frac"], 3), round(d["dense_tflops"]), d["clocks"]["sm_mhz"], round(d["sparsity"], 4))
PY
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3_reference3.json 2>> gpurun_out/r3_sweep3.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3_bench_final4.json 2>> gpurun_out/r3_sweep3.err; echo bench_rc=$?
cut -c1-400 gpurun_out/r3_bench_final4.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke4.log 2>&1; echo smoke_rc=$?
