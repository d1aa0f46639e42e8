# Round 2: every bench workload / length on the round-2 build (one JSON line each)
mkdir -p gpurun_out
python -m paper_2509_24745_b200.build --force > /dev/null
run() { timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" >> gpurun_out/r2_sweep.jsonl 2>> gpurun_out/r2_sweep.err; echo "$* rc=$?"; }
run --workload llama3.1-8b-attn-128k
for n in 16384 32768 65536 262144; do run --workload llama3.1-8b-attn-128k --seq-len $n --no-comparator; done
for w in llama3.1-70b-attn-128k qwen2.5-7b-attn-64k llama3.1-8b-attn-128k-g95 llama3.1-8b-attn-128k-b64 llama3.2-1b-attn-128k; do run --workload $w --no-comparator; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_reference.json 2>> gpurun_out/r2_sweep.err; echo ref_rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/r2_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["config"]["seq_len"], round(d["value"], 2), round(d["estimate_ms"], 3), round(d["prefill_ms"], 2),
          round(d["dense_ms"], 1), (d.get("dense_library") or {}).get("ms"), round(d["speedup_vs_dense"], 2), round(d["tflops_exec"]), round(d["roofline"]["frac"], 3), d["clocks"]["sm_mhz"], round(d["sparsity"], 4))
PY
