"""CPU: bench.py's driver contract.  The reference arm (`--impl reference`: the fp64 oracle on
the host cores, the one other place bench.py may run oracle/) prints ONE JSON line with the
keys the driver reads and the same `config` object as our arm; under torchrun only rank 0
prints; our arm fails loudly without a GPU (no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

ARGS = ["--impl", "reference", "--seq-len", "16384", "--steps", "1", "--warmup", "0"]


def run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("RANK", None)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module")
def reference_line():
    r = run(ARGS)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_line_keys(reference_line):
    d = reference_line
    assert d["impl"] == "reference"
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["unit"] == "ms" and d["higher_is_better"] is False and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 0
    assert d["ms_per_step"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_config_equals_our_config(reference_line):
    # the driver compares the two arms' `config`: built by the same function from the same workload
    class A:
        workload, gamma, seq_len = "llama3.1-8b-attn-128k", 0.0, 16384
    w = bench.workload_of(A)
    assert reference_line["config"] == bench.bench_config(w, 1, bench.parallelism_of(1, "rows", "sharded"))
    assert reference_line["config"]["seq_len"] == 16384 and reference_line["config"]["preset"] == "llama-16k"


def test_reference_nonzero_rank_is_silent():
    r = run(ARGS, {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == "", (r.stdout, r.stderr[-500:])


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_our_arm_fails_loudly_without_a_gpu():
    r = run(["--seq-len", "16384", "--steps", "1", "--warmup", "0", "--no-cpu", "--no-e2e"], timeout=300)
    assert r.returncode != 0 and r.stdout.strip() == ""
