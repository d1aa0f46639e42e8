"""Per-kernel warp-stall breakdown (ncu PC-sampling counters) from an .ncu-rep:
    python scripts/ncu_stalls.py gpurun_out/x.ncu-rep [kernel-regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "."
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, ti = h.index("Kernel Name"), h.index("gpu__time_duration.sum")
cols = [(i, x[len("smsp__pcsamp_warps_issue_stalled_"):]) for i, x in enumerate(h)
        if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("_not_issued")]
for row in r[2:]:
    if not re.search(pat, row[ki]):
        continue
    vals = []
    for i, n in cols:
        try:
            vals.append((float(row[i].replace(",", "")), n))
        except ValueError:
            pass
    tot = sum(v for v, _ in vals) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(vals, reverse=True)[:7])
    print(f"{row[ki][:48]:48s} {row[ti]:>10s} us  {top}")
