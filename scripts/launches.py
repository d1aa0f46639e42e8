"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

    python scripts/launches.py launches.csv [n_steps] [excluded_kernel ...]

Excluded kernels (e.g. the dense comparison launch, not part of the step) are listed
but left out of the step share."""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = {}
for r in rows[1:]:
    name = re.sub(r"_ZN2pa\w*?_GLOBAL__N__\w+?_\d+", "", r[ki])
    name = re.sub(r"^.*?::([a-z_0-9]+)\W.*$", r"\1", name.replace("<unnamed>::", ""))[:40]
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
excl = set(sys.argv[3:])
tot = sum(sum(v) for k, v in agg.items() if k not in excl)
print(f"{'kernel':40s} {'launches':>8s} {'mean_us':>10s} {'per_step_us':>12s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:40s} {len(v):8d} {sum(v)/len(v)/1e3:10.1f} {sum(v)/steps/1e3:12.1f} {"  (excl)" if k in excl else f"{sum(v)/tot*100:6.1f}%"}")
