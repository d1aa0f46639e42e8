"""Per-kernel SASS instruction counts of the built library (tcgen05 / TMA evidence).

    cuobjdump -sass paper_2509_24745_b200/libproxyattn.so > /tmp/sass.txt
    python scripts/sass_summary.py /tmp/sass.txt > profiles/r01_sass_summary.txt
"""
import re
import subprocess
import sys

PAT = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "MUFU.EX2", "HMMA"]
txt = open(sys.argv[1]).read()
rows = []
for s in re.split(r"\n\s*Function : ", txt)[1:]:
    name = s.split("\n", 1)[0].strip()
    c = [len(re.findall(r"\b" + re.escape(p), s)) for p in PAT]
    if any(c):
        rows.append((name, c))
dem = subprocess.run(["c++filt"], input="\n".join(n for n, _ in rows), capture_output=True,
                     text=True).stdout.split("\n")
print("# SASS of paper_2509_24745_b200/libproxyattn.so (cuobjdump -sass, sm_100a), per kernel")
print("# template instantiation: tcgen05 (UTCHMMA, UTCBAR, TMEM LDTM / STTM), TMA (UTMALDG),")
print("# MUFU.EX2; HMMA = legacy mma.sync.  scripts/sass_summary.py.")
print("%-44s %s" % ("kernel<template args>", " ".join("%8s" % p for p in PAT)))
for (n, c), d in sorted(zip(rows, dem), key=lambda x: x[1]):
    d = d.replace("(anonymous namespace)::", "").replace("pa::", "").replace("void ", "")
    d = re.sub(r"\(.*\)$", "", d)
    d = re.sub(r"__nv_bfloat16", "bf16", d)
    print("%-44s %s" % (d[:44], " ".join("%8d" % x for x in c)))
