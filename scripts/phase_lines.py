"""Aggregate scripts/ncu_lines.py output (all lines) into phases given as FILE:A-B=name arguments.
Usage: python scripts/ncu_lines.py REP KERNEL 5000 > lines.txt; python scripts/phase_lines.py lines.txt k3_sparse.cuh:58-98=rows ..."""
import re
import sys

spec = []
for a in sys.argv[2:]:
    fl, name = a.split("=")
    f, rng = fl.split(":")
    lo, hi = map(int, rng.split("-"))
    spec.append((f, lo, hi, name))
ph = {}
for line in open(sys.argv[1]):
    m = re.match(r"(\S+):(\d+)\s+([\d.]+)\s+([\d.]+)\s+([\d.]+)", line)
    if not m:
        continue
    f, ln = m.group(1), int(m.group(2))
    name = next((n for (ff, lo, hi, n) in spec if ff == f and lo <= ln <= hi), f"{f}:other")
    a = ph.setdefault(name, [0.0, 0.0, 0.0])
    for k in range(3):
        a[k] += float(m.group(3 + k))
for k, v in sorted(ph.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} samples {v[0]:6.2f}%  instructions {v[1]:6.2f}%  smem wavefronts {v[2]:6.2f}%")
