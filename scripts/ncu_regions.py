"""Split the SASS of one profiled kernel into regions of similar execution count
and print instruction and stall-sample shares.  Usage: ncu_regions.py REP [min_pct]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
minpct = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def fl(x):
    try:
        return float(x)
    except Exception:
        return 0.0


tot = sum(fl(d['Instructions Executed']) for d in data)
regs = []
cur = None
for i, d in enumerate(data):
    ie = fl(d['Instructions Executed'])
    key = round(ie / 1e6) if ie > 0 else 0
    if cur is None or abs(key - cur[1]) > max(2, 0.03 * cur[1]):
        cur = [i, key, 0, 0, 0]
        regs.append(cur)
    cur[2] += ie
    cur[3] += fl(d['Warp Stall Sampling (All Samples)'])
    cur[4] = i
samp = sum(r[3] for r in regs)
for r in regs:
    if r[2] > minpct / 100 * tot or r[3] > minpct / 100 * samp:
        print(f"lines {r[0]}-{r[4]} exec/line~{r[1]}M  inst {r[2]:.2e} ({r[2] / tot * 100:.1f}%)  samples {r[3] / samp * 100:.1f}%")
