"""Summarize nvcc -Xptxas=-v output: kernel, registers, spill bytes (reads stdin)."""
import re
import subprocess
import sys

cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "spill" not in cur:
        cur["spill"] = (int(m.group(2)), int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m and "regs" not in cur:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True, text=True).stdout.split("\n")
for r, n in zip(rows, names):
    n = re.sub(r"\(.*", "", n)
    if len(sys.argv) > 1 and not re.search(sys.argv[1], n):
        continue
    print(f"{n:60s} regs {r.get('regs')} spill st/ld {r.get('spill')}")
