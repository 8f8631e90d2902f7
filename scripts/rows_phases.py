"""Phase split of k_pairs_rows from an ncu report (source lines of csrc/k3_rows.cuh grouped by phase).
Usage: python scripts/rows_phases.py REP.ncu-rep  (line ranges follow the current source)."""
import re
import subprocess
import sys

PH = {"eval (fp64 survivors)": (56, 130), "row data + stencil statistic": (150, 195), "union + row pieces": (195, 269),
      "lane windows": (269, 299), "i setup": (299, 319), "staging": (319, 358), "filter": (358, 394),
      "epilogue + partials": (394, 440)}
out = subprocess.run([sys.executable, "scripts/ncu_lines.py", sys.argv[1], "k_pairs_rowsILb0E", "1000"],
                     capture_output=True, text=True).stdout
agg = {k: [0.0, 0.0] for k in PH}
agg["helpers (kernels.cuh, intrinsics)"] = [0.0, 0.0]
for line in out.splitlines():
    m = re.match(r"(\S+):(\d+)\s+([\d.]+)\s+([\d.]+)", line)
    if not m:
        continue
    f, ln, s, i = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
    k = "helpers (kernels.cuh, intrinsics)"
    if f == "k3_rows.cuh":
        k = next((n for n, (a, b) in PH.items() if a <= ln < b), k)
    elif f == "k3_sparse.cuh":
        k = "eval (fp64 survivors)"
    agg[k][0] += s
    agg[k][1] += i
for k, v in agg.items():
    print(f"{k:<36} stall samples {v[0]:5.1f}%  instructions {v[1]:5.1f}%")
