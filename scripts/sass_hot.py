"""Summarize an ncu report: headline metrics + hottest SASS lines (stall samples, instruction counts)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(det.splitlines()))
hdr = rows[0]
want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM", "Registers Per Thread",
        "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Theoretical Occupancy", "Block Limit Shared Mem",
        "Block Limit Registers", "Dynamic Shared Memory Per Block", "Memory Throughput"]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<40} {d['Metric Value']:>20} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(f(d[s]) for d in data) for s in stalls}
print("stalls:", ", ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
ti = sum(f(d["Instructions Executed"]) for d in data)
print(f"total warp instructions {ti:.3e}")
if "--all" in sys.argv:
    for i, d in enumerate(data):
        if f(d["Instructions Executed"]) > ti * 2e-3:
            print(i, d["Source"][:64].ljust(64), f"{f(d['Instructions Executed']):.2e}", d["Avg. Threads Executed"],
                  d["Warp Stall Sampling (All Samples)"])
else:
    for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:ntop]:
        print(d["Source"][:64].ljust(64), f"{f(d['Instructions Executed']):.2e}", d["Avg. Threads Executed"],
              d["Warp Stall Sampling (All Samples)"])
