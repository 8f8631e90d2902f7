"""Per-kernel share of ONE SLLOD step in an ncu launch list (--metrics gpu__time_duration.sum --csv):
the launches between two consecutive k_kick_drift_key launches (kick-drift-key, scan, scatter,
rank-gather, pair kernel, reduce), averaged over every complete step window of the list (the bench's
setup launches -- the fluid relaxation, set_state, the e2e calls -- fall outside these windows).
Usage: python scripts/launch_share.py LAUNCHES.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, launches = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "ns": 1.0, "us": 1e3, "ms": 1e6}.get(d.get("Metric Unit", "ns"), 1.0)
        launches.append((d["Kernel Name"].split("(")[0], v))
starts = [i for i, (k, _) in enumerate(launches) if "k_kick_drift_key" in k]
wins = [launches[a:b] for a, b in zip(starts, starts[1:])]
if not wins:
    sys.exit("no complete step window")
tot = {}
for w in wins:
    for k, v in w:
        tot[k] = tot.get(k, 0.0) + v / len(wins)
step = sum(tot.values())
print(f"# {len(wins)} step windows; mean step (serialized, cold) {step / 1e6:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {v / 1e6:9.3f} ms {100 * v / step:6.1f}%")
