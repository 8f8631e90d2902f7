"""Aggregate an ncu SASS source page by CUDA source line.

ncu's CSV export of the CUDA view carries no metrics, so this maps each SASS address of the profiled
kernel to its source line with `nvdisasm -g` of a cubin compiled from the same sources and flags
(compile it from the tree that built the profiled library).

Usage: python scripts/ncu_lines.py REP.ncu-rep KERNEL_SUBSTRING [ntop] [--cubin PATH]
Prints the source lines with the most stall samples: samples %, warp instructions, shared-memory
wavefronts, and the line text.
"""
import csv
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def build_cubin(path):
    sys.path.insert(0, ROOT)
    from paper_1412_3784_b200 import build as b
    flags = [f for f in b.NVCC_FLAGS if f not in ("-shared",)]
    # drop linker-only options
    out, skip = [], False
    for f in flags:
        if skip:
            skip = False
            continue
        if f in ("-cudart", "-Xlinker"):
            skip = True
            continue
        out.append(f)
    subprocess.check_call([b.NVCC, *out, "-cubin", *b.SOURCES, "-o", path])


def line_map(cubin, kname):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
    start = None
    for i, l in enumerate(txt):
        if l.strip().startswith(".section") and ".text." in l and kname in l:
            start = i
            break
    if start is None:
        sys.exit(f"kernel {kname} not in {cubin}")
    cur, m = None, {}
    for l in txt[start + 1:]:
        if l.strip().startswith(".section") and ".text." in l:
            break
        g = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if g:
            cur = (os.path.basename(g.group(1)), int(g.group(2)))
        a = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if a and cur:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    ntop = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else 40
    cubin = "/tmp/ncu_lines.cubin"
    if "--cubin" in sys.argv:
        cubin = sys.argv[sys.argv.index("--cubin") + 1]
    else:
        build_cubin(cubin)
    lm = line_map(cubin, kname)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    agg = {}
    for d in data:
        key = lm.get(int(d["Address"], 16) - base, ("?", 0))
        s = agg.setdefault(key, [0.0, 0.0, 0.0])
        s[0] += f(d["Warp Stall Sampling (All Samples)"])
        s[1] += f(d["Instructions Executed"])
        s[2] += f(d.get("L1 Wavefronts Shared", 0))
    tot = [sum(v[i] for v in agg.values()) or 1.0 for i in range(3)]
    files = {}
    for fn, _ in agg:
        p = os.path.join(ROOT, "paper_1412_3784_b200", "csrc", fn)
        if fn not in files and os.path.exists(p):
            files[fn] = open(p).read().split("\n")
    print(f"# {rep}: samples {tot[0]:.0f}, warp instructions {tot[1]:.3e}, shared wavefronts {tot[2]:.3e}")
    print(f"{'file:line':<22}{'samp%':>7}{'inst%':>7}{'wf%':>7}  source")
    for (fn, ln), v in sorted(agg.items(), key=lambda x: -x[1][0])[:ntop]:
        text = files.get(fn, [""] * (ln + 1))[ln - 1].strip() if ln else ""
        print(f"{fn + ':' + str(ln):<22}{v[0] / tot[0] * 100:7.2f}{v[1] / tot[1] * 100:7.2f}{v[2] / tot[2] * 100:7.2f}  {text[:90]}")


if __name__ == "__main__":
    main()
