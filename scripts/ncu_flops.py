"""Executed floating-point work of one profiled kernel, counted from its SASS.

ncu's sm__sass_thread_inst_executed_op_{ffma,fadd,fmul}_pred_on counters do not count the packed
FFMA2 / FADD2 / FMUL2 instructions k_pairs is built on (they read 0), so this sums the
"Predicated-On Thread Instructions Executed" column of the SASS source page per opcode:
FFMA2 = 4 flop, FADD2 / FMUL2 = 2, FFMA / DFMA = 2, FADD / FMUL / DADD / DMUL = 1 per thread.
Prints fp32 and fp64 executed flop, their rates over the kernel duration, and the FP32 / FP64
peaks at the measured SM clock (148 SMs x 128 FP32 lanes x 2, FP64 at half that).

Usage: python scripts/ncu_flops.py REP.ncu-rep
"""
import csv
import re
import subprocess
import sys

FLOP = {"FFMA2": (4, 32), "FADD2": (2, 32), "FMUL2": (2, 32), "FFMA": (2, 32), "FADD": (1, 32), "FMUL": (1, 32),
        "DFMA": (2, 64), "DADD": (1, 64), "DMUL": (1, 64),
        # tensor cores: HMMA.1684 (mma.sync m16n8k4 tf32) = 2 x 16 x 8 x 4 = 1024 flop per warp instruction,
        # i.e. 32 per predicated-on thread
        "HMMA": (32, 19)}


def main(rep):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hdr = rows[1]
    tot = {32: 0.0, 64: 0.0, 19: 0.0}
    per = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9]+)(\.[A-Z0-9.]+)?\s", d["Source"] + " ")
        if not m or m.group(1) not in FLOP:
            continue
        try:
            n = float(d["Predicated-On Thread Instructions Executed"])
        except ValueError:
            continue
        f, bits = FLOP[m.group(1)]
        tot[bits] += f * n
        per[m.group(1)] = per.get(m.group(1), 0.0) + f * n
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    dd = dict(zip(rr[0], rr[2]))
    dur = float(dd["gpu__time_duration.sum"].replace(",", ""))
    unit = rr[1][rr[0].index("gpu__time_duration.sum")]
    sec = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(unit, 1e-9)
    clk = float(dd["sm__cycles_elapsed.avg.per_second"].replace(",", ""))
    cu = rr[1][rr[0].index("sm__cycles_elapsed.avg.per_second")]
    hz = clk * {"Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6, "hz": 1.0}.get(cu, 1e9)
    p32 = 148 * 128 * 2 * hz
    print(f"duration {sec * 1e3:.4f} ms, SM clock {hz / 1e6:.0f} MHz")
    for k in sorted(per, key=lambda k: -per[k]):
        print(f"  {k:<6} {per[k]:.4e} flop")
    for bits, peak in ((32, p32), (64, p32 / 2)):
        rate = tot[bits] / sec
        print(f"fp{bits}: {tot[bits]:.4e} flop executed, {rate / 1e12:.2f} TFLOP/s = {rate / peak:.3f} of "
              f"{peak / 1e12:.1f}")
    if tot[19]:
        # dense tf32 tensor peak: half the bf16 one (B200_PROFILING: 2.25 PFLOP/s bf16 nominal)
        rate = tot[19] / sec
        print(f"tf32 (tensor cores): {tot[19]:.4e} flop executed, {rate / 1e12:.2f} TFLOP/s = {rate / 1.125e15:.4f} "
              f"of the nominal 1125 TFLOP/s dense tf32")


if __name__ == "__main__":
    main(sys.argv[1])
