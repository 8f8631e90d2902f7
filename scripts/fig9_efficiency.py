"""NEXT item f1: the paper's search-efficiency study (Fig. 9).

Uniaxial stretching A = diag(0.05, -0.025, -0.025) under the
generalized KR boundary conditions (reading R23), box side a ~ 10 d_cut with
d_cut = (3/(4 pi))^(1/3) so a particle's interaction volume is 1.
Along a long run the library's own geometry (nc_set_flow -> DS counts c_k,
DO counts l_k and the neighborhood-size histogram of every cell, computed by
the same code the force kernel uses) gives the neighborhood volumes

    V_DS = 27 V_box / (c1 c2 c3)                          (Eq. 14)
    V_DO = r11 r22 r33 / (l1 l2 l3) * <neighborhood size>  (Eq. 15)

and the search efficiency 1 / V (interaction volume 1).  The paper
reports long-run means of about 0.0688 (DS) and 0.123 (DO) for the
[dobs14] construction, which is absent here, so they are context, not parity.
Writes profiles/fig9_efficiency.json and a CSV time series.
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", type=float, default=10.0, help="box side in units of d_cut")
    ap.add_argument("--tmax", type=float, default=4000.0)
    ap.add_argument("--samples", type=int, default=20000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fig9_efficiency"))
    args = ap.parse_args()
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList, NcError

    dcut = (3.0 / (4.0 * math.pi)) ** (1.0 / 3.0)
    a = args.a * dcut
    M1, M2, L0, om1, om2 = W.gkr_params(a)
    adiag = np.array([2.0, -1.0, -1.0])          # A = 0.025 diag(2, -1, -1) = diag(0.05, -0.025, -0.025)
    eps = 0.025
    A = np.diag(eps * adiag)
    beta = np.linalg.lstsq(np.stack([om1, om2], axis=1), adiag, rcond=None)[0]
    kw = dict(L0=L0, om1=om1, om2=om2, beta=beta, eps=eps)
    cls = {v: CellList(v, "f64", rc=dcut, capacity=16, max_cells=1 << 20) for v in ("ds", "do")}
    ts = np.linspace(0.0, args.tmax, args.samples, endpoint=False)
    rows = []
    degenerate = {"ds": 0, "do": 0}
    for t in ts:
        row = {"t": float(t)}
        for v, cl in cls.items():
            try:
                cl.set_flow(A, "gkr", float(t), **kw)
            except NcError:
                degenerate[v] += 1
                row[v] = None
                continue
            hist = cl.stencil_histogram()
            n_cells = int(hist.sum())
            mean_count = float((hist * np.arange(64)).sum() / n_cells)
            Lb = W.box_at(L0, A, "gkr", float(t), {"beta": beta, "eps": eps, "om1": om1, "om2": om2})
            Vbox = abs(np.linalg.det(Lb))
            # the cell count is the histogram total: V_cell = V_box / n_cells for both variants
            V = Vbox / n_cells * mean_count
            row[v] = {"V": V, "eff": 1.0 / V, "cells": n_cells, "mean_count": mean_count,
                      "hist": {int(k): int(hist[k]) for k in np.nonzero(hist)[0]}}
        rows.append(row)
    out = {"a_over_dcut": args.a, "dcut": dcut, "A": A.tolist(), "tmax": args.tmax, "samples": args.samples,
           "degenerate_samples": degenerate}
    for v in ("ds", "do"):
        Vs = np.array([r[v]["V"] for r in rows if r[v] is not None])
        out[v] = {"mean_V": float(Vs.mean()), "efficiency_of_mean_V": float(1.0 / Vs.mean()),
                  "mean_efficiency": float(np.mean(1.0 / Vs)), "min_V": float(Vs.min()), "max_V": float(Vs.max())}
    out["paper_P745"] = {"ds": 0.0688, "do": 0.123, "note": "context only: [dobs14] construction and Fig. 9 data absent"}
    out["equilibrium_P699"] = (4.0 / 3.0 * math.pi) / 27.0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out + ".json", "w"), indent=1)
    with open(args.out + ".csv", "w") as f:
        f.write("t,V_ds,V_do,cells_ds,cells_do,mean_count_do\n")
        for r in rows[:: max(1, len(rows) // 2000)]:
            ds, do = r["ds"], r["do"]
            f.write(f"{r['t']},{ds['V'] if ds else ''},{do['V'] if do else ''},{ds['cells'] if ds else ''},"
                    f"{do['cells'] if do else ''},{do['mean_count'] if do else ''}\n")
    print(json.dumps({k: out[k] for k in ("ds", "do", "degenerate_samples", "paper_P745")}))
    for cl in cls.values():
        cl.close()


if __name__ == "__main__":
    main()
