"""DS vs DO over the Kraynik-Reinelt period (the paper's comparison is a long-run average
over a deformation that "fluctuates tremendously" for DS).

One relaxed fluid of config C<k> (bench.relaxed_fluid: uniform fractional positions + 200 capped
steepest-descent steps through the library), then for each t0 = f t* (f = 0, 1/16, ..., 15/16) the
same fractional coordinates in the box L(t0) (an affine map of the fluid), both variants: a few SLLOD
steps through nc_step_sllod with live per-kernel timing.  Writes one JSON with the per-t0 rows and
the period means.

    python scripts/period_sweep.py [--config 4] [--npts 16] [--steps 4] [--out profiles/r02_period_sweep_c4.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--npts", type=int, default=16)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import bench
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(a.config)
    assert w.policy == "kr"
    tstar = w.extra["tstar"]
    t_relax = time.time()
    qf, fmax = bench.relaxed_fluid(w, "do", a.config, "cuda:0")
    t_relax = time.time() - t_relax
    lam = np.linalg.solve(w.L, qf.T).T  # fractional coordinates of the fluid in its own box
    del qf
    p = W.momenta(w, dtype=np.float32, k=a.config)
    pd = torch.from_numpy(p).cuda()
    rows = []
    for f in np.arange(a.npts) / a.npts:
        t0 = float(f * tstar)
        L = W.box_at(w.L0, w.A, "kr", t0, w.extra)
        q = torch.from_numpy((lam @ L.T).astype(np.float32)).cuda()
        for variant in ("ds", "do"):
            stream = torch.cuda.Stream()
            cl = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=w.n, max_cells=0,
                          stream=stream.cuda_stream)
            cl.set_flow(w.A, "kr", t0, L0=w.L0, tstar=tstar)
            cl.set_state(q, pd)
            cl.step(w.dt, a.warmup, want_uw=False)
            torch.cuda.synchronize()
            cl.profile(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            cl.step(w.dt, a.steps, want_uw=False)
            e1.record(stream)
            e1.synchronize()
            prof = cl.profile_read()
            st = cl.stats()
            cl.profile(False)
            ev = max(st["acc_evals"], 1)
            row = {"t0_over_period": float(f), "variant": variant, "dims": list(st["dims"]),
                   "ms_per_step": e0.elapsed_time(e1) / a.steps,
                   "pairs_ms": prof["pairs"][0] / max(prof["pairs"][1], 1),
                   "candidates_per_particle": st["acc_candidates"] / ev / w.n,
                   "interactions_per_particle": st["acc_interactions"] / ev / w.n,
                   "stencil_mean": st["stencil_cells"] / max(st["ncells"], 1),
                   "pair_kernel": cl.pair_kernel_used()}
            row["pair_interactions_per_s"] = st["acc_interactions"] / ev / 2.0 / (row["ms_per_step"] * 1e-3)
            rows.append(row)
            print(json.dumps(row), flush=True)
            cl.close()
            del stream
        del q
        torch.cuda.empty_cache()
    mean = {}
    for variant in ("ds", "do"):
        r = [x for x in rows if x["variant"] == variant]
        mean[variant] = {k: float(np.mean([x[k] for x in r])) for k in
                         ("ms_per_step", "pairs_ms", "candidates_per_particle", "interactions_per_particle")}
    out = {"config": f"C{a.config}", "n": w.n, "input": "relaxed fluid (bench.relaxed_fluid)",
           "relax_seconds": t_relax, "relax_max_force": fmax, "npts": a.npts, "steps": a.steps, "rows": rows,
           "period_mean": mean,
           "do_over_ds_period_mean_ms_per_step": mean["do"]["ms_per_step"] / mean["ds"]["ms_per_step"],
           "do_over_ds_period_mean_candidates": mean["do"]["candidates_per_particle"] /
                                                mean["ds"]["candidates_per_particle"]}
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}), flush=True)
    path = a.out or os.path.join(ROOT, "profiles", f"r02_period_sweep_c{a.config}.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
