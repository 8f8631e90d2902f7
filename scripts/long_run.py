"""A long SLLOD run of the bench workload (C4: 67,108,864 LJ particles, KR planar elongation, DO,
fp32) through the public API: nsteps steps in chunks, recording U, W, the box and the kinetic
energy every chunk, so a Kraynik-Reinelt remap of the box happens inside the run.
Writes profiles/r01_long_run_c4.json.  Usage: python scripts/long_run.py [nsteps] [chunk]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1412_3784_b200 import workloads as W  # noqa: E402
from paper_1412_3784_b200.nemdcell import CellList  # noqa: E402


def main():
    nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 250
    w = W.make(4)
    q = W.positions(w, dtype=np.float32, k=4)
    p = W.momenta(w, dtype=np.float32, k=4)
    stream = torch.cuda.Stream()
    cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=w.n, stream=stream.cuda_stream)
    cl.set_flow(w.A, "kr", w.t0, L0=w.L0, tstar=w.extra["tstar"])
    qd, pd = torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()
    torch.cuda.synchronize()
    cl.set_state(qd, pd)
    del qd
    rows = []
    po = torch.empty_like(pd)
    t0 = time.perf_counter()
    done = 0
    L_prev = None
    resets = 0
    while done < nsteps:
        k = min(chunk, nsteps - done)
        U, Wv = cl.step(w.dt, k)
        done += k
        n, L, t, _ = cl.get_state(None, po)
        torch.cuda.synchronize()
        ke = 0.5 * float((po.double() ** 2).sum()) / w.mass
        if L_prev is not None and np.abs(np.linalg.solve(L_prev, L) - np.eye(3)).max() > 0.5:
            resets += 1
        L_prev = L.copy()
        rows.append({"step": done, "t": t, "U_per_particle": U / w.n, "KE_per_particle": ke / w.n,
                     "W_diag_per_particle": (np.asarray(Wv)[:3] / w.n).tolist(), "L": L.tolist(),
                     "finite": bool(np.isfinite(U) and np.isfinite(ke))})
        print(json.dumps(rows[-1]), flush=True)
    wall = time.perf_counter() - t0
    cl.close()
    out = {"workload": "C4 (67,108,864 LJ, KR planar, DO, fp32)", "steps": nsteps, "dt": w.dt, "t0": w.t0,
           "tstar": w.extra["tstar"], "box_remaps_inside_run": resets, "wall_s": wall,
           "ms_per_step_wall": 1e3 * wall / nsteps, "samples": rows,
           "note": "SLLOD without a thermostat: the elongational flow heats the system (KE rises); U, W stay "
                   "finite and the box is remapped by the KR automorphism inside the run"}
    path = os.path.join(ROOT, "profiles", "r01_long_run_c4.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "samples"}))


if __name__ == "__main__":
    main()
