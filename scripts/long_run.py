"""A long SLLOD run of the bench workload (C4: 67,108,864 LJ particles, KR planar elongation, DO,
fp32) through the public API: nsteps steps in chunks, recording U, W, the box and the kinetic
energy every chunk (and the chunk's device time per step, CUDA events), so a Kraynik-Reinelt remap of
the box happens inside the run.  Usage: python scripts/long_run.py [nsteps] [chunk] [fluid|lattice]
(fluid: BASELINE's relaxed fluid, as bench.py; writes profiles/r02_long_run_c4_<input>.json)."""
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
    kind = sys.argv[3] if len(sys.argv) > 3 else "fluid"
    w = W.make(4)
    if kind == "fluid":
        import bench
        q64, _ = bench.relaxed_fluid(w, "do", 4, "cuda:0")
        q = q64.astype(np.float32)
        del q64
    else:
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
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        U, Wv = cl.step(w.dt, k)
        e1.record(stream)
        e1.synchronize()
        chunk_ms = e0.elapsed_time(e1) / k
        done += k
        n, L, t, _ = cl.get_state(None, po)
        torch.cuda.synchronize()
        ke = 0.5 * float((po.double() ** 2).sum()) / w.mass
        if L_prev is not None and np.abs(np.linalg.solve(L_prev, L) - np.eye(3)).max() > 0.5:
            resets += 1
        L_prev = L.copy()
        rows.append({"step": done, "t": t, "ms_per_step_chunk": chunk_ms, "U_per_particle": U / w.n,
                     "KE_per_particle": ke / w.n,
                     "W_diag_per_particle": (np.asarray(Wv)[:3] / w.n).tolist(), "L": L.tolist(),
                     "finite": bool(np.isfinite(U) and np.isfinite(ke))})
        print(json.dumps(rows[-1]), flush=True)
    wall = time.perf_counter() - t0
    cl.close()
    out = {"workload": "C4 (67,108,864 LJ, KR planar, DO, fp32)", "input": kind, "steps": nsteps, "dt": w.dt,
           "t0": w.t0,
           "tstar": w.extra["tstar"], "box_remaps_inside_run": resets, "wall_s": wall,
           "ms_per_step_wall": 1e3 * wall / nsteps, "samples": rows,
           "note": "SLLOD without a thermostat: the elongational flow heats the system (KE rises); U, W stay "
                   "finite and the box is remapped by the KR automorphism inside the run"}
    out["ms_per_step_device_mean"] = float(np.mean([r["ms_per_step_chunk"] for r in rows]))
    path = os.path.join(ROOT, "profiles", f"r02_long_run_c4_{kind}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "samples"}))


if __name__ == "__main__":
    main()
