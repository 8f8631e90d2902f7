"""Profiling driver: set up config C<k> with one variant on the resident SLLOD
state and run a few steps (the bench's launch configuration).  Used under ncu."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", default="do")
    ap.add_argument("--prec", default="f32")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--input", default="lattice", choices=["lattice", "fluid"])
    ap.add_argument("--pair-kernel", default="auto")
    ap.add_argument("--cache", default="gpurun_out/fluid_cache.npy",
                    help="fluid positions are computed once (run without ncu first) and loaded from here")
    a = ap.parse_args()
    import torch

    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(a.config, scale=a.scale)
    dt = np.float32 if a.prec == "f32" else np.float64
    if a.input == "fluid":
        if os.path.exists(a.cache):
            q = np.load(a.cache).astype(dt)
        else:
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            import bench
            q64, _ = bench.relaxed_fluid(w, a.variant, a.config, "cuda:0")
            np.save(a.cache, q64)
            q = q64.astype(dt)
    else:
        q = W.positions(w, dtype=dt, k=a.config)
    p = W.momenta(w, dtype=dt, k=a.config)
    cl = CellList(a.variant, a.prec, rc=w.rc, u_shift=w.ushift, capacity=w.n, max_cells=0)
    if a.pair_kernel != "auto":
        cl.pair_kernel(a.pair_kernel)
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    cl.set_flow(w.A, w.policy, w.t0, **kw)
    cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    U, Wv = cl.step(w.dt, a.steps)
    torch.cuda.synchronize()
    print("ok", U, cl.stats()["interactions"] / w.n)


if __name__ == "__main__":
    main()
