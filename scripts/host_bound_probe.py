"""Is a small system's SLLOD step bound by the host (enqueue) or by the GPU chain?  One nc_step_sllod
call of K steps without U/W (no synchronization inside): host time of the call vs the time until the
GPU has finished (C0 / C1 / E2-size systems)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_3784_b200 import workloads as W  # noqa: E402
from paper_1412_3784_b200.nemdcell import CellList  # noqa: E402

for k, variant, prec in [(0, "do", "f64"), (1, "do", "f32"), (1, "ds", "f32"), (2, "do", "f32")]:
    w = W.make(k)
    dt_ = np.float32 if prec == "f32" else np.float64
    q = W.positions(w, dtype=dt_, k=k)
    p = W.momenta(w, dtype=dt_, k=k)
    cl = CellList(variant, prec, rc=w.rc, eps=w.eps, sigma=w.sigma, u_shift=w.ushift, capacity=len(q))
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    cl.set_flow(w.A, w.policy, w.t0, **kw)
    cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    cl.step(w.dt, 20)
    torch.cuda.synchronize()
    K = 500
    t0 = time.perf_counter()
    cl.step(w.dt, K, want_uw=False)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"C{k} {variant} {prec}: host enqueue {1e6 * (t1 - t0) / K:.1f} us/step, GPU done {1e6 * (t2 - t0) / K:.1f} us/step",
          flush=True)
    cl.close()
