"""Small systems: GPU time per SLLOD step (one nc_step_sllod call of K steps, no U/W, no events inside)
with each sparse-cell pair kernel choice: C1 (32,000 WCA, LE shear) and the paper's E2 system (1,728 WCA,
uniaxial GKR, scripts/e2_runtime.py's construction).  Run with NC_SP_LPP=1 / 4 to compare the
particle-per-thread kernel's two forms."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_3784_b200 import workloads as W  # noqa: E402
from paper_1412_3784_b200.nemdcell import CellList  # noqa: E402
from scripts.small_kernel_probe_lib import e2  # noqa: E402


tag = os.environ.get("NC_SP_LPP", "auto")
for name, (w, k) in [("C1", (W.make(1), 1)), ("E2", e2())]:
    q = W.positions(w, dtype=np.float32, k=k)
    p = W.momenta(w, dtype=np.float32, k=k)
    for variant in ("do", "ds"):
        for kern in ("segment", "sparse", "rows"):
            cl = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=1 << 17)
            cl.pair_kernel(kern)
            kw = dict(L0=w.L0)
            if w.policy == "gkr":
                kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
            cl.set_flow(w.A, w.policy, w.t0, **kw)
            cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
            cl.step(w.dt if hasattr(w, "dt") else 0.002, 50)
            torch.cuda.synchronize()
            K = 1000
            t0 = time.perf_counter()
            cl.step(0.002, K, want_uw=False)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            U, _ = cl.step(0.002, 1)
            print(f"{name} {variant} {kern:8s} lpp={tag}: {1e6 * (t1 - t0) / K:6.1f} us/step  U={U:.6f}", flush=True)
            cl.close()
