"""A few SLLOD steps of a small system (for an ncu launch list): C1 DO (AUTO kernel) or the E2 system."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_3784_b200 import workloads as W  # noqa: E402
from paper_1412_3784_b200.nemdcell import CellList  # noqa: E402
from scripts.small_kernel_probe_lib import e2  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "C1"
w, k = (W.make(1), 1) if which == "C1" else e2()
q = W.positions(w, dtype=np.float32, k=k)
p = W.momenta(w, dtype=np.float32, k=k)
cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=1 << 17)
kw = dict(L0=w.L0)
if w.policy == "gkr":
    kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
cl.set_flow(w.A, w.policy, w.t0, **kw)
cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
cl.step(0.002, 10)
torch.cuda.synchronize()
