"""Force error of the fp32 two-tier evaluation against the fp64 oracle for a given r_split (NC_RSPLIT env,
units of sigma) on C2's relaxed fluid (and its thermalized state after SLLOD steps), plus the pair-kernel
time on C4's relaxed fluid.  Experiment driver, not a test."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import bench
import oracle
from paper_1412_3784_b200 import workloads as W
from paper_1412_3784_b200.nemdcell import CellList

w = W.make(2)
q64, _ = bench.relaxed_fluid(w, 'do', 2, 'cuda:0')
q = q64.astype(np.float32)
p = W.momenta(w, dtype=np.float32, k=2)
# a thermalized state: 400 SLLOD steps at T ~ 1 from the relaxed fluid
cl = CellList('do', 'f32', rc=w.rc, u_shift=w.ushift, capacity=w.n)
kw = dict(L0=w.L0, tstar=w.extra["tstar"])
cl.set_flow(w.A, w.policy, w.t0, **kw)
cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
cl.step(w.dt, 400)
qt = torch.empty((w.n, 3), dtype=torch.float32, device='cuda')
cl.get_state(qt, None)
Lt = W.box_at(w.L0, w.A, w.policy, w.t0 + 400 * w.dt, w.extra)
cl.close()
for name, qq, L in [('relaxed', q, w.L), ('thermal', qt.cpu().numpy(), Lt)]:
    cl = CellList('do', 'f32', rc=w.rc, u_shift=w.ushift, capacity=w.n)
    cl.set_box(L)
    F, U, Wv = cl.compute_forces(torch.from_numpy(np.ascontiguousarray(qq)).cuda())
    F = F.cpu().numpy().astype(np.float64)
    cl.close()
    qo = oracle.wrap(qq, L, 'f32')
    idx = np.random.default_rng(1).choice(w.n, 20000, replace=False)
    r = oracle.evaluate(oracle.DO, qo, L, w.rc, w.eps, w.sigma, w.ushift, idx=idx)
    rms = np.sqrt(np.mean(r.F ** 2))
    err = np.abs(F[idx] - r.F).max()
    print(name, 'rsplit', os.environ.get('NC_RSPLIT', '1.2'), 'max err / rms %.3e (tolerance 2e-5), rms %.3f' % (err / rms, rms), flush=True)
