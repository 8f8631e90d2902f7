# C4 pair-kernel time (library event profile) on the relaxed fluid and the lattice, DO and DS
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1412_3784_b200 import workloads as W
from paper_1412_3784_b200.nemdcell import CellList
w = W.make(4)
q64, _ = bench.relaxed_fluid(w, 'do', 4, 'cuda:0')
for name, q in [('fluid', q64.astype(np.float32)), ('lattice', W.positions(w, dtype=np.float32, k=4))]:
    for v in ('do', 'ds'):
        cl = CellList(v, 'f32', rc=w.rc, u_shift=w.ushift, capacity=w.n, max_cells=0); cl.set_box(w.L)
        qt = torch.from_numpy(np.ascontiguousarray(q)).cuda()
        for _ in range(2): cl.compute_forces(qt)
        cl.profile(True)
        for _ in range(5): cl.compute_forces(qt)
        p = cl.profile_read(); print('C4', name, v, 'pairs_ms %.3f' % (p['pairs'][0] / p['pairs'][1]), flush=True)
        cl.close()
PY
