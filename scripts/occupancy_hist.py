"""Cell occupancy histogram of a config's bench input (relaxed fluid / lattice) through the library."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1412_3784_b200 import workloads as W
from paper_1412_3784_b200.nemdcell import CellList
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = W.make(k)
q64, _ = bench.relaxed_fluid(w, 'do', k, 'cuda:0')
for name, q in [('fluid', q64.astype(np.float32)), ('lattice', W.positions(w, dtype=np.float32, k=k))]:
    cl = CellList('do', 'f32', rc=w.rc, u_shift=w.ushift, capacity=w.n, max_cells=0); cl.set_box(w.L)
    qt = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    cl.compute_forces(qt)
    st = cl.stats()
    cell_of, cs, dims, wq = cl.cells(len(q), st["ncells"])
    occ = np.diff(cs)
    h = np.bincount(occ)
    tot = occ.sum()
    print(name, 'cells', len(occ), 'mean', occ.mean(), 'frac cells >16: %.4f' % (occ > 16).mean(),
          'frac particles in cells >16: %.4f' % (occ[occ > 16].sum() / tot))
    print(' hist', {i: int(c) for i, c in enumerate(h) if c})
    cl.close()
