#!/bin/bash
# A/B of k_pairs builds (varlib/*.so via NC_LIB) on C4 DO, relaxed fluid (cached once): pair-kernel ms
python scripts/prof_step.py --config 4 --input fluid --cache gpurun_out/fluid_c4.npy --steps 1 > /dev/null 2>&1
for rep in 1 2; do for lib in varlib/*.so; do
NC_LIB=$lib python - <<PY
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1412_3784_b200 import workloads as W
from paper_1412_3784_b200.nemdcell import CellList
w = W.make(${CFG:-4})
q = np.load('gpurun_out/fluid_c4.npy').astype(np.float32)
cl = CellList('${V:-do}', 'f32', rc=w.rc, u_shift=w.ushift, capacity=w.n, max_cells=0); cl.set_box(w.L)
qt = torch.from_numpy(np.ascontiguousarray(q)).cuda()
for _ in range(2): cl.compute_forces(qt)
cl.profile(True)
for _ in range(5): cl.compute_forces(qt)
p = cl.profile_read(); print('$lib', 'pairs_ms %.3f' % (p['pairs'][0] / p['pairs'][1]), flush=True)
cl.close()
PY
done; done
rm -f gpurun_out/fluid_c4.npy
