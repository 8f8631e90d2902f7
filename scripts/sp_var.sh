# A/B of k_pairs_sparse build variants (NC_LIB) on C1/C3, DO and DS
for lib in varlib/*.so; do for c in 3; do for v in do ds; do
NC_LIB=$lib python - <<PY
import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1412_3784_b200 import workloads as W
from paper_1412_3784_b200.nemdcell import CellList
w=W.make($c); q=W.positions(w,dtype=np.float32,k=$c)
cl=CellList('$v','f32',rc=w.rc,u_shift=w.ushift,capacity=w.n); cl.pair_kernel('sparse'); cl.set_box(w.L)
qt=torch.from_numpy(q).cuda()
for _ in range(3): cl.compute_forces(qt)
cl.profile(True)
for _ in range(20): cl.compute_forces(qt)
p=cl.profile_read(); print('$lib c$c $v sparse pairs_ms %.4f' % (p['pairs'][0]/p['pairs'][1]))
PY
done; done; done
