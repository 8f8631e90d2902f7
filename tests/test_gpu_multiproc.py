"""Two processes, one GPU: real SlabRank contexts (libnemdcell.so on cuda:0 in each process) exchanging
halo and migration records through torch.distributed gloo with every buffer staged through host memory
(HostStagedTransport: no rank's kernels ever wait on another's on the device), or through the
peer-memory data plane (IpcTransport: the packing kernels write the other process's receive buffers
through CUDA IPC, ordered by interprocess events -- stream waits, no spinning kernels).  Forces, energy, virial
and a short SLLOD run must be BITWISE equal to the single-device path -- the
multi-process slab protocol end to end on the hardware this box has."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _flow_kw(w):
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    return kw


def _worker(rank, P, port, variant, out_dir, dev=False, transport="host"):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList
    from paper_1412_3784_b200.slab import (HostStagedTransport, IpcTransport, SlabRank, SlabRankDev, SlabSystem,
                                           own_particles)

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    full = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    full.set_flow(w.A, w.policy, w.t0, **_flow_kw(w))
    idx = own_particles(full, torch.from_numpy(q).cuda(), rank, P)
    full.close()
    # dev: the host-synchronization-free step (device counts, fixed-capacity messages moved whole)
    sr = (SlabRankDev if dev else SlabRank)(rank, P, variant=variant, prec="f32", rc=w.rc, u_shift=w.ushift,
                                            capacity=len(q), max_cells=4 * len(q) + 4096)
    sr.set_flow(w.A, w.policy, w.t0, **_flow_kw(w))
    sr.load(q[idx], p[idx], idx.astype(np.int32))
    # host: every buffer staged through host memory (gloo); ipc: the packing kernels write the neighbour's
    # receive buffers through CUDA IPC peer memory, ordered by interprocess events (no kernel spins)
    tr = IpcTransport(sr, rank, P) if transport == "ipc" else HostStagedTransport(rank, P)
    sysm = SlabSystem([sr], tr)
    U0, W0, _ = sysm.forces(True)
    out = None
    for _ in range(3):
        out = sysm.step(w.dt, True)
    sysm.flush()
    n = sr.n
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), gid=sr.gid[:n].cpu().numpy(), q=sr.q[:n].cpu().numpy(),
             p=sr.p[:n].cpu().numpy(), U0=U0, W0=W0, U=out[0], W=out[1])
    sr.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dev, transport, P", [(False, "host", 2), (True, "host", 2), (True, "ipc", 2),
                                               (True, "ipc", 3)])
@pytest.mark.parametrize("variant", ["do", "ds"])
def test_two_processes_share_one_gpu_bitwise(variant, dev, transport, P, tmp_path):
    import torch
    import torch.multiprocessing as mp
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    mp.start_processes(_worker, args=(P, _free_port(), variant, str(tmp_path), dev, transport), nprocs=P, join=True,
                       start_method="spawn")
    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    one = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.set_flow(w.A, w.policy, w.t0, **_flow_kw(w))
    one.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    U0, W0 = one.stats()["U"], one.stats()["W"]
    U1, W1 = one.step(w.dt, 3)
    qo = torch.empty((len(q), 3), dtype=torch.float32, device="cuda")
    po = torch.empty_like(qo)
    one.get_state(qo, po)
    one.close()
    qs = np.zeros_like(q)
    ps = np.zeros_like(p)
    seen = np.zeros(len(q), dtype=np.int64)
    for r in range(P):
        d = np.load(tmp_path / f"rank{r}.npz")
        qs[d["gid"]] = d["q"]
        ps[d["gid"]] = d["p"]
        seen[d["gid"]] += 1
        assert float(d["U0"]) == U0 and np.array_equal(d["W0"], W0)
        assert float(d["U"]) == U1 and np.array_equal(d["W"], W1)
    assert np.all(seen == 1)
    assert np.array_equal(qs, qo.cpu().numpy()) and np.array_equal(ps, po.cpu().numpy())
