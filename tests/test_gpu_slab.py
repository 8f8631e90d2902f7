"""Slab decomposition on one GPU in loopback mode (P slabs in one process, buffers
moved by device copies): forces, energy, virial and SLLOD trajectories must be
BITWISE equal to the single-device path."""
import numpy as np
import pytest

from paper_1412_3784_b200 import workloads as W

pytestmark = pytest.mark.gpu


def flow_kw(w):
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    return kw


def make_system(w, q, p, P, variant, prec, dev=False):
    """dev: the host-synchronization-free step (SlabRankDev: device counts, fixed-capacity messages)."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList
    from paper_1412_3784_b200.slab import LoopbackTransport, SlabRank, SlabRankDev, SlabSystem, own_particles

    full = CellList(variant, prec, rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=4 * len(q) + 4096)
    full.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    ranks = []
    for r in range(P):
        idx = own_particles(full, q, r, P)
        sr = (SlabRankDev if dev else SlabRank)(r, P, variant=variant, prec=prec, rc=w.rc, u_shift=w.ushift,
                                                capacity=len(q), max_cells=4 * len(q) + 4096)
        sr.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
        sr.load(q[idx], p[idx], idx.astype(np.int32))
        ranks.append(sr)
    full.close()
    return SlabSystem(ranks, LoopbackTransport())


def gather_state(system, n, dtype):
    system.flush()  # deferred closing kicks
    q = np.zeros((n, 3), dtype=dtype)
    p = np.zeros((n, 3), dtype=dtype)
    F = np.zeros((n, 3), dtype=dtype)
    seen = np.zeros(n, dtype=np.int64)
    for r in system.ranks:
        g = r.gid[:r.n].cpu().numpy()
        q[g] = r.q[:r.n].cpu().numpy()
        p[g] = r.p[:r.n].cpu().numpy()
        F[g] = r.F[:r.n].cpu().numpy()
        seen[g] += 1
    assert np.all(seen == 1), "every particle on exactly one rank"
    return q, p, F


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("variant", ["do", "ds"])
@pytest.mark.parametrize("dev", [False, True])
def test_slab_forces_bitwise(P, variant, dev):
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(2, scale=2)           # 32768 LJ particles, KR box
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    one = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    F1, U1, W1 = one.compute_forces(torch.from_numpy(q).cuda())
    st1 = one.stats()
    one.close()
    sysm = make_system(w, q, p, P, variant, "f32", dev=dev)
    U, Wv, st = sysm.forces(True)
    _, _, F = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(F, F1.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    assert st["interactions"] == st1["interactions"] and st["candidates"] == st1["candidates"]
    for r in sysm.ranks:
        r.close()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("dev", [False, True])
def test_slab_sllod_bitwise(P, dev):
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    one = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    one.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    U1, W1 = one.step(w.dt, 5)
    qo = torch.empty((len(q), 3), dtype=torch.float32, device="cuda")
    po = torch.empty_like(qo)
    one.get_state(qo, po)
    one.close()
    sysm = make_system(w, q, p, P, "do", "f32", dev=dev)
    sysm.forces(False)
    out = None
    for _ in range(5):
        out = sysm.step(w.dt, True)
    U, Wv, _ = out
    qs, ps, _ = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(qs, qo.cpu().numpy()) and np.array_equal(ps, po.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    for r in sysm.ranks:
        r.close()


@pytest.mark.parametrize("kernel", ["auto", "segment"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("variant", ["do", "ds"])
@pytest.mark.parametrize("dev", [False, True])
def test_slab_forces_bitwise_sparse_cells(P, variant, dev, kernel):
    """Sparse WCA cells (C1, ~1.3 per cell): every rank and the single device run the same pair kernel
    -- AUTO's choice (a function of the grid: the particle-per-thread kernel with two threads per particle
    on C1's 24k cells) or the row-segment kernel; forces, U, W and counts stay bitwise equal."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(1)
    q = W.positions(w, dtype=np.float32, k=1)
    p = W.momenta(w, dtype=np.float32, k=1)
    one = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.pair_kernel(kernel)
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    F1, U1, W1 = one.compute_forces(torch.from_numpy(q).cuda())
    st1 = one.stats()
    used = one.pair_kernel_used()
    assert used == ("sparse" if kernel == "auto" else kernel)
    one.close()
    sysm = make_system(w, q, p, P, variant, "f32", dev=dev)
    for r in sysm.ranks:
        r.cl.pair_kernel(kernel)
    U, Wv, st = sysm.forces(True)
    assert all(r.cl.pair_kernel_used() == used for r in sysm.ranks)
    _, _, F = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(F, F1.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    assert st["interactions"] == st1["interactions"] and st["candidates"] == st1["candidates"]
    for r in sysm.ranks:
        r.close()


@pytest.mark.parametrize("dev", [False, True])
@pytest.mark.parametrize("variant", ["do", "ds"])
def test_nccl_data_plane_self_ring_bitwise(variant, dev):
    """The library's NCCL data plane (nc_slab_comm_init / nc_slab_exchange* / nc_slab_allgather) on a
    one-rank communicator: the ring neighbours are the rank itself, so every exchange and the
    all-gather run through NCCL on one GPU; forces and an SLLOD run stay bitwise equal to the
    single-device path."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList
    from paper_1412_3784_b200.slab import NcclTransport, SlabRank, SlabRankDev, SlabSystem

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    one = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    one.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    F1 = torch.empty((len(q), 3), dtype=torch.float32, device="cuda")
    U0, W0 = one.stats()["U"], one.stats()["W"]
    U1, W1 = one.step(w.dt, 3)
    qo = torch.empty((len(q), 3), dtype=torch.float32, device="cuda")
    po = torch.empty_like(qo)
    one.get_state(qo, po)
    one.close()
    sr = (SlabRankDev if dev else SlabRank)(0, 1, variant=variant, prec="f32", rc=w.rc, u_shift=w.ushift,
                                            capacity=len(q), max_cells=4 * len(q) + 4096)
    sr.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    sr.load(q, p, np.arange(len(q), dtype=np.int32))
    sysm = SlabSystem([sr], NcclTransport(sr, 0, 1))
    Uf, Wf, _ = sysm.forces(True)
    assert Uf == U0 and np.array_equal(Wf, W0)
    out = None
    for _ in range(3):
        out = sysm.step(w.dt, True)
    qs, ps, _ = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(qs, qo.cpu().numpy()) and np.array_equal(ps, po.cpu().numpy())
    assert out[0] == U1 and np.array_equal(out[1], W1)
    sr.close()


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("variant", ["do", "ds"])
@pytest.mark.parametrize("dev", [False, True])
def test_slab_repartition_when_l3_changes(P, variant, dev):
    """Generalized KR (uniaxial, fast strain): the cell-layer count l3 changes inside the run (the box
    stretches along v3 and a GKR reset remaps it), so slab ownership is recomputed and particles move
    by many layers (SlabSystem.repartition); the trajectory stays bitwise that of one device."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(3, scale=4)  # 32768 WCA particles, GKR box
    w.A = w.A * 20.0        # eps = 2: several l3 changes within 12 steps
    w.extra = dict(w.extra, eps=w.extra["eps"] * 20.0)
    w.t0 = 0.01
    w.L = W.box_at(w.L0, w.A, w.policy, w.t0, w.extra)
    q = W.positions(w, dtype=np.float32, k=3)
    p = W.momenta(w, dtype=np.float32, k=3)
    nsteps = 12
    one = CellList(variant, "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=4 * len(q) + 4096)
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    one.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    l3s = [one.stats()["dims"][2]]
    for _ in range(nsteps):
        U1, W1 = one.step(w.dt, 1)
        l3s.append(one.stats()["dims"][2])
    qo = torch.empty((len(q), 3), dtype=torch.float32, device="cuda")
    po = torch.empty_like(qo)
    one.get_state(qo, po)
    one.close()
    assert len(set(l3s)) > 1, l3s  # the layer count really changes
    sysm = make_system(w, q, p, P, variant, "f32", dev=dev)
    sysm.forces(False)
    for _ in range(nsteps):
        out = sysm.step(w.dt, True)
    assert sysm.repartitions >= 1
    qs, ps, _ = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(qs, qo.cpu().numpy()) and np.array_equal(ps, po.cpu().numpy())
    assert out[0] == U1 and np.array_equal(out[1], W1)
    for r in sysm.ranks:
        r.close()


@pytest.mark.parametrize("kernel", ["sparse", "rows"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("dev", [False, True])
def test_slab_forces_bitwise_particle_per_thread_kernel(P, dev, kernel):
    """The particle-per-thread sparse kernel (NC_PK_SPARSE) on every rank and on one device: its
    block partials are fixed particle ranges of one layer, so U and W stay bitwise P-invariant."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(1)
    q = W.positions(w, dtype=np.float32, k=1)
    p = W.momenta(w, dtype=np.float32, k=1)
    one = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.pair_kernel(kernel)
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    F1, U1, W1 = one.compute_forces(torch.from_numpy(q).cuda())
    st1 = one.stats()
    one.close()
    sysm = make_system(w, q, p, P, "do", "f32", dev=dev)
    for r in sysm.ranks:
        r.cl.pair_kernel(kernel)
    U, Wv, st = sysm.forces(True)
    assert all(r.cl.pair_kernel_used() == kernel for r in sysm.ranks)
    _, _, F = gather_state(sysm, len(q), np.float32)
    assert np.array_equal(F, F1.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    assert st["interactions"] == st1["interactions"] and st["candidates"] == st1["candidates"]
    for r in sysm.ranks:
        r.close()


def test_device_count_step_reads_nothing_back():
    """The host-synchronization-free step: steps and force evaluations without energies issue no
    device-to-host read from the Python side (torch's sync debug mode raises on one), the library side
    never synchronizes either (its only synchronizing calls are nc_sd_status and a forces_end with
    parts); the count read afterwards matches the particles."""
    import torch

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    sysm = make_system(w, q, p, 3, "do", "f32", dev=True)
    sysm.forces(False)
    torch.cuda.set_sync_debug_mode("error")
    try:
        for _ in range(4):
            sysm.step(w.dt, False)
    finally:
        torch.cuda.set_sync_debug_mode("default")
    assert sum(r.n for r in sysm.ranks) == len(q)
    assert all(r.status()[1] == 0 for r in sysm.ranks)
    for r in sysm.ranks:
        r.close()


def test_device_count_message_overflow_is_flagged():
    """A halo message smaller than the boundary layer: the excess is dropped (never written out of
    bounds) and nc_sd_status reports NC_E_OOM."""
    from paper_1412_3784_b200.nemdcell import NcError
    from paper_1412_3784_b200.slab import LoopbackTransport, SlabRankDev, SlabSystem, own_particles
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float32, k=2)
    p = W.momenta(w, dtype=np.float32, k=2)
    full = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=4 * len(q) + 4096)
    full.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    ranks = []
    for r in range(2):
        idx = own_particles(full, q, r, 2)
        sr = SlabRankDev(r, 2, variant="do", prec="f32", rc=w.rc, u_shift=w.ushift, capacity=len(q), hcap=64,
                         max_cells=4 * len(q) + 4096)
        sr.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
        sr.load(q[idx], p[idx], idx.astype(np.int32))
        ranks.append(sr)
    full.close()
    sysm = SlabSystem(ranks, LoopbackTransport())
    sysm.forces(False)
    with pytest.raises(NcError, match="NC_E_OOM"):
        ranks[0].status()
    for r in ranks:
        r.close()


@pytest.mark.parametrize("dev", [False, True])
@pytest.mark.parametrize("variant", ["do", "ds"])
def test_slab_fp64_forces_and_steps_bitwise(variant, dev):
    """NC_F64 through the slab paths (host-count and host-synchronization-free): C2 scaled to 32,768 LJ
    particles in its KR box, P = 2: forces, U, W and 3 SLLOD steps bitwise equal to one device."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float64, k=2)
    p = W.momenta(w, dtype=np.float64, k=2)
    one = CellList(variant, "f64", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    F1, U1, W1 = one.compute_forces(torch.from_numpy(q).cuda())
    one.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    Us, Ws = one.step(w.dt, 3)
    qo = torch.empty((len(q), 3), dtype=torch.float64, device="cuda")
    po = torch.empty_like(qo)
    one.get_state(qo, po)
    one.close()
    sysm = make_system(w, q, p, 2, variant, "f64", dev=dev)
    U, Wv, _ = sysm.forces(True)
    _, _, F = gather_state(sysm, len(q), np.float64)
    assert np.array_equal(F, F1.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    out = None
    for _ in range(3):
        out = sysm.step(w.dt, True)
    qs, ps, _ = gather_state(sysm, len(q), np.float64)
    assert np.array_equal(qs, qo.cpu().numpy()) and np.array_equal(ps, po.cpu().numpy())
    assert out[0] == Us and np.array_equal(out[1], Ws)
    for r in sysm.ranks:
        r.close()


@pytest.mark.parametrize("P", [2, 3])
def test_slab_forces_bitwise_fp64_sparse_kernel(P):
    """NC_F64 on the particle-per-thread kernel (k_pairs_sparse64) on every rank and on one device:
    F, U and W bitwise P-invariant (block partials are fixed particle ranges of one layer)."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(1, scale=2)
    q = W.positions(w, dtype=np.float64, k=1)
    p = W.momenta(w, dtype=np.float64, k=1)
    one = CellList("do", "f64", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    one.pair_kernel("sparse")
    one.set_flow(w.A, w.policy, w.t0, **flow_kw(w))
    F1, U1, W1 = one.compute_forces(torch.from_numpy(q).cuda())
    assert one.pair_kernel_used() == "sparse"
    one.close()
    sysm = make_system(w, q, p, P, "do", "f64")
    for r in sysm.ranks:
        r.cl.pair_kernel("sparse")
    U, Wv, st = sysm.forces(True)
    assert all(r.cl.pair_kernel_used() == "sparse" for r in sysm.ranks)
    _, _, F = gather_state(sysm, len(q), np.float64)
    assert np.array_equal(F, F1.cpu().numpy())
    assert U == U1 and np.array_equal(Wv, W1)
    for r in sysm.ranks:
        r.close()
