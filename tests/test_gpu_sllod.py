"""GPU parity of the SLLOD step (K4 + box update + remap + rebuild) against the
oracle's SLLOD map (reading R19), for the three remap policies of the paper:
Lees-Edwards shear, Kraynik-Reinelt planar elongation
and generalized KR uniaxial / biaxial (reading R23).  Each run
starts just before a remap so that at least one reset happens inside it.

fp64: positions within 1e-9 sigma (modulo the lattice), momenta within 1e-9,
box bit-for-bit (same closed forms, same fp64 sequence); fp32: 1e-4 / 1e-3.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import box as obox
from paper_1412_3784_b200 import workloads as W

pytestmark = pytest.mark.gpu


def run_gpu(w, q, p, prec, variant, dt, nsteps, per_call=None, kernel="auto"):
    """SLLOD on the GPU on a side (non-default) stream: one nc_step_sllod call of nsteps or, with
    per_call = k, nsteps / k calls."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    cl = CellList(variant, prec, rc=w.rc, eps=w.eps, sigma=w.sigma, u_shift=w.ushift, mass=w.mass,
                  capacity=len(q), max_cells=4 * len(q) + 4096, stream=side.cuda_stream)
    cl.pair_kernel(kernel)
    kw = dict(L0=w.L0)
    if w.policy == "kr":
        kw["tstar"] = w.extra["tstar"]
    if w.policy == "gkr":
        kw.update(om1=w.extra["om1"], om2=w.extra["om2"], beta=w.extra["beta"], eps=w.extra["eps"])
    cl.set_flow(w.A, w.policy, w.t0, **kw)
    qd, pd = torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()
    qo = torch.empty_like(qd)
    po = torch.empty_like(qo)
    torch.cuda.synchronize()
    cl.set_state(qd, pd)
    if per_call is None:
        Ugpu, Wgpu = cl.step(dt, nsteps)
    else:
        for _ in range(nsteps // per_call):
            Ugpu, Wgpu = cl.step(dt, per_call)
    n, L, t, gid = cl.get_state(qo, po, want_gid=True)
    side.synchronize()
    cl.close()
    assert np.array_equal(gid, np.arange(len(q)))
    return qo.double().cpu().numpy(), po.double().cpu().numpy(), L, t, Ugpu


def run_oracle(w, q, p, prec, variant, dt, nsteps):
    m = oracle.DS if variant == "ds" else oracle.DO
    b = obox.Box(w.L0, w.A, w.policy, w.t0, om1=w.extra.get("om1"), om2=w.extra.get("om2"),
                 beta=w.extra.get("beta"), tstar=w.extra.get("tstar"), eps=w.extra.get("eps"))
    assert np.array_equal(b.L, w.L) or np.abs(b.L - w.L).max() < 1e-12 * np.abs(w.L).max()
    qd = oracle.wrap(np.asarray(q, dtype=np.float64), b.L, prec)
    pd = np.asarray(p, dtype=np.float64)

    def forces(qq, L):
        r = oracle.evaluate(m, qq, L, w.rc, w.eps, w.sigma, w.ushift, want=("F", "U", "W"))
        return r.F, r.U, r.W

    F, U, _ = forces(qd, b.L)
    resets = 0
    Lprev = b.L.copy()
    for _ in range(nsteps):
        qd, pd, F, U, _ = obox.sllod_step(qd, pd, F, b, dt, forces, mass=w.mass, prec=prec)
        X = np.linalg.solve(Lprev, b.L)
        if np.abs(X - np.eye(3)).max() > 0.5:
            resets += 1
        Lprev = b.L.copy()
    return qd, pd, b.L, b.t, U, resets


def lattice_diff(dq, L):
    """Displacement modulo the lattice: dq - L round(L^-1 dq)."""
    lam = np.linalg.solve(L, dq.T).T
    return dq - np.round(lam) @ L.T


def near_reset(w, nsteps, dt):
    """Move t0 so that a remap happens inside the run."""
    if w.policy == "le":
        eps = w.A[0, 1]
        g0 = w.L0[0, 1] / w.L0[1, 1]
        tx = (0.5 - g0) / eps
        w.t0 = tx - 0.4 * nsteps * dt
    elif w.policy == "kr":
        w.t0 = w.extra["tstar"] - 0.4 * nsteps * dt
    elif w.policy == "gkr":
        rate = np.asarray(w.extra["beta"]) * w.extra["eps"]
        a0 = rate * w.t0
        # next half-integer crossing of either alpha_k after t0
        nxt = [((np.floor(a + 0.5) + 0.5) / r if r > 0 else (np.ceil(a - 0.5) - 0.5) / r) for a, r in zip(a0, rate)]
        w.t0 = min(nxt) - 0.4 * nsteps * dt
    w.L = W.box_at(w.L0, w.A, w.policy, w.t0, w.extra)
    return w


CASES = [
    # (config, scale, flow, prec, variant)
    (1, 2, "uniaxial", "f64", "do"),
    (1, 2, "uniaxial", "f64", "ds"),
    (2, 2, "uniaxial", "f64", "do"),
    (2, 2, "uniaxial", "f64", "ds"),
    (3, 4, "uniaxial", "f64", "do"),
    (3, 4, "biaxial", "f64", "ds"),
    (2, 2, "uniaxial", "f32", "do"),
    (3, 4, "biaxial", "f32", "do"),
    # fp32 on every config / variant pair the fp64 cases cover
    (1, 2, "uniaxial", "f32", "do"),
    (1, 2, "uniaxial", "f32", "ds"),
    (2, 2, "uniaxial", "f32", "ds"),
    (3, 4, "uniaxial", "f32", "do"),
    (3, 4, "biaxial", "f32", "ds"),
]


@pytest.mark.parametrize("k,scale,flow,prec,variant", CASES)
def test_sllod_trajectory(k, scale, flow, prec, variant):
    w = W.make(k, scale=scale, flow=flow)
    nsteps, dt = 20, 0.002
    w = near_reset(w, nsteps, dt)
    dty = np.float64 if prec == "f64" else np.float32
    q = W.positions(w, dtype=dty, k=k)
    p = W.momenta(w, dtype=dty, k=k)
    try:
        oracle.cell_keys(oracle.DO if variant == "do" else oracle.DS, oracle.wrap(q, w.L, prec), w.L, w.rc)
    except ValueError:
        pytest.skip("degenerate grid for this scaled box")
    qg, pg, Lg, tg, Ug = run_gpu(w, q, p, prec, variant, dt, nsteps)
    qo, po, Lo, to, Uo, resets = run_oracle(w, q, p, prec, variant, dt, nsteps)
    assert resets >= 1
    assert tg == pytest.approx(to, abs=1e-12)
    assert np.abs(Lg - Lo).max() <= 1e-13 * np.abs(Lo).max()
    tq, tp = (1e-9, 1e-9) if prec == "f64" else (1e-4, 1e-3)
    assert np.abs(lattice_diff(qg - qo, Lo)).max() < tq
    assert np.abs(pg - po).max() < tp * max(1.0, np.abs(po).max())
    assert Ug == pytest.approx(Uo, rel=1e-9 if prec == "f64" else 1e-5)


def test_gkr_reset_inside_run():
    """C3's seeding puts an alpha_2 half-integer crossing inside the 100-step run (reading R22)."""
    for flow in ("uniaxial", "biaxial"):
        w = W.make(3, flow=flow)
        a0 = w.extra["beta"] * w.extra["eps"] * w.t0
        a1 = w.extra["beta"] * w.extra["eps"] * (w.t0 + w.steps * w.dt)
        m0 = np.floor(a0 + 0.5)
        m1 = np.floor(a1 + 0.5)
        assert (m0 != m1).any()


def test_equilibrium_energy_conservation_gpu():
    """A = 0: SLLOD reduces to velocity Verlet; total energy is conserved (fp64, C0)."""
    w = W.make(0)
    q = W.positions(w, dtype=np.float64, k=0)
    p = W.momenta(w, dtype=np.float64, k=0)
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    cl = CellList("do", "f64", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.set_flow(w.A, "none", 0.0, L0=w.L)
    cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    st = cl.stats()
    E0 = st["U"] + 0.5 * float((p ** 2).sum())
    Es = []
    for _ in range(10):
        U, _ = cl.step(0.002, 20)
        po = torch.empty((len(q), 3), dtype=torch.float64, device="cuda")
        cl.get_state(None, po)
        Es.append(U + 0.5 * float((po ** 2).sum()))
    cl.close()
    assert max(abs(e - E0) for e in Es) < 1e-3 * abs(E0)


@pytest.mark.parametrize("prec,variant", [("f64", "do"), ("f64", "ds"), ("f32", "do")])
def test_sllod_general_flow_lattice_reduction(prec, variant):
    """A general traceless, non-diagonal, non-nilpotent flow (shear plus an elliptic
    part; "general three dimensional linear flows") under the lattice-
    reduction remap policy (NC_REMAP_REDUCE, reading R30): C1's WCA system starting
    from a basis at tilt 0.45, so the reduction (the LE reset) fires inside
    the 20-step run; trajectory and box against the oracle's SLLOD map."""
    w = W.make(1, scale=2)
    a = w.L0[1, 1]
    w.L0 = np.array([[a, 0.45 * a, 0.0], [0.0, a, 0.0], [0.0, 0.0, a]])
    w.A = np.array([[0.0, 2.5, 0.3], [-0.2, 0.0, 0.0], [0.0, 0.4, 0.0]])
    w.policy, w.t0, w.extra = "reduce", 0.0, {}
    w.L = w.L0.copy()
    nsteps, dt = 20, 0.002
    dty = np.float64 if prec == "f64" else np.float32
    q = W.positions(w, dtype=dty, k=1)
    p = W.momenta(w, dtype=dty, k=1)
    qg, pg, Lg, tg, Ug = run_gpu(w, q, p, prec, variant, dt, nsteps)
    qo, po, Lo, to, Uo, resets = run_oracle(w, q, p, prec, variant, dt, nsteps)
    assert resets >= 1
    assert tg == pytest.approx(to, abs=1e-12)
    assert np.abs(Lg - Lo).max() <= 1e-12 * np.abs(Lo).max()
    tq, tp = (1e-9, 1e-9) if prec == "f64" else (1e-4, 1e-3)
    assert np.abs(lattice_diff(qg - qo, Lo)).max() < tq
    assert np.abs(pg - po).max() < tp * max(1.0, np.abs(po).max())
    assert Ug == pytest.approx(Uo, rel=1e-9 if prec == "f64" else 1e-5)



@pytest.mark.parametrize("prec,variant", [("f64", "do"), ("f32", "ds")])
def test_one_call_equals_stepwise(prec, variant):
    """One nc_step_sllod call of 20 steps equals 20 calls of one step bit for bit (C2, KR, a
    remap inside the run): the host-side step state carries nothing between calls."""
    w = W.make(2, scale=2)
    nsteps, dt = 20, 0.002
    w = near_reset(w, nsteps, dt)
    dty = np.float64 if prec == "f64" else np.float32
    q = W.positions(w, dtype=dty, k=2)
    p = W.momenta(w, dtype=dty, k=2)
    a = run_gpu(w, q, p, prec, variant, dt, nsteps)
    b = run_gpu(w, q, p, prec, variant, dt, nsteps, per_call=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2]) and a[3] == b[3] and a[4] == b[4]


def test_deferred_kick_dropped_by_set_state():
    """The closing half kick of a step is held back until the state is read; loading a new state
    in between must discard it (the new momenta are returned untouched)."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(2, scale=2)
    q = W.positions(w, dtype=np.float64, k=2)
    p = W.momenta(w, dtype=np.float64, k=2)
    cl = CellList("do", "f64", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.set_flow(w.A, w.policy, w.t0, L0=w.L0, tstar=w.extra["tstar"])
    qd, pd = torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda()
    cl.set_state(qd, pd)
    cl.step(0.002, 1, want_uw=False)  # leaves a closing kick pending
    cl.set_state(qd, pd)
    po = torch.empty_like(pd)
    cl.get_state(None, po)
    cl.close()
    assert torch.equal(po, pd)


@pytest.mark.parametrize("k,scale,flow,variant", [(1, 1, "uniaxial", "do"), (1, 1, "uniaxial", "ds"),
                                                  (3, 4, "uniaxial", "do"), (3, 4, "biaxial", "ds")])
def test_rows_kernel_trajectory_bitwise_equals_sparse(k, scale, flow, variant):
    """k_pairs_rows gives bitwise k_pairs_sparse's per-particle forces, so whole fp32 SLLOD trajectories
    (Lees-Edwards / generalized KR resets inside the run) are bitwise the same with either kernel."""
    w = near_reset(W.make(k, flow=flow, scale=scale), 20, W.make(k, flow=flow, scale=scale).dt)
    q = W.positions(w, dtype=np.float32, k=k)
    p = W.momenta(w, dtype=np.float32, k=k)
    a = run_gpu(w, q, p, "f32", variant, w.dt, 20, kernel="rows")
    b = run_gpu(w, q, p, "f32", variant, w.dt, 20, kernel="sparse")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
