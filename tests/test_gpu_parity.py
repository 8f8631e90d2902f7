"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north star):
  * cell assignments, cell contents (cell_start) and wrapped positions: bit-exact
  * pair sets: bit-exact (per-particle digests over (gid_j, image n))
  * fp64: max |dF| <= 1e-12 RMS(F), |dU|/|U| <= 1e-12, max |dW| <= 1e-12 max|W|
  * fp32: max |dF| <= 2e-5 RMS(F), |dU|/|U| <= 1e-6, max |dW| <= 1e-6 max|W|
"""
import numpy as np
import pytest

import oracle
from tests.helpers import inputs, oracle_side

pytestmark = pytest.mark.gpu

TOL = {"f64": (1e-12, 1e-12, 1e-12), "f32": (2e-5, 1e-6, 1e-6)}
VAR = {"ds": oracle.DS, "do": oracle.DO}


def gpu_eval(w, q, variant, prec, digest=True, kernel="auto"):
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    cl = CellList(variant, prec, rc=w.rc, eps=w.eps, sigma=w.sigma, u_shift=w.ushift, capacity=max(1, len(q)))
    cl.pair_kernel(kernel)
    cl.set_box(w.L)
    qt = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    F, U, W = cl.compute_forces(qt)
    torch.cuda.synchronize()
    counts = cl.pair_counts(len(q))  # per-particle counts from the TIMED kernel (before any digest run)
    used = cl.pair_kernel_used()
    if kernel != "auto":
        assert used == kernel, (used, kernel)
    st = cl.stats()
    cell_of, cs, dims, wq = cl.cells(len(q), st["ncells"])
    gids = cl.cell_gids(len(q))
    dig = cl.digest(len(q)) if digest else None
    out = dict(F=F.double().cpu().numpy(), U=U, W=W, stats=st, cell_of=cell_of, cs=cs, dims=dims, wq=wq, dig=dig,
               hist=cl.stencil_histogram(), launches=cl.launches(), kernel=used, counts=counts, gids=gids)
    cl.close()
    return out


def check_against_oracle(w, q, variant, prec, idx=None, kernel="auto"):
    g = gpu_eval(w, q, variant, prec, kernel=kernel)
    qo = oracle_side(q, w.L, prec)
    # wrapped positions: bit-exact (same stored values)
    assert np.array_equal(g["wq"].astype(np.float64), qo)
    # cells: bit-exact
    cell, nh, dims = oracle.cell_keys(VAR[variant], qo, w.L, w.rc)
    assert list(g["dims"]) == list(dims)
    assert np.array_equal(g["cell_of"], cell)
    cs, order = oracle.cell_sort(cell, int(np.prod(dims.astype(np.int64))))
    assert np.array_equal(g["cs"], cs)
    # cell contents: the gid sequence of the counting sort, (cell, gid) order (R27), bit-exact
    assert np.array_equal(g["gids"], order)
    # stencil histogram: exact
    hist, _ = oracle.stencil_histogram(VAR[variant], w.L, w.rc)
    assert np.array_equal(g["hist"], hist)
    # pair sets + forces
    r = oracle.evaluate(VAR[variant], qo, w.L, w.rc, w.eps, w.sigma, w.ushift, idx=idx)
    cnt, hs, hx = g["dig"]
    sel = slice(None) if idx is None else idx
    assert np.array_equal(cnt[sel], r.cnt)
    # the timed kernel's own membership decisions (all tiers), not only the digest instantiation's
    assert np.array_equal(g["counts"][sel], r.cnt)
    assert np.array_equal(hs[sel], r.hsum)
    assert np.array_equal(hx[sel], r.hxor)
    tF, tU, tW = TOL[prec]
    Fo = r.F
    rms = np.sqrt(np.mean(Fo ** 2))
    err = np.abs(g["F"][sel] - Fo).max()
    assert err <= tF * rms, (err, rms, err / rms)
    if idx is None:
        assert abs(g["U"] - r.U) <= tU * abs(r.U), (g["U"], r.U)
        assert np.abs(g["W"] - r.W).max() <= tW * np.abs(r.W).max()
        assert g["stats"]["candidates"] == r.candidates
        assert g["stats"]["interactions"] == r.interactions
    return g, r


@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c0_equilibrium_fp64_vs_brute_force(variant):
    w, q = inputs(0, "f64")
    g, r = check_against_oracle(w, q, variant, "f64")
    b = oracle.evaluate(oracle.BRUTE, oracle_side(q, w.L, "f64"), w.L, w.rc)
    assert np.array_equal(b.cnt, r.cnt) and np.array_equal(b.hsum, r.hsum)
    # equilibrium: every neighborhood has 27 cells
    assert g["hist"][27] == np.prod(g["dims"])


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c1_shear(variant, prec):
    w, q = inputs(1, prec)
    check_against_oracle(w, q, variant, prec)


@pytest.mark.parametrize("kernel", ["cell", "segment", "sparse", "rows"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c1_both_pair_kernels(variant, kernel):
    """Sparse WCA cells (C1, ~1.3 per cell): the warp-per-cell, the row-segment and the
    particle-per-thread pair kernels each reproduce the oracle's pair set and forces."""
    w, q = inputs(1, "f32")
    g, _ = check_against_oracle(w, q, variant, "f32", kernel=kernel)
    assert g["kernel"] == kernel


@pytest.mark.parametrize("kernel", ["sparse", "rows"])
@pytest.mark.parametrize("scale", [3, 4])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_sparse_kernel_tiny_grid_many_rows_per_warp(variant, scale, kernel):
    """k_pairs_sparse on a tiny WCA grid (C1 scaled to 7-10 cells a side, ~9-13 particles a cell
    row): a warp's 32 particles span 3-5 cell rows, so most lanes build their own row data instead of
    reading the warp's two shared rows -- both paths must give the oracle's pair set and forces."""
    w, q = inputs(1, "f32", scale=scale)
    g, _ = check_against_oracle(w, q, variant, "f32", kernel=kernel)
    assert g["kernel"] == kernel
    dims = g["dims"]
    assert 32 > 2 * dims[0] * 1.0  # rows of < 16 cells: a warp spans >= 3 cell rows


@pytest.mark.parametrize("kernel", ["segment", "sparse", "rows"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_segment_kernel_on_dense_lj_cells(variant, kernel):
    """The sparse-cell kernels forced onto dense LJ cells (~13 per cell; the segment kernel's
    staged union overflows for long segments and must shrink them, the particle-per-thread
    kernel's queues flush often): both still match the oracle."""
    w, q = inputs(2, "f32", scale=2)
    check_against_oracle(w, q, variant, "f32", kernel=kernel)


@pytest.mark.parametrize("kernel", ["segment", "sparse", "rows"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_segment_kernel_deterministic_and_equal_pair_set(kernel, variant):
    w, q = inputs(3, "f32", scale=2)
    a = gpu_eval(w, q, variant, "f32", kernel=kernel)
    b = gpu_eval(w, q, variant, "f32", kernel=kernel)
    c = gpu_eval(w, q, variant, "f32", kernel="cell")
    assert np.array_equal(a["F"], b["F"]) and a["U"] == b["U"] and np.array_equal(a["W"], b["W"])
    for x, y in zip(a["dig"], c["dig"]):
        assert np.array_equal(x, y)
    assert a["stats"]["candidates"] == c["stats"]["candidates"]
    assert a["stats"]["stencil_cells"] == c["stats"]["stencil_cells"]
    assert np.abs(a["F"] - c["F"]).max() <= 2e-5 * np.sqrt(np.mean(c["F"] ** 2))


def test_pair_kernel_option_errors():
    from paper_1412_3784_b200.nemdcell import CellList, NcError

    cl = CellList("do", "f64", rc=2.5, capacity=16)
    with pytest.raises(NcError, match="NC_E_ARG"):
        cl.pair_kernel("segment")
    cl.pair_kernel("sparse")  # NC_F64 has a particle-per-thread kernel too (k_pairs_sparse64)
    with pytest.raises(NcError, match="NC_E_ARG"):
        cl.pair_kernel("rows")
    with pytest.raises(NcError, match="NC_E_ARG"):
        cl.pair_kernel(7)
    cl.close()


@pytest.mark.parametrize("variant", ["ds", "do"])
@pytest.mark.parametrize("t0", [0.3, 2.0, 5.0, 9.0])
def test_kr_boxes_scaled(variant, t0):
    from paper_1412_3784_b200 import workloads as W

    w, q = inputs(2, "f32", scale=2)
    w.L = W.box_at(w.L0, w.A, "kr", t0, w.extra)
    q = W.positions(w, dtype=np.float32, k=2)
    try:
        oracle.cell_keys(VAR[variant], oracle_side(q, w.L, "f32"), w.L, w.rc)
    except ValueError:
        pytest.skip("degenerate grid at this t0 for the scaled box")
    check_against_oracle(w, q, variant, "f32")


@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c2_full(variant):
    w, q = inputs(2, "f32")
    check_against_oracle(w, q, variant, "f32")


@pytest.mark.parametrize("flow", ["uniaxial", "biaxial"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c3_gkr_full(variant, flow):
    w, q = inputs(3, "f32", flow=flow)
    check_against_oracle(w, q, variant, "f32")


@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c3_fp64(variant):
    w, q = inputs(3, "f64", scale=2)
    check_against_oracle(w, q, variant, "f64")


def test_ds_equals_do_pair_set():
    w, q = inputs(2, "f32")
    a = gpu_eval(w, q, "ds", "f32")
    b = gpu_eval(w, q, "do", "f32")
    for x, y in zip(a["dig"], b["dig"]):
        assert np.array_equal(x, y)
    assert np.abs(a["F"] - b["F"]).max() < 1e-4 * np.sqrt(np.mean(a["F"] ** 2))


def test_deterministic_bitwise():
    w, q = inputs(2, "f32")
    a = gpu_eval(w, q, "do", "f32", digest=False)
    b = gpu_eval(w, q, "do", "f32", digest=False)
    assert np.array_equal(a["F"], b["F"]) and a["U"] == b["U"] and np.array_equal(a["W"], b["W"])


def test_wrap_of_outside_positions():
    """Positions far outside Omega are wrapped by the same rule on both sides."""
    w, q = inputs(1, "f64", scale=2)
    rng = np.random.default_rng(5)
    shift = rng.integers(-3, 4, size=(len(q), 3)) @ w.L.T
    q2 = q + shift
    check_against_oracle(w, q2, "do", "f64")


def test_edge_cases():
    import torch
    from paper_1412_3784_b200.nemdcell import CellList, NcError

    cl = CellList("do", "f32", rc=2.5, capacity=16)
    L = np.eye(3) * 12.0
    cl.set_box(L)
    # empty input
    q = torch.zeros((0, 3), dtype=torch.float32, device="cuda")
    F, U, W = cl.compute_forces(q)
    assert U == 0.0 and np.all(W == 0)
    # single particle: no self interaction
    q = torch.tensor([[1.0, 2.0, 3.0]], device="cuda")
    F, U, W = cl.compute_forces(q)
    assert U == 0.0 and torch.all(F == 0)
    # two particles across the periodic boundary
    q = torch.tensor([[0.2, 5.0, 5.0], [11.5, 5.0, 5.0]], device="cuda")
    F, U, W = cl.compute_forces(q)
    assert F[0, 0] > 0 and F[1, 0] < 0
    # errors
    with pytest.raises(NcError, match="NC_E_DEGENERATE"):
        cl.set_box(np.eye(3) * 9.0)
    with pytest.raises(NcError, match="NC_E_BOX"):
        cl.set_box(np.diag([12.0, 12.0, -12.0]))
    with pytest.raises(NcError, match="NC_E_FLOW"):
        cl.set_flow(np.diag([0.1, 0.1, 0.1]), "none", 0.0, L0=L)
    with pytest.raises(NcError, match="NC_E_OOM"):
        cl.compute_forces(torch.zeros((17, 3), device="cuda"))
    cl.close()


def test_host_pointers_e2e():
    """The ABI accepts host (numpy) buffers and copies through device staging."""
    w, q = inputs(1, "f32", scale=2)
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.set_box(w.L)
    Fh, Uh, Wh = cl.compute_forces(np.ascontiguousarray(q))
    Fd, Ud, Wd = cl.compute_forces(torch.from_numpy(q).cuda())
    assert np.array_equal(Fh, Fd.cpu().numpy()) and Uh == Ud
    cl.close()


@pytest.mark.parametrize("variant", ["ds", "do"])
def test_c4_full_size_sampled(variant):
    """BASELINE configs[4] at full size (67M particles), in the bench's launch
    configuration: cells exact on a sample, digests and forces on a sample."""
    w, q = inputs(4, "f32")
    rng = np.random.default_rng(44)
    idx = np.sort(rng.choice(len(q), size=2000, replace=False))
    g = gpu_eval(w, q, variant, "f32")
    qo = oracle_side(q, w.L, "f32")
    assert np.array_equal(g["wq"].astype(np.float64), qo)
    cell, nh, dims = oracle.cell_keys(VAR[variant], qo, w.L, w.rc)
    assert np.array_equal(g["cell_of"], cell)
    r = oracle.evaluate(VAR[variant], qo, w.L, w.rc, w.eps, w.sigma, w.ushift, idx=idx)
    cnt, hs, hx = g["dig"]
    assert np.array_equal(cnt[idx], r.cnt) and np.array_equal(hs[idx], r.hsum) and np.array_equal(hx[idx], r.hxor)
    rms = np.sqrt(np.mean(g["F"] ** 2))
    assert np.abs(g["F"][idx] - r.F).max() <= 2e-5 * rms
    # Newton's third law over the whole system
    assert np.abs(g["F"].sum(axis=0)).max() < 1e-3 * rms * np.sqrt(len(q))


def _cluster_workload(prec):
    """A sheared box (L = 14 sigma, l = 5 DO cells per side) holding a dense jittered cube of 9^3 = 729
    particles at spacing 0.4 sigma next to 400 uniformly spread ones: cells of ~150-300 particles
    (staging in several chunks, i-batches of 32 with one stream, survivors queued well past the
    close-tier queue), beside ordinary cells.  Seeded; no physics intended."""
    from paper_1412_3784_b200 import workloads as W

    rng = W.rng_for(90, 0)
    L = np.array([[14.0, 3.1, 0.0], [0.0, 14.0, 0.0], [0.0, 0.0, 14.0]])
    g = np.arange(9) * 0.4
    cube = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 4.3
    cube += rng.uniform(-0.04, 0.04, cube.shape)
    lam = rng.uniform(0.0, 1.0, (400, 3))
    q = np.concatenate([cube, lam @ L.T]).astype(np.float32 if prec == "f32" else np.float64)
    w = W.Workload(name="cluster", n=len(q), L0=L, A=np.zeros((3, 3)), policy="none", t0=0.0, L=L, rc=2.5)
    return w, q


@pytest.mark.parametrize("variant", ["ds", "do"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_dense_cluster_stress(variant, prec):
    """Overcrowded cells: pair sets bit-exact and forces within the bars through the multi-chunk,
    one-stream and queue-flush paths of k_pairs (and of the fp64 kernel)."""
    w, q = _cluster_workload(prec)
    g, r = check_against_oracle(w, q, variant, prec, kernel="cell")
    assert r.interactions > 100000  # the cluster really is dense


def test_tier_counting_mode():
    """nc_profile mode 3 runs k_pairs' counting instantiation: the fp32-tier share of the
    interactions is reported, the results equal the plain kernel's bit for bit, and fp64 /
    sparse-cell (all-fp64) evaluations report no fp32-tier interactions."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w, q = inputs(2, "f32", scale=2)
    qt = torch.from_numpy(q).cuda()
    cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.set_box(w.L)
    F0, U0, W0 = cl.compute_forces(qt)
    cl.profile(3)
    F1, U1, W1 = cl.compute_forces(qt)
    st = cl.stats()
    cl.profile(False)
    cl.close()
    assert torch.equal(F0, F1) and U0 == U1 and np.array_equal(W0, W1)
    assert 0.5 * st["interactions"] < st["interactions_fp32"] < st["interactions"]
    assert st["acc_interactions_fp32"] == st["interactions_fp32"]
    for prec, k in (("f64", 2), ("f32", 1)):
        w, q = inputs(k, prec, scale=2)
        cl = CellList("do", prec, rc=w.rc, u_shift=w.ushift, capacity=len(q))
        cl.set_box(w.L)
        cl.profile(3)
        cl.compute_forces(torch.from_numpy(q).cuda())
        st = cl.stats()
        cl.profile(False)
        cl.close()
        assert st["interactions"] > 0 and st["interactions_fp32"] == 0


def test_async_host_pipeline_equals_sync():
    """nc_compute_forces_async on pinned host buffers (copies on the library's streams, double-
    buffered) gives the synchronous call's forces bit for bit, for several calls in flight, and
    nc_compute_sync returns the last call's U and W."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList, NcError

    w, q = inputs(2, "f32", scale=2)
    cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.set_box(w.L)
    F0, U0, W0 = cl.compute_forces(q)
    qs = [torch.from_numpy(q + np.float32(0.01 * k)).pin_memory() for k in range(3)]
    Fs = [torch.empty_like(x).pin_memory() for x in qs]
    for x, f in zip(qs, Fs):
        cl.compute_forces_async(x, f)
    U2, W2 = cl.compute_sync()
    for k, (x, f) in enumerate(zip(qs, Fs)):
        Fk, Uk, Wk = cl.compute_forces(x.numpy())
        assert np.array_equal(Fk, f.numpy()), k
    assert U2 == Uk and np.array_equal(W2, Wk)
    with pytest.raises(NcError, match="NC_E_STATE"):
        cl.compute_sync()
    with pytest.raises(NcError, match="NC_E_ARG"):
        cl.compute_forces_async(torch.from_numpy(q).cuda(), torch.empty((len(q), 3), device="cuda"))
    cl.close()


def _minimal_grid_workload(prec, tilt):
    """A sheared box at the smallest grids the variants allow (R9): DO l = (4, 4, 3), DS c = (4, 4, 3)
    at tilt 0, fewer DS columns when tilted; a jittered 9 x 9 x 7 simple-cubic lattice (567
    particles, min distance ~0.9 sigma).  Every stencil wraps onto itself through the periodic
    images; seeded."""
    from paper_1412_3784_b200 import workloads as W

    rng = W.rng_for(91, 0)
    L = np.array([[10.6, tilt * 10.6, 0.0], [0.0, 10.6, 0.0], [0.0, 0.0, 8.1]])
    g = np.stack(np.meshgrid(np.arange(9) / 9, np.arange(9) / 9, np.arange(7) / 7, indexing="ij"), -1).reshape(-1, 3)
    lam = g + rng.uniform(-0.02, 0.02, g.shape)
    q = (lam @ L.T).astype(np.float32 if prec == "f32" else np.float64)
    w = W.Workload(name="minimal", n=len(q), L0=L, A=np.zeros((3, 3)), policy="none", t0=0.0, L=L, rc=2.5)
    return w, q


@pytest.mark.parametrize("variant", ["ds", "do"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("tilt", [0.0, 0.45])
def test_minimal_grids(variant, prec, tilt):
    """Parity at the smallest legal grids, where neighbor cells are reached through several
    periodic images (pair sets bit-exact, forces within the bars)."""
    w, q = _minimal_grid_workload(prec, tilt)
    try:
        oracle.cell_keys(VAR[variant], oracle.wrap(q.astype(np.float64), w.L, prec), w.L, w.rc)
    except ValueError:
        pytest.skip("degenerate grid for this variant and tilt")
    check_against_oracle(w, q, variant, prec)


@pytest.mark.parametrize("kernel", ["cell", "segment", "sparse", "rows"])
def test_user_order_force_output_host_device_async_agree(kernel):
    """The pair kernels write F straight into the caller's order (no unsort pass): device q / F, host
    q / F (staged) and the pipelined host-buffer calls give bitwise the same F, in the caller's own
    (shuffled) order."""
    import torch
    from paper_1412_3784_b200.nemdcell import CellList

    w, q = inputs(1, "f32")
    perm = np.random.default_rng(7).permutation(len(q))
    qs = np.ascontiguousarray(q[perm])  # a random caller order
    cl = CellList("do", "f32", rc=w.rc, u_shift=w.ushift, capacity=len(q))
    cl.pair_kernel(kernel)
    cl.set_box(w.L)
    Fd, Ud, Wd = cl.compute_forces(torch.from_numpy(qs).cuda())
    Fh, Uh, Wh = cl.compute_forces(qs)
    qp = torch.from_numpy(qs).pin_memory()
    Fa = [torch.empty((len(q), 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    cl.compute_forces_async(qp, Fa[0])
    cl.compute_forces_async(qp, Fa[1])
    Ua, Wa = cl.compute_sync()
    Fo, _, _ = cl.compute_forces(torch.from_numpy(np.ascontiguousarray(q)).cuda())  # the original order
    cl.close()
    Fd = Fd.cpu().numpy()
    assert np.array_equal(Fd, Fh) and np.array_equal(Fd, Fa[0].numpy()) and np.array_equal(Fd, Fa[1].numpy())
    assert Ud == Uh == Ua and np.array_equal(Wd, Wh) and np.array_equal(Wd, Wa)
    # F follows the particles (within-cell order follows the caller's indices: the fp64 sums may
    # differ in their last bits before the fp32 rounding)
    Fo = Fo.cpu().numpy()[perm]
    assert np.abs(Fd - Fo).max() <= 1e-6 * np.sqrt(np.mean(Fo ** 2))


@pytest.mark.parametrize("cfg, scale", [(1, 1), (3, 4), (3, 2)])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_rows_kernel_bitwise_equals_sparse_kernel(cfg, scale, variant):
    """k_pairs_rows evaluates every lane's candidates in k_pairs_sparse's order with its fp64
    arithmetic: per-particle forces, counts and pair digests are bitwise equal; U and W differ only
    by the block partition of their fixed-order sums."""
    w, q = inputs(cfg, "f32", scale=scale)
    a = gpu_eval(w, q, variant, "f32", kernel="rows")
    b = gpu_eval(w, q, variant, "f32", kernel="sparse")
    assert np.array_equal(a["F"], b["F"])
    for x, y in zip(a["dig"], b["dig"]):
        assert np.array_equal(x, y)
    for k in ("candidates", "interactions", "stencil_cells", "rechecks"):
        assert a["stats"][k] == b["stats"][k], k
    assert abs(a["U"] - b["U"]) <= 1e-12 * abs(b["U"])


@pytest.mark.parametrize("cfg, scale", [(1, 1), (1, 3), (3, 4), (0, 1)])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_sparse_kernel_fp64(cfg, scale, variant):
    """NC_F64 on the particle-per-thread kernel (k_pairs_sparse64): the canonical fp64 test on every
    candidate and error-free displacements, as the warp-per-cell kernel, mapped one thread per particle --
    the oracle's cells, pair set (bit-exact), candidate counts and forces within 1e-12 RMS(F); C0's dense
    LJ cells included (long stencil rows, frequent queue flushes)."""
    w, q = inputs(cfg, "f64", scale=scale)
    g, _ = check_against_oracle(w, q, variant, "f64", kernel="sparse")
    assert g["kernel"] == "sparse"
    c = gpu_eval(w, q, variant, "f64", kernel="cell")
    assert g["stats"]["candidates"] == c["stats"]["candidates"]
    assert g["stats"]["stencil_cells"] == c["stats"]["stencil_cells"]
