"""GPU parity at the edges of the method (SPEC acceptance S:637 as a test idea):

* full (i, j, n) pair lists across the C-ABI (nc_get_pairs) against the oracle's list, on tiny
  random deformed boxes, C0 and C1;
* >= 10^4 pairs placed EXACTLY on the cutoff, one grid step inside / outside it and at
  r_c (1 +- 1e-6), across lattice images, in tilted LE, KR and GKR boxes, fp32 and fp64, DS and DO,
  both pair kernels: digests of the digest instantiation AND per-particle counts of the timed kernel
  equal the oracle's; the canonical fp64 band test really runs (rechecks > 0);
* r_c^2 moved by k ulp around those exact squares (fp64): the strict inequality at the last bit;
* a truncated stencil (one neighborhood entry dropped) must FAIL these checks (negative control);
* pair sets every step of an SLLOD run with Lees-Edwards resets.
"""
import numpy as np
import pytest

import oracle
from tests import edges
from tests.helpers import inputs, oracle_side

pytestmark = pytest.mark.gpu

VAR = {"ds": oracle.DS, "do": oracle.DO}


def _cl(variant, prec, rc, n, sigma=1.0, u_shift=0.0, kernel="auto"):
    from paper_1412_3784_b200.nemdcell import CellList

    cl = CellList(variant, prec, rc=rc, sigma=sigma, u_shift=u_shift, capacity=max(1, n))
    cl.pair_kernel(kernel)
    return cl


def _eval(cl, L, q, prec):
    """One timed evaluation, then its per-particle counts, stored state, digests and stats."""
    import torch

    cl.set_box(L)
    dt = torch.float32 if prec == "f32" else torch.float64
    cl.compute_forces(torch.from_numpy(np.ascontiguousarray(q)).to(dt).cuda())
    counts = cl.pair_counts(len(q))
    st = cl.stats()
    _, _, _, wq = cl.cells(len(q), st["ncells"])
    dig = cl.digest(len(q))
    return counts, wq.astype(np.float64), dig, st


# ----------------------------------------------------------------- full pair lists


@pytest.mark.parametrize("variant", ["ds", "do"])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_full_pair_lists_tiny_random_boxes(variant, prec):
    rng = np.random.default_rng([1412, 3784, 91])
    for trial in range(4):
        while True:
            L = 9.0 * (np.eye(3) + rng.uniform(-0.35, 0.35, size=(3, 3)))
            if np.linalg.det(L) > 0.4 * 9.0 ** 3:
                break
        rc = 0.9 * min(min(oracle.heights(L)) / 3.05, oracle.qr(L)[1][0, 0] / 4.05, oracle.qr(L)[1][1, 1] / 4.05,
                       oracle.qr(L)[1][2, 2] / 3.05)
        q = (rng.uniform(0, 1, size=(300, 3)) @ L.T).astype(np.float32 if prec == "f32" else np.float64)
        cl = _cl(variant, prec, rc, len(q), sigma=0.3)
        _, wq, _, _ = _eval(cl, L, q, prec)
        got = cl.pairs(1 << 16)
        cl.close()
        ref = oracle.evaluate(oracle.BRUTE, wq, L, rc, 1.0, 0.3, 0.0, pairs_cap=1 << 16).pairs
        assert len(got) > 100 and np.array_equal(got, ref), (trial, len(got), len(ref))


@pytest.mark.parametrize("k, prec, variant", [(0, "f64", "ds"), (0, "f64", "do"), (1, "f32", "do"),
                                              (1, "f32", "ds"), (1, "f64", "do")])
def test_full_pair_lists_c0_c1(k, prec, variant):
    """C0 (4,000 LJ, brute force) and C1 (32,000 WCA, tilted LE box): every ordered (i, j, n)."""
    w, q = inputs(k, prec)
    cl = _cl(variant, prec, w.rc, len(q), sigma=w.sigma, u_shift=w.ushift)
    _, wq, _, _ = _eval(cl, w.L, q, prec)
    got = cl.pairs(1 << 22)
    cl.close()
    method = oracle.BRUTE if k == 0 else VAR[variant]
    ref = oracle.evaluate(method, wq, w.L, w.rc, w.eps, w.sigma, w.ushift, pairs_cap=1 << 22).pairs
    assert np.array_equal(got, ref), (len(got), len(ref))
    # symmetric under (i, j, n) <-> (j, i, -n) (the pair set of a lattice)
    sw = np.stack([got[:, 1], got[:, 0], -got[:, 2], -got[:, 3], -got[:, 4]], axis=1)
    sw = sw[np.lexsort(sw.T[::-1])]
    assert np.array_equal(sw, got)


def test_pair_list_cap_reports_the_count():
    from paper_1412_3784_b200.nemdcell import NcError

    w, q = inputs(0, "f64")
    cl = _cl("do", "f64", w.rc, len(q), u_shift=w.ushift)
    _eval(cl, w.L, q, "f64")
    with pytest.raises(NcError) as e:
        cl.pairs(10)
    cl.close()
    assert "NC_E_OOM" in str(e.value)


# ----------------------------------------------------------------- pairs on the cutoff


def _edge_case(kind, prec, variant, kernel):
    # the sparse-cell kernel gets the same pairs in a box 8x the volume (~2 particles per cell, its regime)
    a = 20.0 if kernel in ("segment", "sparse", "rows") else 10.0
    L, rc, q, d0 = edges.edge_pairs(kind, npairs=6000, seed={"le": 1, "kr": 2, "gkr": 3}[kind], a=a)
    qs = q.astype(np.float32 if prec == "f32" else np.float64)
    cl = _cl(variant, prec, rc, len(qs), sigma=0.1, kernel=kernel)
    counts, wq, (cnt, hs, hx), st = _eval(cl, L, qs, prec)
    cl.close()
    r = oracle.evaluate(VAR[variant], wq, L, rc, 1.0, 0.1, 0.0)
    # the stored pairs: how many sit exactly on / within 1e-5 of the cutoff
    d = wq[1::2] - wq[0::2]
    d = d - np.round(np.linalg.solve(L, d.T).T) @ L.T
    r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    return r, counts, cnt, hs, hx, st, np.sum(r2 == rc * rc), np.sum(np.abs(r2 / (rc * rc) - 1.0) < 1e-5)


@pytest.mark.parametrize("kind", ["le", "kr", "gkr"])
@pytest.mark.parametrize("prec, variant, kernel", [("f32", "do", "cell"), ("f32", "ds", "cell"),
                                                   ("f32", "do", "segment"), ("f32", "ds", "segment"),
                                                   ("f32", "do", "sparse"), ("f32", "ds", "sparse"),
                                                   ("f32", "do", "rows"), ("f32", "ds", "rows"),
                                                   ("f64", "do", "cell"), ("f64", "ds", "cell"),
                                                   ("f64", "do", "sparse"), ("f64", "ds", "sparse")])
def test_pairs_on_the_cutoff(kind, prec, variant, kernel):
    r, counts, cnt, hs, hx, st, n_on, n_edge = _edge_case(kind, prec, variant, kernel)
    assert 2 * n_edge >= 10000 and n_on >= 200  # >= 10^4 ordered pairs at the edge, hundreds exactly on it
    assert np.array_equal(cnt, r.cnt) and np.array_equal(hs, r.hsum) and np.array_equal(hx, r.hxor)
    assert np.array_equal(counts, r.cnt)  # the timed kernel's own membership decisions
    assert st["interactions"] == r.interactions and st["candidates"] == r.candidates
    if prec == "f32":  # (NC_F64 runs the canonical test on every candidate: no separate re-checks)
        assert st["rechecks"] > 0  # the canonical fp64 test decided the pairs on the cutoff


@pytest.mark.parametrize("kernel", ["cell", "sparse"])
@pytest.mark.parametrize("variant", ["ds", "do"])
def test_cutoff_at_the_last_bit_fp64(variant, kernel):
    """r_c^2 = X0 + k ulp(X0) around the exact squares X0 of the constructed pairs: pairs at r^2 = X0
    are inside for k > 0 and outside for k <= 0, decided by the canonical fp64 comparison."""
    L, rc0, q, d0 = edges.edge_pairs("le", npairs=3000, seed=4)
    X0 = rc0 * rc0
    seen = {}
    for k in range(-6, 7):
        rc = edges.rc_with_square(X0, k)
        if rc is None:
            continue
        cl = _cl(variant, "f64", rc, len(q), sigma=0.1, kernel=kernel)
        counts, wq, (cnt, hs, hx), st = _eval(cl, L, q, "f64")
        cl.close()
        r = oracle.evaluate(VAR[variant], wq, L, rc, 1.0, 0.1, 0.0)
        assert np.array_equal(cnt, r.cnt) and np.array_equal(hs, r.hsum) and np.array_equal(counts, r.cnt)
        seen[k] = r.interactions
    ks = sorted(seen)
    assert ks[0] <= 0 < ks[-1], ks  # r_c^2 landed on both sides of the exact squares
    # pairs at r^2 = X0 are out for r_c^2 <= X0 and in above: the count jumps between k <= 0 and k > 0
    assert max(seen[k] for k in ks if k <= 0) < min(seen[k] for k in ks if k > 0), seen


@pytest.mark.parametrize("prec, kernel", [("f32", "cell"), ("f32", "segment"), ("f32", "sparse"), ("f32", "rows"),
                                          ("f64", "cell"), ("f64", "sparse")])
def test_truncated_stencil_is_caught(prec, kernel):
    """Negative control: with the last entry of every neighborhood dropped (nc_debug), the same
    checks must fail -- the parity tests can see a missing stencil cell."""
    L, rc, q, _ = edges.edge_pairs("le", npairs=3000, seed=5)
    qs = q.astype(np.float32 if prec == "f32" else np.float64)
    cl = _cl("do", prec, rc, len(qs), sigma=0.1, kernel=kernel)
    cl.debug_drop_entries(True)
    counts, wq, (cnt, hs, hx), st = _eval(cl, L, qs, prec)
    cl.close()
    r = oracle.evaluate(oracle.DO, wq, L, rc, 1.0, 0.1, 0.0)
    assert not np.array_equal(cnt, r.cnt) and not np.array_equal(counts, r.cnt)
    assert st["candidates"] < r.candidates and st["interactions"] < r.interactions


# ----------------------------------------------------------------- pair sets along a trajectory


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_pair_sets_every_sllod_step(prec):
    """P5: an LE SLLOD run through two Lees-Edwards resets; after EVERY step the pair set of the
    state the GPU holds equals the oracle's on that state (digests and the timed kernel's counts)."""
    import torch
    from paper_1412_3784_b200 import workloads as W
    from paper_1412_3784_b200.nemdcell import CellList

    w = W.make(1, scale=2)
    w.A = np.zeros((3, 3))
    w.A[0, 1] = 2.0  # fast shear: resets inside a short run
    g0 = w.L0[0, 1] / w.L0[1, 1]
    w.t0 = (0.5 - g0) / 2.0 - 0.01
    w.L = W.box_at(w.L0, w.A, "le", w.t0, w.extra)
    dt = np.float32 if prec == "f32" else np.float64
    q = W.positions(w, dtype=dt, k=1)
    p = W.momenta(w, dtype=dt, k=1)
    cl = CellList("do", prec, rc=w.rc, u_shift=w.ushift, capacity=len(q), max_cells=4 * len(q) + 4096)
    cl.set_flow(w.A, "le", w.t0, L0=w.L0)
    cl.set_state(torch.from_numpy(q).cuda(), torch.from_numpy(p).cuda())
    gammas = []
    for step in range(12):
        cl.step(0.002, 1)
        counts = cl.pair_counts(len(q))
        st = cl.stats()
        _, _, _, wq = cl.cells(len(q), st["ncells"])
        cnt, hs, hx = cl.digest(len(q))
        _, L, _, _ = cl.get_state()
        gammas.append(L[0, 1] / L[1, 1])
        r = oracle.evaluate(oracle.DO, wq.astype(np.float64), L, w.rc, w.eps, w.sigma, w.ushift)
        assert np.array_equal(cnt, r.cnt) and np.array_equal(hs, r.hsum) and np.array_equal(hx, r.hxor), step
        assert np.array_equal(counts, r.cnt), step
    cl.close()
    assert np.any(np.diff(gammas) < 0)  # a Lees-Edwards reset happened inside the run


def test_rows_kernel_overfull_neighbour_row_fails_loudly():
    """k_pairs_rows stages a batch's neighbour rows in a fixed shared-memory buffer; a row it cannot
    stage even for a single particle (one cell holding > 512 particles) is reported as NC_E_OOM, never
    evaluated from a truncated buffer.  The particle-per-thread kernel streams its rows from global
    memory and still reproduces the oracle's pair set on the same input."""
    import torch
    from paper_1412_3784_b200.nemdcell import NcError

    rng = np.random.default_rng([1412, 3784, 77])
    L = np.eye(3) * 12.0
    rc = 2.5
    q = np.concatenate([rng.uniform(0.1, 2.9, size=(600, 3)), rng.uniform(0.0, 12.0, size=(400, 3))])
    cl = _cl("do", "f32", rc, len(q), sigma=0.1, kernel="rows")
    cl.set_box(L)
    with pytest.raises(NcError, match="NC_E_OOM"):
        cl.compute_forces(torch.from_numpy(q.astype(np.float32)).cuda())
    cl.close()
    cl = _cl("do", "f32", rc, len(q), sigma=0.1, kernel="sparse")
    counts, wq, (cnt, hs, hx), st = _eval(cl, L, q.astype(np.float32), "f32")
    cl.close()
    r = oracle.evaluate(oracle.DO, wq, L, rc, 1.0, 0.1, 0.0)
    assert np.array_equal(cnt, r.cnt) and np.array_equal(hs, r.hsum) and np.array_equal(counts, r.cnt)
