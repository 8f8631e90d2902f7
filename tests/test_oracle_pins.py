"""Pins for the CPU oracle against what the paper and the mathematics fix.

None of these re-types the oracle's own formulas: each checks a printed value
(tests/golden/paper_values.json, cited), a closed form, an invariant, a
special case that reduces to a textbook routine, or brute force on tiny
inputs by an independent enumeration.  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import box as obox
from paper_1412_3784_b200 import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def safe_rc(L, frac=1.0):
    """Largest cutoff keeping both grids non-degenerate (DS c >= 3, DO l >= 4,4,3)."""
    _, R = oracle.qr(L)
    return frac * min(min(oracle.heights(L)) / 3.05, R[0, 0] / 4.05, R[1, 1] / 4.05, R[2, 2] / 3.05)


def rand_box(rng, a=10.0, skew=0.4):
    """A random deformed, positively oriented box."""
    while True:
        L = a * (np.eye(3) + rng.uniform(-skew, skew, size=(3, 3)))
        if np.linalg.det(L) > 0.3 * a ** 3:
            return L


# ------------------------------------------------------------------ printed values

def test_search_efficiency_printed():
    g = GOLD["search_efficiency_equilibrium"]
    assert abs(oracle.search_efficiency_equilibrium() - g["value"]) < g["abs_tol"]
    # cube divisible by d_cut: V_DS = 27 d^3
    L = np.eye(3) * 7.5
    assert oracle.v_ds(L, 2.5) == pytest.approx(27 * 2.5 ** 3, rel=1e-15)


def test_heights_spec_example_corrected():
    g = GOLD["ds_heights_shear_example"]
    h = oracle.heights(g["L"])
    assert np.allclose(h, g["h"], rtol=0, atol=1e-12)
    assert list(oracle.ds_dims(g["L"], g["rc"])) == g["c"]
    assert oracle.v_ds(g["L"], g["rc"]) == pytest.approx(GOLD["ds_volume_shear_example"]["value"], abs=1e-12)


def test_heights_identity_random():
    rng = np.random.default_rng(1)
    for _ in range(20):
        L = rand_box(rng)
        h = oracle.heights(L)
        det = np.linalg.det(L)
        v = [L[:, 0], L[:, 1], L[:, 2]]
        for k in range(3):
            cross = np.cross(v[(k + 1) % 3], v[(k + 2) % 3])
            assert h[k] * np.linalg.norm(cross) == pytest.approx(det, rel=1e-13)
            assert h[k] <= np.linalg.norm(v[k]) * (1 + 1e-14)


def test_heights_shear_closed_form():
    a = 33.592
    for gamma in (-0.5, -0.2, 0.0, 0.3, 0.49):
        L = a * np.array([[1, gamma, 0], [0, 1, 0], [0, 0, 1.0]])
        h = oracle.heights(L)
        assert h[0] == pytest.approx(a / math.sqrt(1 + gamma ** 2), rel=1e-14)
        assert h[1] == pytest.approx(a, rel=1e-14) and h[2] == pytest.approx(a, rel=1e-14)
    # C1 at |gamma| = 1/2: h1 = 30.046 -> c1 = 26 with r_c = 2^(1/6)
    L = a * np.array([[1, 0.5, 0], [0, 1, 0], [0, 0, 1.0]])
    assert oracle.ds_dims(L, oracle.WCA_RC)[0] == 26


def test_inverse_and_qr():
    rng = np.random.default_rng(2)
    for _ in range(20):
        L = rand_box(rng)
        Li, det = oracle.inv3(L)
        assert np.abs(Li @ L - np.eye(3)).max() < 1e-14
        assert det == pytest.approx(np.linalg.det(L), rel=1e-13)
        Q, R = oracle.qr(L)
        assert np.abs(Q @ R - L).max() < 1e-13
        assert np.abs(Q.T @ Q - np.eye(3)).max() < 1e-14
        assert R[1, 0] == R[2, 0] == R[2, 1] == 0.0 and np.all(np.diag(R) > 0)
        assert np.linalg.det(Q) == pytest.approx(1.0, abs=1e-14)
    # QR of an upper-triangular basis is itself, exactly
    L = np.array([[1.0, 0.5, 0.25], [0.0, 1.3, -0.7], [0.0, 0.0, 0.9]])
    Q, R = oracle.qr(L)
    assert np.array_equal(Q, np.eye(3)) and np.array_equal(R, L)
    with pytest.raises(ValueError):
        oracle.inv3(np.diag([1.0, 1.0, -1.0]))


def test_do_dims_spec_example():
    g = GOLD["do_dims_uniaxial_example"]
    L = np.diag([math.exp(0.5), math.exp(-0.25), math.exp(-0.25)]) * 10
    l, w = oracle.do_dims(L, g["rc"])
    assert list(l) == g["value"]
    v = oracle.v_do_cell(L, 1.0)
    assert v == pytest.approx(1000.0 / 784.0, rel=1e-13)
    assert abs(v - GOLD["do_cell_volume_uniaxial_example"]["value"]) < GOLD["do_cell_volume_uniaxial_example"]["abs_tol"]


def test_rearrangement_spec_example():
    g = GOLD["rearrange_example"]
    out, nh = oracle.do_rearrange([g["point"]], g["R"])
    assert np.allclose(out[0], g["value"], atol=g["abs_tol"], rtol=0)


def test_rearrangement_is_lattice_translate_into_rectangle():
    """Eqs. (11)-(12) with the 'mod r11' reading (R1): the image lies in
    [0,r11) x [0,r22) x [0,r33) and differs from the input by R n, n integer.
    A 'mod r22' implementation fails this whenever r11 != r22."""
    rng = np.random.default_rng(3)
    for _ in range(10):
        L = rand_box(rng)
        _, R = oracle.qr(L)
        lam = rng.uniform(0, 1, size=(500, 3))
        xyz = lam @ R.T
        out, nh = oracle.do_rearrange(xyz, R)
        assert np.all(out[:, 0] >= 0) and np.all(out[:, 0] < R[0, 0])
        assert np.all(out[:, 1] >= 0) and np.all(out[:, 1] < R[1, 1])
        assert np.all(out[:, 2] >= 0) and np.all(out[:, 2] < R[2, 2])
        assert np.allclose(out - xyz, nh @ R.T, atol=1e-12)


# ------------------------------------------------------------------ stencils

def _generic_box(rng, l, rc=1.0):
    """Upper-triangular box with r_kk slightly above l_k rc and generic offsets."""
    r = [(lk + rng.uniform(0.1, 0.9)) * rc for lk in l]
    R = np.array([[r[0], rng.uniform(0.1, 0.9) * r[0], rng.uniform(0.1, 0.9) * r[0]],
                  [0, r[1], rng.uniform(0.1, 0.9) * r[1]],
                  [0, 0, r[2]]])
    return R


def test_do_case_counts_and_closed_form():
    """Histogram of neighborhood sizes equals the paper's case populations
    S1..S4 and its mean the closed form, for every
    l in [4..8]^3."""
    rng = np.random.default_rng(4)
    for l1 in range(4, 9):
        for l2 in range(4, 9):
            for l3 in range(4, 9):
                R = _generic_box(rng, (l1, l2, l3))
                hist, dims = oracle.stencil_histogram(oracle.DO, R, 1.0)
                assert list(dims) == [l1, l2, l3]
                S2, S3, S4 = 2 * l1 * l3 - 4 * l1, 2 * l1 * l2 - 4 * l1, 4 * l1
                S1 = l1 * l2 * l3 - S2 - S3 - S4
                expect = np.zeros(64, dtype=np.int64)
                expect[27], expect[30], expect[34], expect[36] = S1, S2, S3, S4
                assert np.array_equal(hist, expect), (l1, l2, l3)
                mean = (hist * np.arange(64)).sum() / hist.sum()
                assert mean == pytest.approx(oracle.do_average_count((l1, l2, l3)), abs=1e-12)
    assert oracle.do_average_count((10, 10, 10)) == pytest.approx(GOLD["do_average_count_10_10_10"]["value"], abs=1e-12)


def test_stencils_equilibrium_27():
    for L in (np.eye(3) * 10.0, np.eye(3) * 12.5):
        for v in (oracle.DS, oracle.DO):
            hist, dims = oracle.stencil_histogram(v, L, 2.5 if L[0, 0] == 12.5 else 1.0)
            assert hist[27] == np.prod(dims) and hist.sum() == hist[27]
    rng = np.random.default_rng(5)
    for _ in range(5):
        L = rand_box(rng, a=12)
        hist, dims = oracle.stencil_histogram(oracle.DS, L, 1.0)
        assert hist[27] == np.prod(dims)        # DS: always 27


# ------------------------------------------------------------------ pair sets

def naive_pairs(q, L, rc):
    """Independent enumeration over all n in {-2..2}^3 (tiny N only)."""
    rng_n = np.array([(a, b, c) for a in range(-2, 3) for b in range(-2, 3) for c in range(-2, 3)])
    shifts = rng_n @ L.T
    out = []
    n = len(q)
    for i in range(n):
        d = q[None, :, None, :] if False else None
        dd = (q[:, None, :] + shifts[None, :, :]) - q[i][None, None, :]
        r2 = (dd ** 2).sum(axis=2)
        js, ks = np.nonzero(r2 < rc * rc)
        for j, k in zip(js, ks):
            if j == i and not rng_n[k].any():
                continue
            out.append((i, j, *rng_n[k]))
    return np.array(sorted(out), dtype=np.int64).reshape(-1, 5)


@pytest.mark.parametrize("seed", range(6))
def test_pair_sets_brute_ds_do_agree(seed):
    rng = np.random.default_rng(100 + seed)
    L = rand_box(rng, a=8.0, skew=0.35)
    rc = safe_rc(L)
    n = 300
    q = oracle.wrap(rng.uniform(0, 1, size=(n, 3)) @ L.T, L)
    res = {m: oracle.evaluate(m, q, L, rc, pairs_cap=200000) for m in (oracle.BRUTE, oracle.DS, oracle.DO)}
    pb = res[oracle.BRUTE].pairs
    assert len(pb) > 0
    for m in (oracle.DS, oracle.DO):
        assert np.array_equal(res[m].pairs, pb), m
        assert np.abs(res[m].F - res[oracle.BRUTE].F).max() < 1e-9 * max(1.0, np.abs(res[oracle.BRUTE].F).max())
    if seed < 2:
        assert np.array_equal(naive_pairs(q, L, rc), pb.astype(np.int64))


def test_equilibrium_reduces_to_textbook_cell_list():
    """Cube divisible by d_cut: DS cells are floor(q c / a) and the DS,
    DO and brute-force pair sets coincide."""
    rng = np.random.default_rng(7)
    a, rc = 10.0, 2.5
    L = np.eye(3) * a
    q = rng.uniform(0, a, size=(400, 3))
    q = oracle.wrap(q, L)
    cell, _, dims = oracle.cell_keys(oracle.DS, q, L, rc)
    ijk = np.floor(q * 4 / a).astype(np.int64)
    assert np.array_equal(cell, ijk[:, 0] + 4 * (ijk[:, 1] + 4 * ijk[:, 2]))
    cdo, nh, _ = oracle.cell_keys(oracle.DO, q, L, rc)
    assert np.array_equal(cdo, cell) and not nh.any()
    p = [oracle.evaluate(m, q, L, rc, pairs_cap=100000).pairs for m in (oracle.BRUTE, oracle.DS, oracle.DO)]
    assert np.array_equal(p[0], p[1]) and np.array_equal(p[0], p[2])


def test_cutoff_is_strict():
    L = np.eye(3) * 10.0
    rc = 2.5
    for f, expect in ((1 - 1e-6, 1), (1 + 1e-6, 0)):
        q = np.array([[1.0, 1.0, 1.0], [1.0 + rc * f, 1.0, 1.0]])
        r = oracle.evaluate(oracle.DO, q, L, rc)
        assert r.interactions == 2 * expect


def test_digest_matches_independent_mix():
    def mix(z):
        m = (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & m
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & m
        return z ^ (z >> 31)

    rng = np.random.default_rng(8)
    L = rand_box(rng, a=7.0, skew=0.3)
    rc = safe_rc(L, 0.98)
    q = oracle.wrap(rng.uniform(0, 1, size=(150, 3)) @ L.T, L)
    r = oracle.evaluate(oracle.DO, q, L, rc, pairs_cap=50000)
    for i in range(len(q)):
        sel = r.pairs[r.pairs[:, 0] == i]
        hs, hx = 0, 0
        for (_, j, a, b, c) in sel:
            k = int(j) | ((int(a) + 8) << 32) | ((int(b) + 8) << 36) | ((int(c) + 8) << 40)
            h = mix(k)
            hs = (hs + h) & ((1 << 64) - 1)
            hx ^= h
        assert r.cnt[i] == len(sel) and int(r.hsum[i]) == hs and int(r.hxor[i]) == hx


# ------------------------------------------------------------------ forces

def lj(r, eps=1.0, sig=1.0):
    s6 = (sig / r) ** 6
    return 4 * eps * (s6 * s6 - s6), 24 * eps * (2 * s6 * s6 - s6) / r


def test_two_particle_values():
    L = np.eye(3) * 20.0
    g = GOLD["wca_at_sigma"]
    q = np.array([[5.0, 5.0, 5.0], [6.0, 5.0, 5.0]])
    r = oracle.evaluate(oracle.DS, q, L, oracle.WCA_RC)
    assert abs(r.F[0, 0] + g["F"]) < g["abs_tol"] and abs(r.F[1, 0] - g["F"]) < g["abs_tol"]
    assert abs(r.U - g["U"]) < g["abs_tol"]
    # LJ minimum at 2^(1/6): zero force; U = -1 - phi(rc) (energy-shifted, R11)
    q = np.array([[5.0, 5.0, 5.0], [5.0 + 2 ** (1 / 6), 5.0, 5.0]])
    r = oracle.evaluate(oracle.DO, q, L, 2.5)
    assert np.abs(r.F).max() < 1e-13
    assert r.U == pytest.approx(-1.0 - lj(2.5)[0], abs=1e-13)
    assert r.U == pytest.approx(-0.983683108864, abs=1e-12)


def test_fcc_lattice_sums():
    """Perfect FCC at rho = 0.8442, r_c = 2.5: shells 12/6/24/12 at a/sqrt2 *
    sqrt(1,2,3,4) (textbook lattice sums), so U/N = sum_s n_s phi(r_s)/2,
    W/N = sum_s n_s fr(r_s) r_s^2 / 6 * I, F_i = 0 by inversion symmetry."""
    q, L = W.perfect_fcc(10)
    a = (4 / W.RHO) ** (1 / 3)
    shells = [(12, a / math.sqrt(2)), (6, a), (24, a * math.sqrt(1.5)), (12, a * math.sqrt(2))]
    assert a * math.sqrt(2.5) > 2.5 > shells[-1][1]
    shift = lj(2.5)[0]
    u = sum(ns * (lj(r)[0] - shift) for ns, r in shells) / 2
    w = sum(ns * lj(r)[1] * r for ns, r in shells) / 6   # fr r^2 = (-phi'/r) r^2
    for m in (oracle.DS, oracle.DO):
        r = oracle.evaluate(m, q, L, 2.5)
        N = len(q)
        assert r.U / N == pytest.approx(u, rel=1e-13)
        assert r.U / N == pytest.approx(-6.332811992581, abs=1e-11)
        assert np.abs(r.F).max() < 1e-11
        assert np.allclose(r.W[:3] / N, w, rtol=1e-13) and np.abs(r.W[3:]).max() / N < 1e-13
        assert r.interactions == 54 * N


def test_simple_cubic_neighbor_count():
    K = 8
    L = np.eye(3) * K
    g = np.stack(np.meshgrid(*[np.arange(K)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(float) + 0.25
    for rc, cnt in ((2.5, 80), (2 ** (1 / 6), 6)):
        r = oracle.evaluate(oracle.DS, g, L, rc)
        assert r.interactions == cnt * len(g)


def test_newton_translation_remap_invariance():
    rng = np.random.default_rng(9)
    w = W.make(2, scale=4)
    w.L = W.box_at(w.L0, w.A, "kr", 0.3, w.extra)
    q = oracle.wrap(W.positions(w), w.L)
    r = oracle.evaluate(oracle.DO, q, w.L, w.rc)
    Fs = np.abs(r.F).max()
    assert np.abs(r.F.sum(axis=0)).max() < 1e-10 * Fs * len(q) ** 0.5
    # translation
    t = rng.uniform(-3, 3, size=3)
    q2 = oracle.wrap(q + t, w.L)
    r2 = oracle.evaluate(oracle.DS, q2, w.L, w.rc)
    assert np.abs(r2.F - r.F).max() < 1e-9 * Fs and r2.U == pytest.approx(r.U, rel=1e-12)
    # SL(3,Z) remap L -> L M leaves the lattice and all pair forces unchanged
    M = np.array([[1, 1, 0], [0, 1, 0], [0, 1, 1]])
    LM = w.L @ M
    q3 = oracle.wrap(q, LM)
    for m in (oracle.BRUTE, oracle.DO):
        r3 = oracle.evaluate(m, q3, LM, w.rc) if m == oracle.DO else None
        if r3 is not None:
            assert np.abs(r3.F - r.F).max() < 1e-9 * Fs and r3.U == pytest.approx(r.U, rel=1e-12)
            assert r3.interactions == r.interactions


# ------------------------------------------------------------------ boxes / remaps

def test_kr_identity_and_bases_agree():
    a = 67.717
    L0, lam = obox.kr_initial_basis(a)
    L0w, lamw = W.kr_basis(a)
    assert np.abs(L0 - L0w).max() < 1e-13 and lam == pytest.approx(GOLD["kr_stretch_at_period"]["value"], abs=1e-15)
    eps = 0.1
    A = np.diag([eps, -eps, 0.0])
    ts = math.log(lam) / eps
    E = obox.expm(A, ts)
    assert np.abs(E @ L0 - L0 @ obox.M_KR).max() < 1e-13 * a
    b = obox.Box(L0, A, "kr", 0.0)
    for t in np.linspace(0, 3 * ts, 37):
        L = b.at(t)
        assert np.linalg.det(L) == pytest.approx(a ** 3, rel=1e-13)


def test_le_angle_bound():
    g = GOLD["le_max_angle_deg"]
    a = 10.0
    L0 = np.eye(3) * a
    A = np.zeros((3, 3)); A[0, 1] = 0.37
    b = obox.Box(L0, A, "le", 0.0)
    worst = 0.0
    for t in np.linspace(0, 20, 4001):
        L = b.at(t)
        v1, v2 = L[:, 0], L[:, 1]
        ang = 90 - math.degrees(math.acos(np.dot(v1, v2) / np.linalg.norm(v1) / np.linalg.norm(v2)))
        worst = max(worst, abs(ang))
        assert np.linalg.det(L) == pytest.approx(a ** 3, rel=1e-13)
    assert worst <= 90 - math.degrees(math.atan(2)) + 1e-9
    # at the reset instant the tilt is -a/2: the printed maximum angle
    L = b.at(0.5 / 0.37)
    ang = math.degrees(math.atan(abs(L[0, 1]) / L[1, 1]))
    assert abs(ang - g["value"]) < g["abs_tol"]
    # unremapped shear at t* = 1/eps is 45 degrees and the undeformed lattice
    E = obox.expm(A, 1 / 0.37) @ L0
    assert np.allclose(E @ obox.M_SHEAR, L0, atol=1e-12)


def test_gkr_construction():
    a = 10.0
    L0, om1, om2 = obox.gkr_construction(a)
    M1 = obox.M1_GKR.astype(float)
    M2 = (M1 - np.eye(3)) @ (M1 - np.eye(3))
    assert np.allclose(np.round(M2), M2) and round(np.linalg.det(M2)) == 1
    for M, om in ((M1, om1), (M2, om2)):
        assert np.abs(L0 @ M - np.diag(np.exp(om)) @ L0).max() < 1e-13 * a
        assert abs(om.sum()) < 1e-14
    assert np.allclose(M1 @ M2, M2 @ M1)
    _, _, L0w, o1w, o2w = W.gkr_params(a)
    assert np.abs(L0w - L0).max() < 1e-13 and np.abs(o1w - om1).max() < 1e-14 and np.abs(o2w - om2).max() < 1e-14
    for ad in ((-1, -1, 2), (1, 1, -2)):
        A = np.diag(0.1 * np.array(ad, dtype=float))
        b = obox.Box(L0, A, "gkr", 0.0, om1=om1, om2=om2)
        for t in np.linspace(0, 40, 81):
            L = b.at(t)
            # the remapped box generates the same lattice as e^{At} L0
            X = np.linalg.solve(L, obox.expm(A, t) @ L0)
            assert np.abs(X - np.round(X)).max() < 1e-8 and abs(round(np.linalg.det(np.round(X)))) == 1
            assert np.linalg.det(L) == pytest.approx(a ** 3, rel=1e-12)
            alpha = b.beta * b.eps * t
            f = alpha - np.floor(alpha + 0.5)
            assert np.all(f >= -0.5) and np.all(f < 0.5)


# ------------------------------------------------------------------ SLLOD

def _zero_forces(q, L):
    return np.zeros_like(q), 0.0, np.zeros(6)


def test_sllod_free_streaming_keeps_fractional_coordinates():
    """F = 0, p = 0: particles ride the flow, lambda = L^{-1} q is invariant
    (mod 1, through remaps) -- images move as q + L_t n."""
    for k in (1, 2):
        w = W.make(k, scale=4)
        q = oracle.wrap(W.positions(w)[:200], w.L)
        p = np.zeros_like(q)
        b = obox.Box(w.L0, w.A, w.policy, w.t0, tstar=w.extra.get("tstar"))
        lam0 = q @ np.linalg.inv(b.L).T
        F = np.zeros_like(q)
        for _ in range(50):
            q, p, F, _, _ = obox.sllod_step(q, p, F, b, 0.05, _zero_forces)
        # remaps change the basis; compare lattices through positions: q - e^{A t}... use lab frame
        E = obox.expm(w.A, 50 * 0.05)
        q_expect = (lam0 @ (E @ w.L).T)
        dlam = np.linalg.solve(b.L, (q - q_expect).T).T
        assert np.abs(dlam - np.round(dlam)).max() < 1e-10


def test_sllod_equilibrium_is_velocity_verlet_energy_conserving():
    w = W.make(0, scale=2)
    q = oracle.wrap(W.positions(w), w.L)
    p = W.momenta(w) * 0.5
    b = obox.Box(w.L0, w.A, "none", 0.0)

    def forces(q, L):
        r = oracle.evaluate(oracle.DS, q, L, w.rc, want=("F", "U", "W"))
        return r.F, r.U, r.W

    F, U, _ = forces(q, w.L)
    E0 = U + 0.5 * (p ** 2).sum()
    Es = []
    for _ in range(100):
        q, p, F, U, _ = obox.sllod_step(q, p, F, b, 0.002, forces)
        Es.append(U + 0.5 * (p ** 2).sum())
    assert max(abs(e - E0) for e in Es) < 2e-3 * abs(E0)


def _lattice_residual(q, q_ref, L):
    """max over particles of the distance (in fractional units of L) from q - q_ref to the
    nearest lattice vector L n: zero iff q is an image of q_ref."""
    d = np.linalg.solve(L, (q - q_ref).T).T
    return np.abs(d - np.round(d)).max()


def test_sllod_shear_free_flight_is_a_straight_line():
    """F = 0, p0 != 0, shear A (A^2 = 0): SLLOD's lab velocity v = p/m + A q
    is a constant of the free motion (dq/dt = p/m + A q, dp/dt = -A p, so
    dv/dt = A^2 q = 0), hence the lab trajectory is the straight line
    q_n = q0 + n dt (p0/m + A q0) -- exactly, for any dt, since the discrete
    map's E(dt/2) E(-dt/2) = I - A^2 dt^2/4 = I.  Wrapping and the Lees-Edwards
    resets only replace q by a lattice image q + L_t n, whose velocity is
    v + A L_t n, so q_n must equal the straight line modulo
    the lattice L_t at every step.  Fails for E(+dt/2) on p, for a
    drift without the E(dt/2) factor, or for a lab/peculiar mix-up."""
    rng = np.random.default_rng(11)
    a, rate, m = 10.0, 0.7, 1.3
    for gamma0 in (0.0, 0.31, -0.45):
        L0 = np.array([[a, gamma0 * a, 0.0], [0.0, a, 0.0], [0.0, 0.0, a]])
        A = np.zeros((3, 3)); A[0, 1] = rate
        b = obox.Box(L0, A, "le", 0.0)
        q0 = oracle.wrap(rng.uniform(0, 1, size=(64, 3)) @ L0.T, L0)
        p0 = rng.normal(size=(64, 3))
        v0 = p0 / m + q0 @ A.T
        q, p, F = q0.copy(), p0.copy(), np.zeros_like(q0)
        dt = 0.05
        nres = 0
        for n in range(1, 121):  # t = 6: the tilt passes the half-spacing reset ~4 times
            g_before = b.L[0, 1]
            q, p, F, _, _ = obox.sllod_step(q, p, F, b, dt, _zero_forces, mass=m)
            nres += int(b.L[0, 1] < g_before)
            assert _lattice_residual(q, q0 + n * dt * v0, b.L) < 1e-12
            # peculiar momenta themselves follow p(t) = e^{-At} p0 = (I - A t) p0 exactly
            assert np.abs(p - p0 @ (np.eye(3) - A * n * dt).T).max() < 1e-12 * np.abs(p0).max() * (1 + rate * n * dt)
        assert nres >= 3


def _exact_free_flight_diag(q0, p0, a_diag, t, m):
    """Closed form of dq/dt = p/m + A q, dp/dt = -A p for diagonal A = diag(a):
    p(t) = e^{-at} p0, q(t) = e^{at} q0 + (e^{at} - e^{-at}) / (2a) p0/m  (t p0/m for a = 0)."""
    a = np.asarray(a_diag, dtype=np.float64)
    g = np.where(a != 0.0, np.sinh(a * t) / np.where(a != 0.0, a, 1.0), t)
    return np.exp(a * t) * q0 + g * p0 / m, np.exp(-a * t) * p0


def _free_flight_run(box_factory, q0, p0, T, nsteps, m):
    b = box_factory()
    q, p, F = q0.copy(), p0.copy(), np.zeros_like(q0)
    dt = T / nsteps
    nremap = 0
    for _ in range(nsteps):
        Lb = b.L.copy()
        q, p, F, _, _ = obox.sllod_step(q, p, F, b, dt, _zero_forces, mass=m)
        nremap += int(np.abs(np.linalg.solve(obox.expm(b.A, dt) @ Lb, b.L) - np.eye(3)).max() > 0.5)
    return q, p, b, nremap


def test_sllod_elongational_free_flight_converges_to_exact_solution():
    """F = 0, diagonal A (KR planar, and the generalized-KR uniaxial /
    biaxial flows, P:431-439 with R23): the momentum factor gives
    p_n = e^{-A n dt} p0 exactly (to rounding) and the positions converge at
    SECOND order to the exact ODE solution e^{At} q0 + (e^{At} - e^{-At}) (2A)^{-1} p0/m,
    modulo the lattice of the remapped box (the remaps happen inside the runs):
    halving dt quarters the error.  A wrong sign in E(-dt/2), a missing E(dt/2) drift
    factor or a first-order splitting fails this."""
    rng = np.random.default_rng(12)
    m = 0.8
    a = 12.0
    cases = []
    L0kr, _ = obox.kr_initial_basis(a)
    eps = 0.5
    Akr = np.diag([eps, -eps, 0.0])
    tstar = math.log((3.0 + math.sqrt(5.0)) / 2.0) / eps
    cases.append((Akr, lambda: obox.Box(L0kr, Akr, "kr", tstar - 0.6), tstar - 0.6))
    L0g, om1, om2 = obox.gkr_construction(a)
    for ad in ((-1.0, -1.0, 2.0), (1.0, 1.0, -2.0)):
        Ag = np.diag(eps * np.array(ad))
        bb = obox.Box(L0g, Ag, "gkr", 0.0, om1=om1, om2=om2)
        # start 0.6 before alpha_2 crosses a half-integer: a reset inside the run
        t_cross = (0.5 / abs(bb.beta[1] * bb.eps))
        t0 = t_cross - 0.6
        cases.append((Ag, (lambda Ag=Ag, t0=t0: obox.Box(L0g, Ag, "gkr", t0, om1=om1, om2=om2)), t0))
    T = 1.5
    for A, factory, t0 in cases:
        Lstart = factory().L
        q0 = oracle.wrap(rng.uniform(0, 1, size=(48, 3)) @ Lstart.T, Lstart)
        p0 = rng.normal(size=(48, 3)) * 2.0
        errs = []
        for nsteps in (60, 120, 240):
            q, p, b, nremap = _free_flight_run(factory, q0, p0, T, nsteps, m)
            assert nremap >= 1, "the run must cross a remap"
            q_ex, p_ex = _exact_free_flight_diag(q0, p0, np.diag(A), T, m)
            assert np.abs(p - p_ex).max() < 1e-13 * np.abs(p0).max() * 4
            errs.append(_lattice_residual(q, q_ex, b.L))
        assert errs[0] > 1e-9  # the splitting error is visible at all (not trivially exact)
        r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
        assert 3.6 < r1 < 4.4 and 3.6 < r2 < 4.4, (errs, r1, r2)


def test_expm_matches_closed_forms():
    """e^{As} for non-diagonal, non-nilpotent A (the scaling-and-squaring branch) against
    closed forms (to 1e-14 per unit of |As|): (a) a rotation generator gives the rotation
    matrix by angle theta s;
    (b) a random diagonalizable traceless A = V D V^{-1} gives V e^{Ds} V^{-1} (eigen-
    decomposition written out, not through expm); (c) diagonal and shear (nilpotent)
    branches: elementwise exp and exactly I + As."""
    for theta, s in ((0.3, 1.0), (1.7, 2.5), (-4.0, 3.0), (1e-3, 0.5)):
        G = np.array([[0.0, -theta, 0.0], [theta, 0.0, 0.0], [0.0, 0.0, 0.0]])
        c, sn = math.cos(theta * s), math.sin(theta * s)
        R = np.array([[c, -sn, 0.0], [sn, c, 0.0], [0.0, 0.0, 1.0]])
        # scaling and squaring amplifies rounding ~ linearly in |As| (each squaring doubles it)
        assert np.abs(obox.expm(G, s) - R).max() < 1e-14 * max(1.0, abs(theta * s))
    rng = np.random.default_rng(13)
    for _ in range(20):
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        V = Q + 0.2 * rng.normal(size=(3, 3))  # non-orthogonal, well conditioned
        if np.linalg.cond(V) > 5:
            continue
        dvals = rng.uniform(-1.0, 1.0, size=3)
        dvals -= dvals.mean()  # traceless
        Vi = np.linalg.inv(V)
        A = V @ np.diag(dvals) @ Vi
        for s in (0.1, 1.0, 3.0):
            E = V @ np.diag(np.exp(dvals * s)) @ Vi
            nrm = max(1.0, np.abs(A * s).sum(axis=1).max())
            assert np.abs(obox.expm(A, s) - E).max() < 1e-14 * nrm * max(1.0, np.abs(E).max()) * np.linalg.cond(V)
    D = np.diag([0.2, -0.5, 0.3])
    assert np.array_equal(obox.expm(D, 2.0), np.diag(np.exp(np.array([0.4, -1.0, 0.6]))))
    S = np.zeros((3, 3)); S[0, 1] = 0.75
    assert np.array_equal(obox.expm(S, 3.0), np.array([[1.0, 2.25, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]))


def test_fig9_long_run_efficiency_matches_paper():
    """Paper's efficiency study: uniaxial A = diag(0.05, -0.025, -0.025),
    a = 10 d_cut, d_cut = (3/4pi)^(1/3) (interaction volume 1); long-run mean
    neighborhood volumes give search efficiencies ~0.0688 (DS) and ~0.123 (DO).
    Computed here from the oracle's own DS counts (Eq. 14) and DO stencil
    histogram (Eq. 15) along the derived GKR construction (R23); the
    printed values pin the construction + stencil + volume formulas to ~3%."""
    dcut = (3.0 / (4.0 * math.pi)) ** (1.0 / 3.0)
    a = 10.0 * dcut
    L0, om1, om2 = obox.gkr_construction(a)
    A = np.diag([0.05, -0.025, -0.025])
    b = obox.Box(L0, A, "gkr", 0.0, om1=om1, om2=om2, eps=0.025,
                 beta=obox.gkr_beta(om1, om2, np.array([2.0, -1.0, -1.0])))
    V = {oracle.DS: [], oracle.DO: []}
    for t in np.linspace(0.0, 4000.0, 1500, endpoint=False):
        L = b.at(t)
        vbox = np.linalg.det(L)
        for m in (oracle.DS, oracle.DO):
            hist, dims = oracle.stencil_histogram(m, L, dcut)
            ncell = int(np.prod(dims.astype(np.int64)))
            V[m].append(vbox / ncell * (hist * np.arange(64)).sum() / ncell)
    eff_ds = 1.0 / np.mean(V[oracle.DS])
    eff_do = 1.0 / np.mean(V[oracle.DO])
    assert eff_ds == pytest.approx(GOLD["fig9_efficiency_ds"]["value"], rel=0.04)
    assert eff_do == pytest.approx(GOLD["fig9_efficiency_do"]["value"], rel=0.04)
    # and DS never beats the equilibrium efficiency; DO approaches it for large boxes
    assert eff_ds < eff_do < oracle.search_efficiency_equilibrium()


# ---------------------------------------------------------------- lattice reduction policy (R30)

def test_lattice_reduce_is_the_lees_edwards_reset():
    """For a sheared basis the greedy Lagrange reduction is exactly the LE remap
    L -> L M with M = [[1,-1,0],[0,1,0],[0,0,1]] at half a lattice spacing."""
    a = 10.0
    for g, g_red in ((0.3, 0.3), (0.7, -0.3), (-0.7, 0.3), (1.6, -0.4), (0.49, 0.49), (-0.49, -0.49)):
        L = np.array([[a, g * a, 0.0], [0.0, a, 0.0], [0.0, 0.0, a]])
        Lr, changed = obox.lattice_reduce(L)
        assert changed == (g != g_red)
        assert Lr[0, 1] == pytest.approx(g_red * a, abs=1e-12)
        assert np.array_equal(Lr[:, 0], L[:, 0]) and np.array_equal(Lr[:, 2], L[:, 2])
    # a long shear run under the reduction policy reproduces the LE boxes (away from the tie)
    A = np.zeros((3, 3))
    A[0, 1] = 0.1
    b = obox.Box(np.eye(3) * a, A, "reduce", 0.0)
    le = obox.Box(np.eye(3) * a, A, "le", 0.0)
    for _ in range(400):
        b.advance(0.1)
        le.advance(0.1)
        if abs(abs(le.L[0, 1] / a) - 0.5) > 0.01:
            assert np.abs(b.L - le.L).max() < 1e-12 * a


def test_lattice_reduce_keeps_the_lattice():
    """Random skewed bases: L' = L M with M integer, det M = +1 (same lattice),
    and L' is pairwise reduced: no single step v_i - mu v_j shortens any column."""
    rng = np.random.default_rng(30)
    for _ in range(200):
        L = np.eye(3) * 5.0 + rng.normal(scale=4.0, size=(3, 3))
        if np.linalg.det(L) <= 0:
            L[:, 0] *= -1
        Lr, _ = obox.lattice_reduce(L)
        M = np.linalg.solve(L, Lr)
        assert np.abs(M - np.round(M)).max() < 1e-8
        assert round(np.linalg.det(np.round(M))) == 1
        assert np.linalg.det(Lr) == pytest.approx(np.linalg.det(L), rel=1e-12)
        for i in range(3):
            for j in range(3):
                if i == j:
                    continue
                for mu in (-2, -1, 1, 2):
                    w = Lr[:, i] - mu * Lr[:, j]
                    assert w @ w >= Lr[:, i] @ Lr[:, i] * (1 - 1e-9)


def test_reduce_policy_general_flow_stays_a_bounded_lattice():
    """A general traceless, non-diagonal, non-nilpotent A (an elliptic flow with a
    shear component): under the reduction policy the box is always e^{At} L0 times
    an integer det-1 matrix, det L is constant, and the reduced box keeps every
    height above 0.4 det^{1/3} over many flow periods (R30)."""
    a = 8.0
    A = np.array([[0.0, 0.3, 0.1], [-0.2, 0.0, 0.0], [0.0, 0.15, 0.0]])
    L0 = np.eye(3) * a
    b = obox.Box(L0, A, "reduce", 0.0)
    det0 = np.linalg.det(L0)
    nred = 0
    Lprev = b.L.copy()
    for k in range(3000):
        L = b.advance(0.05)
        M = np.linalg.solve(obox.expm(A, b.t) @ L0, L)
        assert np.abs(M - np.round(M)).max() < 1e-6
        assert np.linalg.det(L) == pytest.approx(det0, rel=1e-9)
        Li = np.linalg.inv(L)
        h = 1.0 / np.linalg.norm(Li, axis=1)
        assert h.min() > 0.4 * det0 ** (1.0 / 3.0)
        if np.abs(np.linalg.solve(Lprev, L) - np.eye(3)).max() > 0.5:
            nred += 1
        Lprev = L.copy()
    assert nred >= 5
