"""Seeded synthetic workloads C0-C4 (BASELINE.json configs[0..4]).

This module only DRAWS inputs: box matrices, flow/remap parameters, particle
positions and momenta.  It holds none of the method's arithmetic (no wrap,
cell keys, stencils, pair forces or SLLOD update) and imports neither the CUDA
binding nor the oracle; both sides consume what it returns.  The recipe is
written out in DESIGN.md section 4 (readings R20-R25).

Positions: a crystal of K^3 sites (simple cubic when N = K^3, FCC when N = 4K^3)
laid out in FRACTIONAL coordinates of the box, each site displaced by an
independent uniform jitter, then mapped to the lab frame by q = L_t lambda.
This is BASELINE.json's "seeded uniform in fractional coords" with a bounded
minimum pair distance, so LJ forces stay finite without any force-based
overlap removal (reading R21).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

RHO = 0.8442
WCA_RC = 2.0 ** (1.0 / 6.0)
CHUNK = 1 << 22


@dataclass
class Workload:
    name: str
    n: int
    L0: np.ndarray                 # reference basis (columns = box vectors)
    A: np.ndarray                  # flow matrix
    policy: str                    # none | le | kr | gkr
    t0: float
    L: np.ndarray                  # box at t0 (remapped representative)
    rc: float
    eps: float = 1.0
    sigma: float = 1.0
    mass: float = 1.0
    potential: str = "lj"
    dt: float = 0.002
    steps: int = 0
    prec: tuple = ("f64",)
    lattice: str = "sc"
    K: int = 0
    jitter: float = 0.0            # fraction of the site spacing (fractional units)
    seed: tuple = ()
    extra: dict = field(default_factory=dict)

    @property
    def ushift(self) -> float:
        s6 = (self.sigma / self.rc) ** 6
        return 4.0 * self.eps * (s6 * s6 - s6)


def rng_for(k: int, r: int = 0, stream: int = 0) -> np.random.Generator:
    """numpy PCG64 seeded by [1412, 3784, k, r, stream]."""
    return np.random.default_rng([1412, 3784, k, r, stream])


# ----------------------------------------------------------------- box parameters

def kr_basis(a: float):
    """Planar KR (reading R25): rows of the rotation are the unit
    eigenvectors of M = [[2,1],[1,1]], expanding eigenvector on x."""
    s5 = math.sqrt(5.0)
    lam = (3.0 + s5) / 2.0
    v1 = np.array([1.0, (lam - 2.0)])             # (M - lam I) v = 0 -> v = (1, lam-2)
    v1 /= np.linalg.norm(v1)
    v2 = np.array([-v1[1], v1[0]])
    L0 = np.eye(3) * a
    L0[0, :2] = a * v1
    L0[1, :2] = a * v2
    return L0, lam


def gkr_params(a: float):
    """Derived generalized-KR construction (reading R23): M1, M2 = (M1 - I)^2,
    L0 = a V^T (eigenvectors of M1 ascending along x, y, z; largest component
    positive; last row negated if det < 0), omega_k = log eig(M_k)."""
    M1 = np.array([[2.0, -1.0, -1.0], [-1.0, 2.0, 0.0], [-1.0, 0.0, 1.0]])
    M2 = (M1 - np.eye(3)) @ (M1 - np.eye(3))
    w, V = np.linalg.eigh(M1)
    for k in range(3):
        if V[np.argmax(np.abs(V[:, k])), k] < 0:
            V[:, k] *= -1.0
    B = V.T.copy()
    if np.linalg.det(B) < 0:
        B[2] *= -1.0
    om1 = np.log(w)
    om2 = np.log(np.array([(x - 1.0) ** 2 for x in w]))
    return M1, M2, a * B, om1, om2


def box_at(L0, A, policy, t, extra) -> np.ndarray:
    """Input box L~_{t0} for the chosen policy (closed forms of P:342, 369, 428, 433)."""
    if policy == "none":
        return np.array(L0, dtype=np.float64)
    if policy == "le":
        eps = A[0, 1]
        g = L0[0, 1] / L0[1, 1] + eps * t
        g -= math.floor(g + 0.5)
        L = np.array(L0, dtype=np.float64)
        L[0, 1] = g * L0[1, 1]
        return L
    if policy == "kr":
        ts = extra["tstar"]
        tt = t - math.floor(t / ts) * ts
        return np.diag(np.exp(np.diag(A) * tt)) @ L0
    if policy == "gkr":
        alpha = np.asarray(extra["beta"]) * extra["eps"] * t
        f = alpha - np.floor(alpha + 0.5)
        return np.diag(np.exp(f[0] * extra["om1"] + f[1] * extra["om2"])) @ L0
    raise ValueError(policy)


# ----------------------------------------------------------------- particles

FCC_BASIS = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])


def fractional_sites(lattice: str, K: int, lo: int, hi: int, Kz: int = 0) -> np.ndarray:
    """Fractional site coordinates for site ids [lo, hi): id = b + nb*(x + K*(y + K*z)); K x K x Kz
    lattice cells (Kz = K unless given: the weak-scaling boxes are elongated along v3)."""
    Kz = Kz or K
    nb = 4 if lattice == "fcc" else 1
    ids = np.arange(lo, hi, dtype=np.int64)
    b = ids % nb
    cell = ids // nb
    x = cell % K
    y = (cell // K) % K
    z = cell // (K * K)
    basis = FCC_BASIS if lattice == "fcc" else np.zeros((1, 3))
    lam = np.stack([x, y, z], axis=1).astype(np.float64) + basis[b]
    return lam / np.array([K, K, Kz], dtype=np.float64)


def positions(w: Workload, dtype=np.float64, k: int = 0, r: int = 0) -> np.ndarray:
    """Lab-frame positions q = L lambda, lambda = jittered lattice sites (R21).
    Generated in fixed chunks so the values do not depend on memory limits."""
    out = np.empty((w.n, 3), dtype=dtype)
    for c, lo in enumerate(range(0, w.n, CHUNK)):
        hi = min(w.n, lo + CHUNK)
        Kz = w.extra.get("Kz", w.K)
        lam = fractional_sites(w.lattice, w.K, lo, hi, Kz)
        g = rng_for(k, r, 1000 + c)
        lam += g.uniform(-w.jitter, w.jitter, size=lam.shape) / np.array([w.K, w.K, Kz], dtype=np.float64)
        lam -= np.floor(lam)  # sites stay in [0,1)^3 fractional
        q = lam[:, 0:1] * w.L[:, 0] + lam[:, 1:2] * w.L[:, 1] + lam[:, 2:3] * w.L[:, 2]
        out[lo:hi] = q.astype(dtype)
    return out


def uniform_positions(w: Workload, dtype=np.float64, k: int = 0, r: int = 0) -> np.ndarray:
    """Lab-frame positions q = L lambda with lambda uniform in [0,1)^3 ("positions seeded uniform in
    fractional coords", BASELINE configs 1-4, taken literally): the starting point of the overlap
    removal that bench.py runs through the library; no method arithmetic here."""
    out = np.empty((w.n, 3), dtype=dtype)
    for c, lo in enumerate(range(0, w.n, CHUNK)):
        hi = min(w.n, lo + CHUNK)
        lam = rng_for(k, r, 3000 + c).uniform(0.0, 1.0, size=(hi - lo, 3))
        q = lam[:, 0:1] * w.L[:, 0] + lam[:, 1:2] * w.L[:, 1] + lam[:, 2:3] * w.L[:, 2]
        out[lo:hi] = q.astype(dtype)
    return out


def momenta(w: Workload, dtype=np.float64, T: float = 1.0, k: int = 0, r: int = 0) -> np.ndarray:
    """Peculiar momenta: Gaussian at temperature T, zero net momentum (R24)."""
    out = np.empty((w.n, 3), dtype=np.float64)
    for c, lo in enumerate(range(0, w.n, CHUNK)):
        hi = min(w.n, lo + CHUNK)
        out[lo:hi] = rng_for(k, r, 5000 + c).normal(0.0, math.sqrt(T * w.mass), size=(hi - lo, 3))
    out -= out.mean(axis=0)
    return out.astype(dtype)


# ----------------------------------------------------------------- the five configs

def _side(n: int) -> float:
    return (n / RHO) ** (1.0 / 3.0)


def make(k: int, r: int = 0, *, flow: str = "uniaxial", scale: int = 1) -> Workload:
    """Config C<k> of BASELINE.json (0-based), replicate r.  `scale` shrinks the
    particle count by scale^3 (same density, same geometry class) for tests."""
    g = rng_for(k, r, 0)
    if k == 0:
        K = 10 // scale
        n = 4 * K ** 3
        a_fcc = (4.0 / RHO) ** (1.0 / 3.0)
        a = K * a_fcc                               # 16.796 sigma (reading R20)
        L0 = np.eye(3) * a
        A = np.zeros((3, 3))
        w = Workload("C0", n, L0, A, "none", 0.0, L0.copy(), 2.5, prec=("f64",), lattice="fcc", K=K,
                     jitter=0.05 / a_fcc, seed=(k, r))
        return w
    if k == 1:
        K = 20 // scale
        n = 4 * K ** 3
        a = _side(n)                                # 33.592 sigma
        gamma = g.uniform(-0.5, 0.5)
        eps = 1.0
        L0 = np.eye(3) * a
        L0[0, 1] = gamma * a
        A = np.zeros((3, 3)); A[0, 1] = eps
        return Workload("C1", n, L0, A, "le", 0.0, L0.copy(), WCA_RC, potential="wca", prec=("f32", "f64"),
                        lattice="fcc", K=K, jitter=0.05, seed=(k, r), steps=0)
    if k in (2, 4):
        K = (64 if k == 2 else 256) // scale
        lattice = "sc" if k == 2 else "fcc"
        n = K ** 3 * (4 if lattice == "fcc" else 1)
        a = _side(n)
        L0, lam = kr_basis(a)
        eps = 0.1
        A = np.diag([eps, -eps, 0.0])
        tstar = math.log(lam) / eps
        t0 = g.uniform(0.0, tstar)
        extra = {"tstar": tstar, "M": np.array([[2, 1, 0], [1, 1, 0], [0, 0, 1]])}
        L = box_at(L0, A, "kr", t0, extra)
        return Workload(f"C{k}", n, L0, A, "kr", t0, L, 2.5, prec=("f32",), lattice=lattice, K=K,
                        jitter=0.05, seed=(k, r), steps=100 if k == 2 else 50, extra=extra)
    if k == 3:
        K = 128 // scale
        n = K ** 3
        a = _side(n)
        M1, M2, L0, om1, om2 = gkr_params(a)
        eps = 0.1
        adiag = np.array([-1.0, -1.0, 2.0]) if flow == "uniaxial" else np.array([1.0, 1.0, -2.0])
        A = np.diag(eps * adiag)
        beta = np.linalg.lstsq(np.stack([om1, om2], axis=1), adiag, rcond=None)[0]
        dt = 0.002
        steps = 100
        # box highly skewed, with a reset of alpha_2 inside the run (reading R22)
        rate2 = beta[1] * eps
        tau2 = 1.0 / abs(rate2)
        ts = g.uniform(0.0, tau2)
        a2 = rate2 * ts
        if rate2 > 0:
            tx = (math.floor(a2 - 0.5) + 1.5) / rate2
        else:
            tx = (math.ceil(a2 + 0.5) - 1.5) / rate2
        t0 = tx - g.uniform(0.1, 0.9) * steps * dt
        extra = {"beta": beta, "eps": eps, "om1": om1, "om2": om2, "M1": M1, "M2": M2, "flow": flow}
        L = box_at(L0, A, "gkr", t0, extra)
        return Workload("C3" + ("u" if flow == "uniaxial" else "b"), n, L0, A, "gkr", t0, L, WCA_RC,
                        potential="wca", prec=("f32",), lattice="sc", K=K, jitter=0.05, seed=(k, r), steps=steps,
                        extra=extra)
    raise ValueError(k)


def make_weak(P: int, r: int = 0) -> Workload:
    """Weak-scaling workload: C4's construction with 8,388,608 particles per GPU --
    an FCC lattice of 128 x 128 x 128P cells in the KR box Rot diag(a, a, P a), a = 214.99 sigma
    (85.5 cell layers per GPU along v3, which the planar flow leaves untouched)."""
    w = make(4, r)
    K = 128
    a = _side(4 * K ** 3)
    L0, lam = kr_basis(a)
    L0[2, 2] = P * a
    w.L0 = L0
    w.K = K
    w.n = 4 * K * K * (K * P)
    w.extra = dict(w.extra, Kz=K * P)
    w.L = box_at(L0, w.A, "kr", w.t0, w.extra)
    w.name = f"C4w{P}"
    return w


def perfect_fcc(K: int = 10):
    """Zero-jitter C0 (the FCC pin): returns (q, L)."""
    w = make(0)
    w.K = K
    w.jitter = 0.0
    a_fcc = (4.0 / RHO) ** (1.0 / 3.0)
    w.L = np.eye(3) * (K * a_fcc)
    w.n = 4 * K ** 3
    return positions(w), w.L
