"""Seeded inputs that put many pairs exactly AT the cutoff (test fixtures only; no method arithmetic).

Positions and box entries are multiples of a power-of-two grid small enough that every stored value,
every lattice image q + L n of the LE box and every squared distance is exact in binary floating
point (grid 2^-18, |x| < 64: 24 significant bits).  A base displacement d0 on the grid fixes X0 = |d0|^2 exactly, and r_c is chosen so that
r_c * r_c == X0 in fp64: the 48 signed permutations of d0 then sit EXACTLY on the cutoff (strict
r^2 < r_c^2: not pairs, P:443 with reading R10), one grid step outward / inward on a component gives
r^2 = r_c^2 (1 +- ~2e-6), and a rescaled d0 gives r = r_c (1 +- 1e-6) up to the grid.  Pairs are placed
at random points of the box, about a third of them across a face, so the partner is stored as a
lattice image (the LE box keeps those exact too; KR / GKR boxes only approximately).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from paper_1412_3784_b200 import workloads as W


def base_displacement(rng, grid: float, rc_target: float):
    """d0 on the grid with rc * rc == |d0|^2 exactly for rc = sqrt(|d0|^2) (fp64)."""
    for _ in range(10000):
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        d0 = np.round(u * rc_target / grid) * grid
        X0 = (d0[0] * d0[0] + d0[1] * d0[1]) + d0[2] * d0[2]  # exact: every term is an integer times grid^2
        rc = math.sqrt(X0)
        if rc * rc == X0 and len(set(np.abs(d0))) == 3 and np.all(d0 != 0):
            return d0, rc
    raise RuntimeError("no exact base displacement")


def families(d0: np.ndarray, grid: float):
    """Displacement families: on the cutoff, one grid step out / in, and r_c (1 +- 1e-6) rescaled."""
    on = []
    for perm in itertools.permutations(range(3)):
        for sg in itertools.product((-1.0, 1.0), repeat=3):
            on.append(np.array([sg[k] * d0[perm[k]] for k in range(3)]))
    on = np.array(on)
    big = np.argmax(np.abs(on), axis=1)
    step = np.zeros_like(on)
    step[np.arange(len(on)), big] = np.sign(on[np.arange(len(on)), big]) * grid
    out1, in1 = on + step, on - step
    out6 = np.round(on * (1.0 + 1e-6) / grid) * grid
    in6 = np.round(on * (1.0 - 1e-6) / grid) * grid
    return np.concatenate([on, out1, in1, out6, in6])


def box(kind: str, a: float):
    if kind == "le":  # exact binary entries: a, gamma a with gamma = 3/8
        return np.array([[a, 0.375 * a, 0.0], [0.0, a, 0.0], [0.0, 0.0, a]])
    if kind == "kr":
        L0, lam = W.kr_basis(a)
        eps = 0.1
        t = 0.31 * math.log(lam) / eps
        return np.diag([math.exp(eps * t), math.exp(-eps * t), 1.0]) @ L0
    if kind == "gkr":
        _, _, L0, om1, om2 = W.gkr_params(a)
        return np.diag(np.exp(0.23 * om1 - 0.31 * om2)) @ L0
    raise ValueError(kind)


def edge_pairs(kind: str, npairs: int = 6000, seed: int = 0, rc_target: float = 1.1225, a: float = 10.0):
    """(L, rc, q fp64 [2 npairs, 3], d0): pairs (2k, 2k+1) at the constructed displacements."""
    rng = np.random.default_rng([1412, 3784, 77, seed])
    grid = 2.0 ** -18  # |x| < 64: 24 significant bits, exact in fp32 as well
    L = box(kind, a)
    d0, rc = base_displacement(rng, grid, rc_target)
    fam = families(d0, grid)
    Li = np.linalg.inv(L)
    q = np.empty((2 * npairs, 3))
    k = 0
    while k < npairs:
        lam = rng.uniform(0.0, 1.0, 3)
        if k % 3 == 0:  # a third of the pairs straddle a face: the partner is stored as an image
            ax = rng.integers(3)
            lam[ax] = rng.uniform(0.995, 1.0)
        qi = np.round((L @ lam) / grid) * grid
        li = Li @ qi
        if np.any(li < 0.0) or np.any(li >= 1.0):
            continue
        q[2 * k] = qi
        q[2 * k + 1] = qi + fam[rng.integers(len(fam))]
        k += 1
    return L, rc, q, d0


def rc_with_square(X: float, k: int):
    """An fp64 rc whose rounded square rc * rc is X + k ulp(X) (searching the neighbours of the
    correctly rounded root), or None."""
    target = X + k * math.ulp(X) if k >= 0 else X - (-k) * math.ulp(X)
    r = math.sqrt(target)
    for _ in range(8):
        s = r * r
        if s == target:
            return r
        r = math.nextafter(r, math.inf if s < target else -math.inf)
    return None
