"""Oracle part 2: box evolution, lattice remapping and the SLLOD map (plain numpy fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Box evolution dL/dt = A L, L_t = e^{At} L_0                  (Eqs. 4-5)
* Lees-Edwards shear remap with M = [[1,-1,0],[0,1,0],[0,0,1]]
  applied at half a lattice spacing (max angle 26.57 deg)      (Eqs. 6-8)
* Kraynik-Reinelt planar elongation: e^{At*} L_0 = L_0 M       (Eq. 9)
* generalized KR for diagonal 3D flows: L~_t = exp(diag(eps_t)) L_0 with the
  stretch confined to a bounded set, via a pair of commuting automorphisms
  (Eq. 10).  The construction itself is in [dobs14], absent here;
  reading R23 derives one: M1 = [[2,-1,-1],[-1,2,0],[-1,0,1]],
  M2 = (M1 - I)^2, L_0 = a V^T with V the eigenvectors of M1, centered
  representative f_k = alpha_k - floor(alpha_k + 1/2).
* general traceless A ("general three dimensional linear flows"): the
  lattice-reduction policy of reading R30 -- L_t = e^{A (t - t_r)} L_r, and
  whenever a box vector can be shortened by adding an integer multiple of
  another (greedy pairwise Lagrange reduction, a unimodular change of basis of
  the same lattice), L_r <- the reduced basis, t_r <- t.  For shear it
  reproduces the Lees-Edwards reset at half a lattice spacing.
* SLLOD velocity-Verlet map on peculiar momenta (reading R19; the paper states
  only dq/dt = p/m and image consistency).
"""
from __future__ import annotations

import math

import numpy as np

# ------------------------------------------------------------------ flows


def is_diagonal(A) -> bool:
    A = np.asarray(A, dtype=np.float64)
    return bool(np.all(A == np.diag(np.diag(A))))


def expm(A, s: float) -> np.ndarray:
    """e^{A s}.  Diagonal: elementwise exp; nilpotent (A^2 = 0, e.g. shear,
    P:352): exactly I + A s; otherwise scaling-and-squaring Taylor."""
    A = np.asarray(A, dtype=np.float64).reshape(3, 3)
    if is_diagonal(A):
        return np.diag(np.exp(np.diag(A) * s))
    if np.all(A @ A == 0.0):
        return np.eye(3) + A * s
    X = A * s
    nrm = np.abs(X).sum(axis=1).max()
    k = max(0, int(math.ceil(math.log2(nrm))) + 4) if nrm > 0 else 0
    X = X / (2.0 ** k)
    E = np.eye(3)
    term = np.eye(3)
    for j in range(1, 30):
        term = term @ X / j
        E = E + term
    for _ in range(k):
        E = E @ E
    return E


def check_flow(A) -> None:
    """Incompressible linear flow: |tr A| <= 1e-12 max|A_ij| (SPEC-style check)."""
    A = np.asarray(A, dtype=np.float64)
    if abs(np.trace(A)) > 1e-12 * max(1.0, np.abs(A).max()):
        raise ValueError("flow matrix A must be traceless")


# ------------------------------------------------------------------ remap policies

M_SHEAR = np.array([[1, -1, 0], [0, 1, 0], [0, 0, 1]], dtype=np.int64)  # Eq. (8)
M_KR = np.array([[2, 1, 0], [1, 1, 0], [0, 0, 1]], dtype=np.int64)      # reading R25
M1_GKR = np.array([[2, -1, -1], [-1, 2, 0], [-1, 0, 1]], dtype=np.int64)  # reading R23


def kr_initial_basis(a: float):
    """KR planar elongation: L_0 = a (V^T (+) 1) whose rows are the
    unit eigenvectors of M = [[2,1],[1,1]], expanding one on x (R25).  Returns
    (L0, lam_max) with lam_max = (3+sqrt 5)/2 so that e^{eps t*} = lam_max."""
    w, V = np.linalg.eigh(M_KR[:2, :2].astype(np.float64))
    order = np.argsort(w)[::-1]          # expanding eigenvector first (x axis)
    V = V[:, order]
    for k in range(2):
        if V[np.argmax(np.abs(V[:, k])), k] < 0:
            V[:, k] *= -1
    B = V.T
    if np.linalg.det(B) < 0:
        B[1] *= -1
    L0 = np.eye(3) * a
    L0[:2, :2] = a * B
    return L0, float(w[order[0]])


def gkr_construction(a: float):
    """Derived generalized-KR construction (reading R23): returns
    (L0, omega1, omega2) with L0 M_k = diag(exp(omega_k)) L0, k = 1, 2."""
    M1 = M1_GKR.astype(np.float64)
    I = np.eye(3)
    M2 = (M1 - I) @ (M1 - I)
    w, V = np.linalg.eigh(M1)            # ascending eigenvalues along x, y, z
    for k in range(3):
        if V[np.argmax(np.abs(V[:, k])), k] < 0:
            V[:, k] *= -1
    B = V.T.copy()
    if np.linalg.det(B) < 0:
        B[2] *= -1
    L0 = a * B
    om1 = np.log(w)
    lam2 = np.diag(B @ M2 @ B.T)         # eigenvalues of M2 in the same order
    om2 = np.log(lam2)
    return L0, om1, om2


def gkr_beta(om1, om2, adiag):
    """beta solving [omega1 omega2] beta = a for traceless diagonal a (R23)."""
    Om = np.stack([om1, om2], axis=1)
    beta, *_ = np.linalg.lstsq(Om, np.asarray(adiag, dtype=np.float64), rcond=None)
    return beta


class Box:
    """Time-dependent, remapped simulation box L~_t for one flow and policy.

    policy 'none' : L_t = e^{At} L0
    policy 'le'   : shear A = eps e1 e2^T, L0 upper triangular; the tilt
                    gamma = gamma0 + eps t is kept in [-1/2, 1/2) by M
    policy 'kr'   : A = diag(eps, -eps, 0); L~_t = e^{A (t mod t*)} L0
    policy 'gkr'  : A = eps diag(a); alpha = beta eps t; f = alpha - floor(alpha+1/2);
                    L~_t = exp(diag(f1 om1 + f2 om2)) L0 (R23)
    """

    def __init__(self, L0, A, policy="none", t=0.0, om1=None, om2=None, beta=None, tstar=None, eps=None):
        self.L0 = np.array(L0, dtype=np.float64).reshape(3, 3)
        self.A = np.array(A, dtype=np.float64).reshape(3, 3)
        check_flow(self.A)
        self.policy = policy
        self.t = float(t)
        if policy == "reduce":  # R30: reduced basis Lr at time tr, L_t = e^{A (t - tr)} Lr
            self.Lr, _ = lattice_reduce(expm(self.A, self.t) @ self.L0)
            self.tr = self.t
        self.om1, self.om2 = om1, om2
        self.beta = beta
        self.tstar = tstar
        if policy == "kr" and tstar is None:
            eps = self.A[0, 0]
            self.tstar = math.log((3.0 + math.sqrt(5.0)) / 2.0) / eps
        if policy == "gkr":
            assert is_diagonal(self.A)
            # rate scale of A = eps diag(a): given with beta, else the largest |A_kk|
            self.eps = float(eps) if eps is not None else float(np.max(np.abs(np.diag(self.A))))
            if self.beta is None:
                self.beta = gkr_beta(self.om1, self.om2, np.diag(self.A) / self.eps)
        self.L = self.at(self.t)

    def at(self, t: float) -> np.ndarray:
        if self.policy == "none":
            return expm(self.A, t) @ self.L0
        if self.policy == "reduce":  # without committing a reduction (advance() commits)
            L, _ = lattice_reduce(expm(self.A, t - self.tr) @ self.Lr)
            return L
        if self.policy == "le":
            eps = self.A[0, 1]
            a_y = self.L0[1, 1]
            gamma0 = self.L0[0, 1] / a_y
            g = gamma0 + eps * t
            g = g - math.floor(g + 0.5)          # remap by M at half spacing
            L = self.L0.copy()
            L[0, 1] = g * a_y
            return L
        if self.policy == "kr":
            tt = t - math.floor(t / self.tstar) * self.tstar
            return expm(self.A, tt) @ self.L0
        if self.policy == "gkr":
            alpha = self.beta * self.eps * t
            f = alpha - np.floor(alpha + 0.5)
            return np.diag(np.exp(f[0] * self.om1 + f[1] * self.om2)) @ self.L0
        raise ValueError(self.policy)

    def advance(self, dt: float) -> np.ndarray:
        self.t += dt
        if self.policy == "reduce":
            L, changed = lattice_reduce(expm(self.A, self.t - self.tr) @ self.Lr)
            if changed:
                self.Lr, self.tr = L, self.t
            self.L = L
            return self.L
        self.L = self.at(self.t)
        return self.L


# ------------------------------------------------------------------ lattice reduction (R30)

REDUCE_PAIRS = ((0, 1), (0, 2), (1, 0), (1, 2), (2, 0), (2, 1))
REDUCE_MARGIN = 1e-12


def _dot(a, b) -> float:
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def lattice_reduce(L):
    """Greedy pairwise Lagrange reduction of the COLUMNS of L (reading R30):
    sweep the ordered pairs (i, j) = (0,1),(0,2),(1,0),(1,2),(2,0),(2,1); with
    mu = floor(v_i.v_j / v_j.v_j + 1/2), replace v_i by v_i - mu v_j when that
    is strictly shorter, |v_i - mu v_j|^2 < |v_i|^2 (1 - 1e-12); repeat sweeps
    until none changes.  Column operations of this kind keep the lattice and
    det L (M = L^-1 L' is integer with det +1).  Returns (L', changed)."""
    v = [np.array(L[:, k], dtype=np.float64) for k in range(3)]
    changed = False
    for _ in range(64):
        any_step = False
        for i, j in REDUCE_PAIRS:
            mu = math.floor(_dot(v[i], v[j]) / _dot(v[j], v[j]) + 0.5)
            if mu == 0:
                continue
            w = np.array([v[i][0] - mu * v[j][0], v[i][1] - mu * v[j][1], v[i][2] - mu * v[j][2]])
            if _dot(w, w) < _dot(v[i], v[i]) * (1.0 - REDUCE_MARGIN):
                v[i] = w
                any_step = True
        if not any_step:
            break
        changed = True
    return np.stack(v, axis=1), changed


# ------------------------------------------------------------------ SLLOD


def sllod_step(q, p, F, box: Box, dt: float, forces, mass: float = 1.0, prec: str = "f64"):
    """One step of the SLLOD velocity-Verlet map (reading R19):
        p <- E(-dt/2)(p + dt/2 F)
        q <- E(dt) q + dt E(dt/2) p / m
        L <- L~_{t+dt} (remapped); q <- wrap(q)   (wrapping leaves p, R19)
        F <- F(q)                                        (cell list rebuilt)
        p <- E(-dt/2) p + dt/2 F
    with E(s) = e^{A s}.  forces(q, L) -> (F, U, W).  Returns (q, p, F, U, W)."""
    from . import wrap as _wrap

    A = box.A
    Em = expm(A, -0.5 * dt)
    Ed = expm(A, dt)
    Eh = expm(A, 0.5 * dt)
    p = (p + 0.5 * dt * F) @ Em.T
    q = q @ Ed.T + dt * (p @ Eh.T) / mass
    if prec == "f32":
        q = q.astype(np.float32).astype(np.float64)
    L = box.advance(dt)
    q = _wrap(q, L, prec)
    F, U, W = forces(q, L)
    p = p @ Em.T + 0.5 * dt * F
    if prec == "f32":
        p = p.astype(np.float32).astype(np.float64)
    return q, p, F, U, W
