"""CPU fp64 oracle for the cell-list force path of arXiv 1412.3784.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_1412_3784_b200``)
and neither imports the other.

Layout:
  * ``nemd_oracle.c``  -- geometry, wrap, cell keys, stencils, brute-force and
    cell-list pair sets, LJ/WCA forces, energy, virial, pair digests (plain
    fp64 C loops, ``-ffp-contract=off``).
  * ``box.py``         -- flow matrix exponentials, Lees-Edwards / KR /
    generalized-KR remapping, the SLLOD map (plain numpy fp64).

Every function cites the PAPER.md line it follows (P:n) or the DESIGN.md
reading (Rn) it takes where the paper is silent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nemd_oracle.c")
_SO = os.path.join(_HERE, "_nemd_oracle.so")
_lock = threading.Lock()
_lib = None

BRUTE, DS, DO = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (fp64, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
             "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            P = ctypes.POINTER
            d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
            vp = ctypes.c_void_p
            L.or_inv3.argtypes = [vp, vp, vp]
            L.or_heights.argtypes = [vp, vp]
            L.or_ds_dims.argtypes = [vp, d, vp]
            L.or_qr.argtypes = [vp, vp, vp]
            L.or_do_dims.argtypes = [vp, d, vp, vp]
            L.or_wrap.argtypes = [i64, vp, vp, i32]
            L.or_wrap.restype = i64
            L.or_cell_keys.argtypes = [i32, i64, vp, vp, d, vp, vp, vp]
            L.or_cell_sort.argtypes = [i64, vp, i64, vp, vp]
            L.or_stencil.argtypes = [i32, vp, d, vp, vp, vp]
            L.or_stencil_histogram.argtypes = [i32, vp, d, vp, vp]
            L.or_evaluate.argtypes = [i32, i64, vp, vp, d, d, d, d, i64, vp, vp, vp, vp, vp, vp, vp,
                                      vp, i64, vp, vp]
            L.or_do_rearrange.argtypes = [i64, vp, vp, vp, vp]
            L.or_num_threads.restype = i32
            del P
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _mat(L) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(L, dtype=np.float64).reshape(3, 3))


# ---------------------------------------------------------------- geometry
def inv3(L):
    """L^{-1} by adjugate/determinant (R16).  Returns (Linv, det)."""
    L = _mat(L)
    Li = np.zeros((3, 3))
    det = np.zeros(1)
    st = lib().or_inv3(_p(L), _p(Li), _p(det))
    if st:
        raise ValueError("box matrix has det <= 0 or is not finite (P:32)")
    return Li, float(det[0])


def heights(L) -> np.ndarray:
    """Face-to-face box heights h_k (R7)."""
    Li, _ = inv3(L)
    h = np.zeros(3)
    lib().or_heights(_p(Li), _p(h))
    return h


def ds_dims(L, rc) -> np.ndarray:
    """Dynamic-size cell counts c_k = floor(h_k/d_cut)."""
    h = heights(L)
    c = np.zeros(3, dtype=np.int32)
    lib().or_ds_dims(_p(h), float(rc), _p(c))
    return c


def qr(L):
    """Gram-Schmidt QR, r_kk > 0 (R8).  Returns (Q, R)."""
    L = _mat(L)
    Q = np.zeros((3, 3))
    R = np.zeros((3, 3))
    lib().or_qr(_p(L), _p(Q), _p(R))
    return Q, R


def do_dims(L, rc):
    """Dynamic-offset counts l_k = floor(r_kk/d_cut) and widths w_k = r_kk/l_k."""
    _, R = qr(L)
    l = np.zeros(3, dtype=np.int32)
    w = np.zeros(3)
    lib().or_do_dims(_p(R), float(rc), _p(l), _p(w))
    return l, w


def search_efficiency_equilibrium() -> float:
    """(4/3 pi)/27 (Eq. 13)."""
    return (4.0 / 3.0 * np.pi) / 27.0


def v_ds(L, rc) -> float:
    """DS neighborhood volume 27 V_box / (c1 c2 c3) (Eq. 14)."""
    c = ds_dims(L, rc)
    return 27.0 * abs(np.linalg.det(_mat(L))) / float(np.prod(c.astype(np.float64)))


def v_do_cell(L, rc) -> float:
    """DO cell volume r11 r22 r33/(l1 l2 l3) (Eq. 15)."""
    _, R = qr(L)
    l, _ = do_dims(L, rc)
    return float(R[0, 0] * R[1, 1] * R[2, 2] / np.prod(l.astype(np.float64)))


def do_average_count(l) -> float:
    """Average DO neighborhood size 27 + 14/l3 + 6/l2 - 4/(l2 l3) (R6)."""
    l1, l2, l3 = (float(x) for x in l)
    return 27.0 + 14.0 / l3 + 6.0 / l2 - 4.0 / (l2 * l3)


# ---------------------------------------------------------------- wrap / keys
def wrap(q, L, prec: str = "f64") -> np.ndarray:
    """Wrap positions into Omega once (R14, R15).  Returns a new fp64
    array holding the stored values (rounded to fp32 first if prec == 'f32')."""
    q = np.array(q, dtype=np.float64, order="C").reshape(-1, 3)
    L = _mat(L)
    lib().or_wrap(q.shape[0], _p(q), _p(L), 0 if prec == "f32" else 1)
    return q


def do_rearrange(xyz, R):
    """Rectangular rearrangement of rotated-frame points (Eqs. 11-12,
    reading R1: x is taken mod r11).  Returns (xyz', nhome)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    R = _mat(R)
    out = np.zeros_like(xyz)
    nh = np.zeros(xyz.shape, dtype=np.int32)
    lib().or_do_rearrange(xyz.shape[0], _p(xyz), _p(R), _p(out), _p(nh))
    return out, nh


def cell_keys(variant: int, q, L, rc):
    """Cell index per particle (x-fastest) and DO home shifts nh.
    variant: DS or DO.  Returns (cell int64[n], nhome int32[n,3], dims int32[3])."""
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
    L = _mat(L)
    n = q.shape[0]
    cell = np.zeros(n, dtype=np.int64)
    nh = np.zeros((n, 3), dtype=np.int32)
    dims = np.zeros(3, dtype=np.int32)
    st = lib().or_cell_keys(0 if variant == DS else 1, n, _p(q), _p(L), float(rc), _p(cell), _p(nh),
                            _p(dims))
    if st:
        raise ValueError({1: "bad box", 2: "degenerate grid"}[st])
    return cell, nh, dims


def cell_sort(cell, ncell: int):
    """Counting sort, ascending gid inside each cell (R27).  Returns (cell_start, order)."""
    cell = np.ascontiguousarray(cell, dtype=np.int64)
    cs = np.zeros(ncell + 1, dtype=np.int64)
    order = np.zeros(cell.shape[0], dtype=np.int64)
    lib().or_cell_sort(cell.shape[0], _p(cell), int(ncell), _p(cs), _p(order))
    return cs, order


def stencil(variant: int, L, rc, cell3):
    """Neighborhood (cell ids, lattice crossings) of one cell."""
    L = _mat(L)
    c3 = np.asarray(cell3, dtype=np.int32)
    cells = np.zeros(64, dtype=np.int64)
    nc = np.zeros((64, 3), dtype=np.int32)
    k = lib().or_stencil(0 if variant == DS else 1, _p(L), float(rc), _p(c3), _p(cells), _p(nc))
    if k < 0:
        raise ValueError("bad box or degenerate grid")
    return cells[:k].copy(), nc[:k].copy()


def stencil_histogram(variant: int, L, rc):
    """Histogram (index = neighborhood size) over all cells, and the grid dims."""
    L = _mat(L)
    hist = np.zeros(64, dtype=np.int64)
    dims = np.zeros(3, dtype=np.int32)
    st = lib().or_stencil_histogram(0 if variant == DS else 1, _p(L), float(rc), _p(hist), _p(dims))
    if st:
        raise ValueError({1: "bad box", 2: "degenerate grid"}[st])
    return hist, dims


# ---------------------------------------------------------------- potentials
def lj_shift(rc, eps=1.0, sigma=1.0) -> float:
    """phi_LJ(rc) = 4 eps ((sigma/rc)^12 - (sigma/rc)^6): the energy shift (R11)."""
    s6 = (sigma / rc) ** 6
    return 4.0 * eps * (s6 * s6 - s6)


WCA_RC = 2.0 ** (1.0 / 6.0)


# ---------------------------------------------------------------- evaluation
class Result(dict):
    __getattr__ = dict.__getitem__


def evaluate(method: int, q, L, rc, eps=1.0, sigma=1.0, ushift=None, idx=None, pairs_cap: int = 0,
             want=("F", "U", "W", "digest")) -> Result:
    """Pair set, forces, energy and virial by brute force (method BRUTE)
    or by the DS / DO cell list on the STORED positions q.

    Returns per-evaluated-particle F [k,3], U_i [k], W_i [k,6] (xx,yy,zz,xy,xz,yz),
    digests cnt/hsum/hxor, totals U = sum U_i, W = sum W_i, and stats
    (candidates, ordered interactions, grid dims)."""
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
    L = _mat(L)
    n = q.shape[0]
    if ushift is None:
        ushift = lj_shift(rc, eps, sigma)
    if idx is not None:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        k = idx.shape[0]
    else:
        k = n
    F = np.zeros((k, 3)) if "F" in want else None
    U = np.zeros(k) if "U" in want else None
    W = np.zeros((k, 6)) if "W" in want else None
    dig = "digest" in want
    cnt = np.zeros(k, dtype=np.uint32) if dig else None
    hsum = np.zeros(k, dtype=np.uint64) if dig else None
    hxor = np.zeros(k, dtype=np.uint64) if dig else None
    pairs = np.zeros((max(pairs_cap, 1), 5), dtype=np.int32) if pairs_cap else None
    npairs = np.zeros(1, dtype=np.int64)
    stats = np.zeros(7, dtype=np.int64)

    def P(a):
        return _p(a) if a is not None else None

    st = lib().or_evaluate(int(method), n, _p(q), _p(L), float(rc), float(eps), float(sigma), float(ushift),
                           k, P(idx), P(F), P(U), P(W), P(cnt), P(hsum), P(hxor), P(pairs), int(pairs_cap),
                           _p(npairs), _p(stats))
    if st:
        raise ValueError({1: "bad box (P:32)", 2: "degenerate grid (R9)"}[st])
    r = Result(F=F, U_i=U, W_i=W, cnt=cnt, hsum=hsum, hxor=hxor, candidates=int(stats[0]),
               interactions=int(stats[1]), dims=tuple(int(x) for x in stats[2:5]),
               t_build=stats[5] * 1e-9, t_eval=stats[6] * 1e-9)
    if U is not None:
        r["U"] = float(np.sum(U))
    if W is not None:
        r["W"] = W.sum(axis=0)
    if pairs_cap:
        m = int(npairs[0])
        if m > pairs_cap:
            raise ValueError(f"pair list overflow: {m} > cap {pairs_cap}")
        p = pairs[:m]
        order = np.lexsort((p[:, 4], p[:, 3], p[:, 2], p[:, 1], p[:, 0]))
        r["pairs"] = p[order]
    return r


def num_threads() -> int:
    return int(lib().or_num_threads())


from . import box  # noqa: E402,F401  (flow / remap / SLLOD, plain numpy)
