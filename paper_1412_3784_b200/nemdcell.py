"""Thin Python binding of the C-ABI in include/nemdcell.h (argument marshalling only).

Every function of the header is exposed under the same name; `CellList` is a
small convenience wrapper that owns one context and takes torch tensors or
numpy arrays.  All arithmetic of the path runs in libnemdcell.so (sm_100a);
there is no CPU fallback: if the library cannot be loaded, or no CUDA device
is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import build as _build

NC_DS, NC_DO = 0, 1
NC_F32, NC_F64 = 0, 1
NC_REMAP_NONE, NC_REMAP_LE, NC_REMAP_KR, NC_REMAP_GKR, NC_REMAP_REDUCE = 0, 1, 2, 3, 4
STATUS = {0: "NC_OK", 1: "NC_E_ARG", 2: "NC_E_BOX", 3: "NC_E_DEGENERATE", 4: "NC_E_FLOW", 5: "NC_E_STATE",
          6: "NC_E_CUDA", 7: "NC_E_NCCL", 8: "NC_E_OOM", 9: "NC_E_NONFINITE"}

EXPORTS = ["nc_create", "nc_destroy", "nc_set_box", "nc_set_flow", "nc_build_cells", "nc_compute_forces",
           "nc_compute_forces_async", "nc_compute_sync",
           "nc_set_state", "nc_step_sllod", "nc_get_state", "nc_get_cells", "nc_get_pair_digest", "nc_get_stats",
           "nc_get_stencil_histogram", "nc_launch_count", "nc_last_error", "nc_version", "nc_profile",
           "nc_profile_read", "nc_slab_layers", "nc_slab_kick_drift", "nc_slab_kick_kick_drift", "nc_slab_migrate",
           "nc_slab_unpack",
           "nc_slab_halo", "nc_slab_forces", "nc_slab_forces_begin", "nc_slab_forces_end", "nc_slab_kick",
           "nc_slab_reduce", "nc_set_pair_kernel",
           "nc_pair_kernel_used", "nc_get_pairs", "nc_get_cell_gids", "nc_get_pair_counts", "nc_debug",
           "nc_nccl_unique_id", "nc_slab_comm_init", "nc_slab_exchange_start", "nc_slab_exchange_wait",
           "nc_slab_exchange", "nc_slab_allgather", "nc_slab_layer_of",
           # host-synchronization-free slab step (csrc/slab_dc.cuh)
           "nc_sd_load", "nc_sd_status", "nc_sd_kick_drift", "nc_sd_kick", "nc_sd_migrate", "nc_sd_absorb",
           "nc_sd_halo", "nc_sd_exchange_start", "nc_sd_forces_begin", "nc_sd_forces_end",
           "nc_sd_forces_end_sorted",
           # peer-memory data plane (csrc/ipc_slab.cuh)
           "nc_ipc_alloc", "nc_ipc_open", "nc_ipc_event", "nc_ipc_event_open", "nc_ipc_record", "nc_ipc_wait"]
NC_DBG_DROP_ENTRIES = 1
NC_PK_AUTO, NC_PK_CELL, NC_PK_SEGMENT, NC_PK_SPARSE, NC_PK_ROWS = 0, 1, 2, 3, 4
PAIR_KERNELS = {"auto": NC_PK_AUTO, "cell": NC_PK_CELL, "segment": NC_PK_SEGMENT, "sparse": NC_PK_SPARSE, "rows": NC_PK_ROWS}
KERNEL_IDS = ["wrap_key", "scan", "scatter", "rank_gather", "pairs", "reduce", "kick", "other"]


class NcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class nc_config(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("prec", ctypes.c_int), ("rc", ctypes.c_double),
                ("eps", ctypes.c_double), ("sigma", ctypes.c_double), ("u_shift", ctypes.c_double),
                ("mass", ctypes.c_double), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("capacity", ctypes.c_int64), ("max_cells", ctypes.c_int64)]


class nc_remap(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("L0", ctypes.c_double * 9), ("tstar", ctypes.c_double),
                ("omega1", ctypes.c_double * 3), ("omega2", ctypes.c_double * 3), ("beta", ctypes.c_double * 2),
                ("eps", ctypes.c_double)]


NPART = 13  # per-layer partials: U, W0..W5, interactions, candidates, stencil cells, rechecks, fp32-tier interactions, non-finite


class nc_stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("dims", ctypes.c_int32 * 3), ("ncells", ctypes.c_int64),
                ("candidates", ctypes.c_double), ("interactions", ctypes.c_double),
                ("stencil_cells", ctypes.c_double), ("rechecks", ctypes.c_double), ("U", ctypes.c_double),
                ("W", ctypes.c_double * 6), ("acc_evals", ctypes.c_double), ("acc_interactions", ctypes.c_double),
                ("acc_candidates", ctypes.c_double), ("interactions_fp32", ctypes.c_double),
                ("acc_interactions_fp32", ctypes.c_double)]


_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libnemdcell.so (building it with nvcc if missing or stale)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and _build.stale():
            _build.build()
        path = os.environ.get("NC_LIB") or _build.LIB  # NC_LIB: an alternative build (A/B experiments)
        if not os.path.exists(path):
            raise ImportError(f"libnemdcell.so not found at {path}; run paper_1412_3784_b200.build.build()")
        L = ctypes.CDLL(path)
        vp, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.nc_create.argtypes = [ctypes.POINTER(nc_config), ctypes.POINTER(vp)]
        L.nc_destroy.argtypes = [vp]
        L.nc_destroy.restype = None
        L.nc_set_box.argtypes = [vp, vp]
        L.nc_set_flow.argtypes = [vp, vp, ctypes.POINTER(nc_remap), d]
        L.nc_build_cells.argtypes = [vp, vp, i64]
        L.nc_compute_forces.argtypes = [vp, vp, i64, vp, vp, vp]
        L.nc_compute_forces_async.argtypes = [vp, vp, i64, vp]
        L.nc_compute_sync.argtypes = [vp, vp, vp]
        L.nc_set_state.argtypes = [vp, vp, vp, vp, i64]
        L.nc_step_sllod.argtypes = [vp, d, i32, vp, vp]
        L.nc_get_state.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.nc_get_cells.argtypes = [vp, vp, vp, vp, vp]
        L.nc_get_pair_digest.argtypes = [vp, vp, vp, vp]
        L.nc_get_stats.argtypes = [vp, ctypes.POINTER(nc_stats)]
        L.nc_get_pairs.argtypes = [vp, i64, vp, vp]
        L.nc_get_cell_gids.argtypes = [vp, vp]
        L.nc_get_pair_counts.argtypes = [vp, vp]
        L.nc_debug.argtypes = [vp, i32, i32]
        L.nc_nccl_unique_id.argtypes = [vp]
        L.nc_slab_comm_init.argtypes = [vp, i32, i32, vp]
        L.nc_slab_exchange_start.argtypes = [vp, vp, i64, vp, i64, vp, vp, i64, i32, vp]
        L.nc_slab_exchange_wait.argtypes = [vp]
        L.nc_slab_exchange.argtypes = [vp, vp, i64, vp, i64, vp, vp, i64, i32, vp]
        L.nc_slab_allgather.argtypes = [vp, vp, i64, i64, vp]
        L.nc_slab_layer_of.argtypes = [vp, vp, i64, vp]
        L.nc_get_stencil_histogram.argtypes = [vp, vp]
        L.nc_profile.argtypes = [vp, i32]
        L.nc_profile_read.argtypes = [vp, vp, vp]
        L.nc_slab_layers.argtypes = [vp, i32, i32, vp, vp, vp]
        L.nc_slab_kick_drift.argtypes = [vp, vp, vp, vp, i64, d]
        L.nc_slab_kick_kick_drift.argtypes = [vp, vp, vp, vp, i64, d, d]
        L.nc_slab_migrate.argtypes = [vp, vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, i64, vp]
        L.nc_slab_unpack.argtypes = [vp, vp, i64, vp, vp, vp]
        L.nc_slab_halo.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, i64, vp]
        L.nc_slab_forces.argtypes = [vp, vp, vp, i64, vp, i64, vp, i64, i32, i32, vp, vp]
        L.nc_slab_forces_begin.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32]
        L.nc_slab_forces_end.argtypes = [vp, vp, vp, vp, vp]
        L.nc_slab_kick.argtypes = [vp, vp, vp, i64, d]
        L.nc_slab_reduce.argtypes = [vp, vp, i32, vp, vp, vp]
        L.nc_sd_load.argtypes = [vp, i64]
        L.nc_sd_status.argtypes = [vp, vp, vp]
        L.nc_sd_kick_drift.argtypes = [vp, vp, vp, vp, i64, d, d]
        L.nc_sd_kick.argtypes = [vp, vp, vp, i64, d]
        L.nc_sd_migrate.argtypes = [vp, vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, i64]
        L.nc_sd_absorb.argtypes = [vp, vp, vp, i64, vp, vp, vp, i64]
        L.nc_sd_halo.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, i64]
        L.nc_sd_exchange_start.argtypes = [vp, vp, vp, vp, vp, i64, i32]
        L.nc_sd_forces_begin.argtypes = [vp, vp, vp, i64, i64, i32, i32]
        L.nc_sd_forces_end.argtypes = [vp, vp, vp, vp, vp]
        L.nc_sd_forces_end_sorted.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.nc_ipc_alloc.argtypes = [vp, i64, ctypes.POINTER(vp), vp]
        L.nc_ipc_open.argtypes = [vp, vp, ctypes.POINTER(vp)]
        L.nc_ipc_event.argtypes = [vp, vp, ctypes.POINTER(i32)]
        L.nc_ipc_event_open.argtypes = [vp, vp, ctypes.POINTER(i32)]
        L.nc_ipc_record.argtypes = [vp, i32]
        L.nc_ipc_wait.argtypes = [vp, i32]
        L.nc_launch_count.argtypes = [vp]
        L.nc_launch_count.restype = i64
        L.nc_set_pair_kernel.argtypes = [vp, i32]
        L.nc_pair_kernel_used.argtypes = [vp]
        L.nc_pair_kernel_used.restype = i32
        L.nc_last_error.argtypes = [vp]
        L.nc_last_error.restype = ctypes.c_char_p
        L.nc_version.restype = ctypes.c_char_p
        for name in EXPORTS:
            if name not in ("nc_destroy", "nc_launch_count", "nc_last_error", "nc_version", "nc_pair_kernel_used"):
                getattr(L, name).restype = i32
        _lib = L
        return L


def _ptr(x):
    """Raw pointer of a torch tensor, numpy array or None."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensor must be contiguous"
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data_as(ctypes.c_void_p)
    if isinstance(x, ctypes.c_void_p):
        return x
    raise TypeError(type(x))


def _check(ctx, st):
    if st != 0:
        raise NcError(st, load().nc_last_error(ctx).decode())


def _d9(L):
    a = np.ascontiguousarray(np.asarray(L, dtype=np.float64).reshape(9))
    return a


# ----------------------------------------------------------------- same-name wrappers

def nc_version() -> str:
    return load().nc_version().decode()


def nc_create(cfg: nc_config):
    h = ctypes.c_void_p()
    _check(None, load().nc_create(ctypes.byref(cfg), ctypes.byref(h)))
    return h


def nc_destroy(ctx) -> None:
    load().nc_destroy(ctx)


def nc_set_box(ctx, L) -> None:
    a = _d9(L)
    _check(ctx, load().nc_set_box(ctx, _ptr(a)))


def nc_set_flow(ctx, A, pol: nc_remap | None, t: float) -> None:
    a = _d9(A)
    _check(ctx, load().nc_set_flow(ctx, _ptr(a), ctypes.byref(pol) if pol is not None else None, float(t)))


def nc_build_cells(ctx, q, n: int) -> None:
    _check(ctx, load().nc_build_cells(ctx, _ptr(q), int(n)))


def nc_compute_forces_async(ctx, q, n: int, F) -> None:
    _check(ctx, load().nc_compute_forces_async(ctx, _ptr(q), int(n), _ptr(F)))


def nc_compute_sync(ctx):
    U = ctypes.c_double(0.0)
    W = np.zeros(6)
    _check(ctx, load().nc_compute_sync(ctx, ctypes.byref(U), _ptr(W)))
    return U.value, W


def nc_compute_forces(ctx, q, n: int, F):
    U = ctypes.c_double()
    W = np.zeros(6)
    _check(ctx, load().nc_compute_forces(ctx, _ptr(q), int(n), _ptr(F), ctypes.byref(U), _ptr(W)))
    return U.value, W


def nc_set_state(ctx, q, p, gid, n: int) -> None:
    g = None if gid is None else np.ascontiguousarray(gid, dtype=np.int64)
    _check(ctx, load().nc_set_state(ctx, _ptr(q), _ptr(p), _ptr(g), int(n)))


def nc_step_sllod(ctx, dt: float, nsteps: int, want_uw: bool = True):
    U = ctypes.c_double()
    W = np.zeros(6)
    _check(ctx, load().nc_step_sllod(ctx, float(dt), int(nsteps), ctypes.byref(U) if want_uw else None,
                                     _ptr(W) if want_uw else None))
    return (U.value, W) if want_uw else None


def nc_get_state(ctx, q=None, p=None, want_gid=False):
    n = ctypes.c_int64()
    L = np.zeros(9)
    t = ctypes.c_double()
    _check(ctx, load().nc_get_state(ctx, None, None, None, ctypes.byref(n), _ptr(L), ctypes.byref(t)))
    gid = np.zeros(n.value, dtype=np.int64) if want_gid else None
    _check(ctx, load().nc_get_state(ctx, _ptr(q), _ptr(p), _ptr(gid), ctypes.byref(n), _ptr(L), ctypes.byref(t)))
    return n.value, L.reshape(3, 3), t.value, gid


def nc_get_cells(ctx, n: int, ncells: int, wrapped_dtype=None):
    cell_of = np.zeros(n, dtype=np.int64)
    cs = np.zeros(ncells + 1, dtype=np.int64)
    dims = np.zeros(3, dtype=np.int32)
    wq = np.zeros((n, 3), dtype=wrapped_dtype) if wrapped_dtype is not None else None
    _check(ctx, load().nc_get_cells(ctx, _ptr(cell_of), _ptr(cs), _ptr(dims), _ptr(wq)))
    return cell_of, cs, dims, wq


def nc_get_pair_digest(ctx, n: int):
    cnt = np.zeros(n, dtype=np.uint32)
    hs = np.zeros(n, dtype=np.uint64)
    hx = np.zeros(n, dtype=np.uint64)
    _check(ctx, load().nc_get_pair_digest(ctx, _ptr(cnt), _ptr(hs), _ptr(hx)))
    return cnt, hs, hx


def nc_get_pairs(ctx, cap: int = 1 << 20) -> np.ndarray:
    """Sorted (npairs, 5) int32 array: gid_i, gid_j, n1, n2, n3 of every ordered pair."""
    n = ctypes.c_int64()
    out = np.zeros((max(int(cap), 1), 5), dtype=np.int32)
    _check(ctx, load().nc_get_pairs(ctx, int(cap), _ptr(out), ctypes.byref(n)))
    return out[: n.value].copy()


def nc_get_cell_gids(ctx, n: int) -> np.ndarray:
    g = np.zeros(n, dtype=np.int64)
    _check(ctx, load().nc_get_cell_gids(ctx, _ptr(g)))
    return g


def nc_get_pair_counts(ctx, n: int) -> np.ndarray:
    c = np.zeros(n, dtype=np.uint32)
    _check(ctx, load().nc_get_pair_counts(ctx, _ptr(c)))
    return c


def nc_debug(ctx, what: int, value: int) -> None:
    _check(ctx, load().nc_debug(ctx, int(what), int(value)))


def nc_get_stats(ctx) -> dict:
    s = nc_stats()
    _check(ctx, load().nc_get_stats(ctx, ctypes.byref(s)))
    return {"n": s.n, "dims": tuple(s.dims), "ncells": s.ncells, "candidates": s.candidates,
            "interactions": s.interactions, "stencil_cells": s.stencil_cells, "rechecks": s.rechecks,
            "U": s.U, "W": np.array(list(s.W)), "acc_evals": s.acc_evals, "acc_interactions": s.acc_interactions,
            "acc_candidates": s.acc_candidates, "interactions_fp32": s.interactions_fp32,
            "acc_interactions_fp32": s.acc_interactions_fp32}


def nc_get_stencil_histogram(ctx) -> np.ndarray:
    h = np.zeros(64, dtype=np.int64)
    _check(ctx, load().nc_get_stencil_histogram(ctx, _ptr(h)))
    return h


def nc_set_pair_kernel(ctx, which) -> None:
    """Pair kernel of the context: "auto" | "cell" | "segment" | "sparse" | "rows" (or NC_PK_*)."""
    _check(ctx, load().nc_set_pair_kernel(ctx, PAIR_KERNELS.get(which, which) if isinstance(which, str) else int(which)))


def nc_pair_kernel_used(ctx) -> str:
    return {0: "none", 1: "cell", 2: "segment", 3: "sparse", 4: "rows"}[load().nc_pair_kernel_used(ctx)]


def nc_profile(ctx, enable) -> None:
    """enable: False / True, or the mode (3 = timing + fp32-tier interaction counts)."""
    mode = int(enable) if not isinstance(enable, bool) else (1 if enable else 0)
    _check(ctx, load().nc_profile(ctx, mode))


def nc_profile_read(ctx) -> dict:
    ms = np.zeros(8)
    cnt = np.zeros(8, dtype=np.int64)
    _check(ctx, load().nc_profile_read(ctx, _ptr(ms), _ptr(cnt)))
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_IDS)}


# ----------------------------------------------------------------- slab (multi-GPU) primitives

def nc_slab_layers(ctx, rank: int, nranks: int):
    lo, hi, l3 = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(ctx, load().nc_slab_layers(ctx, int(rank), int(nranks), ctypes.byref(lo), ctypes.byref(hi),
                                      ctypes.byref(l3)))
    return lo.value, hi.value, l3.value


def nc_slab_kick_drift(ctx, q, p, F, n: int, dt: float) -> None:
    _check(ctx, load().nc_slab_kick_drift(ctx, _ptr(q), _ptr(p), _ptr(F), int(n), float(dt)))


def nc_slab_migrate(ctx, q, p, gid, n, klo, khi, q_out, p_out, gid_out, send_lo, send_hi, cap):
    c = np.zeros(3, dtype=np.int64)
    _check(ctx, load().nc_slab_migrate(ctx, _ptr(q), _ptr(p), _ptr(gid), int(n), int(klo), int(khi), _ptr(q_out),
                                       _ptr(p_out), _ptr(gid_out), _ptr(send_lo), _ptr(send_hi), int(cap), _ptr(c)))
    return int(c[0]), int(c[1]), int(c[2])


def nc_slab_layer_of(ctx, q, n, layer) -> None:
    _check(ctx, load().nc_slab_layer_of(ctx, _ptr(q), int(n), _ptr(layer)))


def nc_slab_unpack(ctx, rec, n, q, p, gid) -> None:
    _check(ctx, load().nc_slab_unpack(ctx, _ptr(rec), int(n), _ptr(q), _ptr(p), _ptr(gid)))


def nc_slab_halo(ctx, q, gid, n, klo, khi, halo_lo, halo_hi, cap):
    c = np.zeros(2, dtype=np.int64)
    _check(ctx, load().nc_slab_halo(ctx, _ptr(q), _ptr(gid), int(n), int(klo), int(khi), _ptr(halo_lo),
                                    _ptr(halo_hi), int(cap), _ptr(c)))
    return int(c[0]), int(c[1])


def nc_slab_forces(ctx, q, gid, n_own, h_lo, n_lo, h_hi, n_hi, klo, khi, F, want_parts=True):
    parts = np.zeros((khi - klo, NPART)) if want_parts else None
    _check(ctx, load().nc_slab_forces(ctx, _ptr(q), _ptr(gid), int(n_own), _ptr(h_lo), int(n_lo), _ptr(h_hi),
                                      int(n_hi), int(klo), int(khi), _ptr(F), _ptr(parts)))
    return parts


def nc_slab_forces_begin(ctx, q, gid, n_own, n_lo, n_hi, klo, khi) -> None:
    _check(ctx, load().nc_slab_forces_begin(ctx, _ptr(q), _ptr(gid), int(n_own), int(n_lo), int(n_hi), int(klo),
                                            int(khi)))


def nc_slab_forces_end(ctx, h_lo, h_hi, F, klo, khi, want_parts=True):
    parts = np.zeros((khi - klo, NPART)) if want_parts else None
    _check(ctx, load().nc_slab_forces_end(ctx, _ptr(h_lo), _ptr(h_hi), _ptr(F), _ptr(parts)))
    return parts


def nc_slab_kick_kick_drift(ctx, q, p, F, n: int, dt_prev: float, dt: float) -> None:
    _check(ctx, load().nc_slab_kick_kick_drift(ctx, _ptr(q), _ptr(p), _ptr(F), int(n), float(dt_prev), float(dt)))


def nc_slab_kick(ctx, p, F, n, dt) -> None:
    _check(ctx, load().nc_slab_kick(ctx, _ptr(p), _ptr(F), int(n), float(dt)))


# ------------------------------------------------ host-synchronization-free slab step (csrc/slab_dc.cuh)
# Counts stay on the device: messages are (1 + cap)-record buffers whose record 0 carries the count;
# own particles are counted in the context.  nc_sd_status is the only call that reads anything back.

def nc_sd_load(ctx, n: int) -> None:
    _check(ctx, load().nc_sd_load(ctx, int(n)))


def nc_sd_status(ctx):
    """(own count, flags) -- synchronizes; raises NcError on an overflow / far move flag."""
    n = np.zeros(1, dtype=np.int64)
    f = np.zeros(1, dtype=np.uint32)
    _check(ctx, load().nc_sd_status(ctx, _ptr(n), _ptr(f)))
    return int(n[0]), int(f[0])


def nc_sd_kick_drift(ctx, q, p, F, ncap: int, dt_prev: float, dt: float) -> None:
    _check(ctx, load().nc_sd_kick_drift(ctx, _ptr(q), _ptr(p), _ptr(F), int(ncap), float(dt_prev), float(dt)))


def nc_sd_kick(ctx, p, F, ncap: int, dt: float) -> None:
    _check(ctx, load().nc_sd_kick(ctx, _ptr(p), _ptr(F), int(ncap), float(dt)))


def nc_sd_migrate(ctx, q, p, gid, ncap, klo, khi, q_out, p_out, gid_out, msg_lo, msg_hi, mcap) -> None:
    _check(ctx, load().nc_sd_migrate(ctx, _ptr(q), _ptr(p), _ptr(gid), int(ncap), int(klo), int(khi), _ptr(q_out),
                                     _ptr(p_out), _ptr(gid_out), _ptr(msg_lo), _ptr(msg_hi), int(mcap)))


def nc_sd_absorb(ctx, msg_lo, msg_hi, mcap, q, p, gid, ncap) -> None:
    _check(ctx, load().nc_sd_absorb(ctx, _ptr(msg_lo), _ptr(msg_hi), int(mcap), _ptr(q), _ptr(p), _ptr(gid),
                                    int(ncap)))


def nc_sd_halo(ctx, q, gid, ncap, klo, khi, msg_lo, msg_hi, hcap) -> None:
    _check(ctx, load().nc_sd_halo(ctx, _ptr(q), _ptr(gid), int(ncap), int(klo), int(khi), _ptr(msg_lo), _ptr(msg_hi),
                                  int(hcap)))


def nc_sd_exchange_start(ctx, send_lo, send_hi, recv_lo, recv_hi, cap, words) -> None:
    _check(ctx, load().nc_sd_exchange_start(ctx, _ptr(send_lo), _ptr(send_hi), _ptr(recv_lo), _ptr(recv_hi),
                                            int(cap), int(words)))


def nc_sd_forces_begin(ctx, q, gid, ncap, hcap, klo, khi) -> None:
    _check(ctx, load().nc_sd_forces_begin(ctx, _ptr(q), _ptr(gid), int(ncap), int(hcap), int(klo), int(khi)))


def nc_sd_forces_end(ctx, msg_lo, msg_hi, F, want_parts: bool, nlayers: int):
    parts = np.zeros((nlayers, NPART)) if want_parts else None
    _check(ctx, load().nc_sd_forces_end(ctx, _ptr(msg_lo), _ptr(msg_hi), _ptr(F),
                                        _ptr(parts) if parts is not None else None))
    return parts


def nc_sd_forces_end_sorted(ctx, msg_lo, msg_hi, p, q_out, p_out, gid_out, F, want_parts: bool, nlayers: int):
    parts = np.zeros((nlayers, NPART)) if want_parts else None
    _check(ctx, load().nc_sd_forces_end_sorted(ctx, _ptr(msg_lo), _ptr(msg_hi), _ptr(p), _ptr(q_out), _ptr(p_out),
                                               _ptr(gid_out), _ptr(F), _ptr(parts) if parts is not None else None))
    return parts


def nc_slab_reduce(ctx, parts: np.ndarray):
    parts = np.ascontiguousarray(parts, dtype=np.float64)
    U = ctypes.c_double()
    W = np.zeros(6)
    st = np.zeros(4)
    _check(ctx, load().nc_slab_reduce(ctx, _ptr(parts), int(parts.shape[0]), ctypes.byref(U), _ptr(W), _ptr(st)))
    return U.value, W, {"interactions": st[0], "candidates": st[1], "stencil_cells": st[2], "rechecks": st[3]}


def nc_ipc_alloc(ctx, nbytes: int):
    """A zeroed device buffer owned by ctx, exported: (raw pointer as c_void_p, 64-byte handle)."""
    p, h = ctypes.c_void_p(), (ctypes.c_uint8 * 64)()
    _check(ctx, load().nc_ipc_alloc(ctx, int(nbytes), ctypes.byref(p), h))
    return p, bytes(h)


def nc_ipc_open(ctx, handle: bytes):
    p, h = ctypes.c_void_p(), (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    _check(ctx, load().nc_ipc_open(ctx, h, ctypes.byref(p)))
    return p


def nc_ipc_event(ctx):
    """An interprocess event of ctx: (id, 64-byte handle)."""
    i, h = ctypes.c_int(), (ctypes.c_uint8 * 64)()
    _check(ctx, load().nc_ipc_event(ctx, h, ctypes.byref(i)))
    return i.value, bytes(h)


def nc_ipc_event_open(ctx, handle: bytes) -> int:
    i, h = ctypes.c_int(), (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    _check(ctx, load().nc_ipc_event_open(ctx, h, ctypes.byref(i)))
    return i.value


def nc_ipc_record(ctx, eid: int) -> None:
    _check(ctx, load().nc_ipc_record(ctx, int(eid)))


def nc_ipc_wait(ctx, eid: int) -> None:
    _check(ctx, load().nc_ipc_wait(ctx, int(eid)))


def nc_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(None, load().nc_nccl_unique_id(buf))
    return bytes(buf)


def nc_slab_comm_init(ctx, rank: int, nranks: int, uid: bytes) -> None:
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(ctx, load().nc_slab_comm_init(ctx, int(rank), int(nranks), buf))


def nc_slab_exchange_start(ctx, send_lo, n_lo, send_hi, n_hi, recv_lo, recv_hi, cap, words):
    c = np.zeros(2, dtype=np.int64)
    _check(ctx, load().nc_slab_exchange_start(ctx, _ptr(send_lo), int(n_lo), _ptr(send_hi), int(n_hi), _ptr(recv_lo),
                                              _ptr(recv_hi), int(cap), int(words), _ptr(c)))
    return int(c[0]), int(c[1])


def nc_slab_exchange_wait(ctx) -> None:
    _check(ctx, load().nc_slab_exchange_wait(ctx))


def nc_slab_exchange(ctx, send_lo, n_lo, send_hi, n_hi, recv_lo, recv_hi, cap, words):
    c = np.zeros(2, dtype=np.int64)
    _check(ctx, load().nc_slab_exchange(ctx, _ptr(send_lo), int(n_lo), _ptr(send_hi), int(n_hi), _ptr(recv_lo),
                                        _ptr(recv_hi), int(cap), int(words), _ptr(c)))
    return int(c[0]), int(c[1])


def nc_slab_allgather(ctx, local: np.ndarray, max_rows: int, nranks: int) -> np.ndarray:
    local = np.ascontiguousarray(local, dtype=np.float64).reshape(-1, NPART)
    out = np.zeros((nranks * max_rows, NPART))
    _check(ctx, load().nc_slab_allgather(ctx, _ptr(local) if len(local) else None, len(local), int(max_rows),
                                         _ptr(out)))
    return out


def nc_launch_count(ctx) -> int:
    return int(load().nc_launch_count(ctx))


def nc_last_error(ctx) -> str:
    return load().nc_last_error(ctx).decode()


# ----------------------------------------------------------------- convenience

def make_remap(policy: str, L0, tstar=0.0, om1=None, om2=None, beta=None, eps=0.0) -> nc_remap | None:
    kinds = {"none": NC_REMAP_NONE, "le": NC_REMAP_LE, "kr": NC_REMAP_KR, "gkr": NC_REMAP_GKR,
             "reduce": NC_REMAP_REDUCE}
    r = nc_remap()
    r.kind = kinds[policy]
    for k, v in enumerate(_d9(L0)):
        r.L0[k] = v
    r.tstar = float(tstar or 0.0)
    if om1 is not None:
        for k in range(3):
            r.omega1[k] = float(om1[k])
            r.omega2[k] = float(om2[k])
    if beta is not None:
        r.beta[0], r.beta[1] = float(beta[0]), float(beta[1])
    r.eps = float(eps)
    return r


class CellList:
    """One nemdcell context: variant 'ds'|'do', precision 'f32'|'f64'."""

    def __init__(self, variant="do", prec="f32", rc=2.5, eps=1.0, sigma=1.0, u_shift=None, mass=1.0,
                 capacity=1 << 16, max_cells=0, device=0, stream=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("nemdcell needs a CUDA device (B200, sm_100a); no CPU fallback")
        load()
        if u_shift is None:
            s6 = (sigma / rc) ** 6
            u_shift = 4.0 * eps * (s6 * s6 - s6)
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        cfg = nc_config()
        cfg.variant = NC_DS if variant == "ds" else NC_DO
        cfg.prec = NC_F32 if prec == "f32" else NC_F64
        cfg.rc, cfg.eps, cfg.sigma, cfg.u_shift, cfg.mass = rc, eps, sigma, u_shift, mass
        cfg.device = device
        cfg.stream = ctypes.c_void_p(stream)
        cfg.capacity = int(capacity)
        cfg.max_cells = int(max_cells)
        self.cfg = cfg
        self.prec = prec
        self.dtype = torch.float32 if prec == "f32" else torch.float64
        self.np_dtype = np.float32 if prec == "f32" else np.float64
        self.device = device
        self.ctx = nc_create(cfg)

    def close(self):
        if getattr(self, "ctx", None):
            nc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _arr3(self, x, name):
        """Refuse arrays whose dtype or shape does not match the context (the C-ABI reads
        n x 3 elements of the context precision through a raw pointer)."""
        if x is None:
            return x
        dt = getattr(x, "dtype", None)
        ok = dt in (self.dtype, self.np_dtype) or (isinstance(x, np.ndarray) and x.dtype == self.np_dtype)
        if not ok:
            raise TypeError(f"{name}: dtype {dt} does not match the context precision {self.prec}")
        if len(x.shape) != 2 or x.shape[1] != 3:
            raise ValueError(f"{name}: shape {tuple(x.shape)} is not (n, 3)")
        return x

    def set_box(self, L):
        nc_set_box(self.ctx, L)

    def set_flow(self, A, policy="none", t=0.0, **kw):
        r = make_remap(policy, kw.pop("L0"), **kw) if policy != "none" or "L0" in kw else None
        nc_set_flow(self.ctx, A, r, t)

    def build_cells(self, q):
        self._arr3(q, "q")
        nc_build_cells(self.ctx, q, q.shape[0])

    def compute_forces(self, q, F=None):
        import torch

        self._arr3(q, "q")
        if F is None:
            F = torch.empty_like(q) if hasattr(q, "data_ptr") and not isinstance(q, np.ndarray) else np.empty_like(q)
        self._arr3(F, "F")
        if F.shape[0] != q.shape[0]:
            raise ValueError("F must have the shape of q")
        U, W = nc_compute_forces(self.ctx, q, q.shape[0], F)
        return F, U, W

    def compute_forces_async(self, q, F):
        """Enqueue one evaluation on host buffers (pinned: copies overlap neighbouring calls)."""
        self._arr3(q, "q")
        self._arr3(F, "F")
        nc_compute_forces_async(self.ctx, q, q.shape[0], F)

    def compute_sync(self):
        """Wait for the pending evaluations; U, W of the last one."""
        return nc_compute_sync(self.ctx)

    def set_state(self, q, p=None, gid=None):
        self._arr3(q, "q")
        self._arr3(p, "p")
        if p is not None and p.shape[0] != q.shape[0]:
            raise ValueError("p must have the shape of q")
        nc_set_state(self.ctx, q, p, gid, q.shape[0])

    def step(self, dt, nsteps=1, want_uw=True):
        return nc_step_sllod(self.ctx, dt, nsteps, want_uw)

    def get_state(self, q=None, p=None, want_gid=False):
        return nc_get_state(self.ctx, q, p, want_gid)

    def cells(self, n, ncells, wrapped=True):
        return nc_get_cells(self.ctx, n, ncells, self.np_dtype if wrapped else None)

    def digest(self, n):
        return nc_get_pair_digest(self.ctx, n)

    def pairs(self, cap=1 << 20):
        return nc_get_pairs(self.ctx, cap)

    def cell_gids(self, n):
        return nc_get_cell_gids(self.ctx, n)

    def pair_counts(self, n):
        return nc_get_pair_counts(self.ctx, n)

    def debug_drop_entries(self, on=True):
        nc_debug(self.ctx, NC_DBG_DROP_ENTRIES, 1 if on else 0)

    def stats(self):
        return nc_get_stats(self.ctx)

    def stencil_histogram(self):
        return nc_get_stencil_histogram(self.ctx)

    def pair_kernel(self, which="auto"):
        nc_set_pair_kernel(self.ctx, which)

    def pair_kernel_used(self):
        return nc_pair_kernel_used(self.ctx)

    def profile(self, enable=True):
        nc_profile(self.ctx, enable)

    def profile_read(self):
        return nc_profile_read(self.ctx)

    def launches(self):
        return nc_launch_count(self.ctx)
